"""Pins of the clean-context re-run variant (reading Q5-clean; oracle side).

kv_mode 1: before chunk X is admitted, finished chunk X-1 goes through the DiT on its
prediction x0 at sigma = 0 (t = 0) and that pass's K/V replace its step-0 K/V in the cache
(CausVid's clean-context pass, EXT).  The pins fix it against things other than its own code:
  * with the noise rate forced to 0 the step input already is the clean latent and x0 = x, so
    the re-run repeats the denoising pass exactly: outputs and cache equal the R1 stream's,
    bit for bit (positions, slots, attended range, refresh and the t = 0 embedding all have to
    match for this to hold);
  * block 0's cached key of chunk X-1 is the block-0 key of x0_{X-1} at t = 0, recomputed
    from the model-card formulas (C.1, C.2, C.5 steps 1-2) outside the stream code;
  * the cache metadata (tags, positions per slot) never differs from R1's: the re-run only
    overwrites contents."""
import dataclasses

import numpy as np
import pytest

import synthgen as sg
from oracle import model as M
from oracle.stream import StreamOracle, run_stream


def _cfg(kv_mode, s=None):
    base = sg.CONFIGS["tiny"]
    g = dataclasses.replace(base.geom, steps=1, kv_mode=kv_mode)
    sd = dataclasses.replace(base.stream, timesteps=sg.SCHEDULES[1])
    if s is not None:
        sd = dataclasses.replace(sd, s_min=s, s_max=s)
    return dataclasses.replace(base, geom=g, stream=sd)


def _inputs(cfg):
    W = sg.gen_weights(cfg.model, seed=0)
    ls = sg.LatentStream(cfg.model.latent_channels, cfg.geom.latent_h, cfg.geom.latent_w, seed=1, segment=3)
    chunks = [ls.chunk(X, cfg.geom.chunk_frames) for X in range(cfg.num_chunks)]
    prompts = [sg.gen_prompt(cfg.model, k) for k in range(1 + len(cfg.prompt_switch))]
    return W, chunks, prompts


def test_clean_rerun_at_zero_noise_equals_step_lanes():
    r1, cl = _cfg(0, s=0.0), _cfg(1, s=0.0)
    W, chunks, prompts = _inputs(r1)
    a = run_stream(r1, W, chunks, prompts)
    b = run_stream(cl, W, chunks, prompts)
    assert any(r["act"]["rebase"] for r in a) and any(any(r["act"]["refresh"]) for r in a)   # exercised
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["out"], rb["out"]), ra["X"]
        assert ra["lane_state"] == rb["lane_state"]


def test_clean_rerun_key_is_block0_key_of_x0_at_t0():
    cfg = _cfg(1)
    W, chunks, prompts = _inputs(cfg)
    md = cfg.model
    o = StreamOracle(md, cfg.geom, cfg.stream, W)
    o.set_prompt(prompts[0])
    w = lambda n: W["blocks.0." + n].astype(np.float64)
    lane = o.lanes[(0, 0)]
    starts = [0, *cfg.prompt_switch]
    prompt_at = lambda X: prompts[starts.index(X)] if X in starts and X > 0 else None
    recs = [o.step_chunk(0, chunks[0])]
    assert any(any(r["act"]["refresh"]) for r in run_stream(cfg, W, chunks, prompts))   # a refresh happens
    for Y in range(cfg.num_chunks - 1):
        recs.append(o.step_chunk(Y + 1, chunks[Y + 1], prompt_at(Y + 1)))   # call Y + 1 re-ran chunk Y
        x = M.patchify(recs[Y]["out"], md) @ W["patch_w"].astype(np.float64).T + W["patch_b"]
        # C.2 at t = 0 (sigma = 0): e0 = W_tp SiLU(W_t2 SiLU(W_t1 sinusoid(0) + b) + b) + b
        emb = np.concatenate([np.ones(md.freq_dim // 2), np.zeros(md.freq_dim // 2)])   # cos 0, sin 0
        silu = lambda z: z / (1 + np.exp(-z))
        e = W["t2_w"].astype(np.float64) @ silu(W["t1_w"].astype(np.float64) @ emb + W["t1_b"]) + W["t2_b"]
        e0 = (W["tp_w"].astype(np.float64) @ silu(e) + W["tp_b"]).reshape(6, md.dim)
        mod = w("mod") + e0
        mu = x.mean(axis=1, keepdims=True) if md.norm_center else 0.0      # C.4 N(x)
        xn = (x - mu) / np.sqrt(((x - mu) ** 2).mean(axis=1, keepdims=True) + md.eps)
        a = xn * (1 + mod[1]) + mod[0]
        k = a @ w("wk").T + w("bk")
        k = w("gk") * k / np.sqrt((k ** 2).mean(axis=1, keepdims=True) + md.eps)
        ents = [e_ for e_ in ([s for s in lane.sinks if s is not None] + lane.window) if e_.tag == Y]
        assert ents, Y
        for e_ in ents:
            np.testing.assert_allclose(e_.k, k, rtol=1e-10, atol=1e-12)


def test_clean_rerun_changes_later_chunks_only():
    r1, cl = _cfg(0), _cfg(1)
    W, chunks, prompts = _inputs(r1)
    a = run_stream(r1, W, chunks, prompts)
    b = run_stream(cl, W, chunks, prompts)
    assert np.array_equal(a[0]["out"], b[0]["out"])          # nothing re-run before chunk 0
    for ra, rb in zip(a[1:], b[1:]):
        d = np.linalg.norm(ra["out"] - rb["out"]) / np.linalg.norm(ra["out"])
        assert d > 1e-6, ra["X"]
        assert ra["lane_state"] == rb["lane_state"]             # contents change, metadata never


def test_clean_rerun_needs_single_step():
    base = sg.CONFIGS["tiny"]
    g = dataclasses.replace(base.geom, kv_mode=1)               # n = 2
    with pytest.raises(ValueError):
        StreamOracle(base.model, g, base.stream, sg.gen_weights(base.model, seed=0))


def _mut_rerun(kind):
    """Misreadings of the clean re-run patched into StreamOracle.clean_rerun / LaneCache.overwrite."""
    from oracle import control as C

    def rerun(self, rec):
        md, dt, W = self.md, self.dt, self.W
        act = rec["act"]
        src = rec["entries"][0]["x_in"] if kind == "noisy_input" else rec["out"]
        u = M.patchify(src.astype(dt), md)
        x = M.linear(u, W["patch_w"].astype(dt), W["patch_b"].astype(dt))
        sig = rec["motion"]["sigmas"][0] if kind == "own_sigma" else np.float32(0.0)
        _, e0 = M.time_embed(sig, W, md, dt)
        for b in self.blocks:
            x = self.block(x, e0, b, self.lanes[(b, 0)], act, rerun=True)

    def overwrite_window_only(self, act, k, v):
        X = act["X"]
        if act["sink_fill"] >= 0:
            e = self.sinks[act["sink_fill"]]
        else:
            e = self.window[-1]
        assert e.tag == X
        e.k, e.v = k, v

    if kind == "window_only":
        return [(C.LaneCache, "overwrite", overwrite_window_only)]
    return [(StreamOracle, "clean_rerun", rerun)]


@pytest.mark.parametrize("kind", ["noisy_input", "own_sigma", "window_only"])
def test_pins_catch_rerun_misreadings(monkeypatch, kind):
    for obj, attr, rep in _mut_rerun(kind):
        monkeypatch.setattr(obj, attr, rep)
    with pytest.raises(AssertionError):
        test_clean_rerun_key_is_block0_key_of_x0_at_t0()
