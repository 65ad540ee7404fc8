"""Pins of the CPU oracle against values fixed by the paper, SPEC worked examples,
closed forms, library routines and brute force (no GPU).  Each test names the
pin of SURVEY.md §8(c) it implements (P1..P14)."""
import json
import os

import numpy as np
import pytest
import torch

import synthgen as sg
from oracle import control as C
from oracle import model as M
from oracle.philox import gaussian_noise, philox4x32_10
from oracle.stream import StreamOracle, run_stream


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ P10 Philox
def test_philox_kat(golden_dir):
    rows = [l.split() for l in open(os.path.join(golden_dir, "philox_kat.txt")) if not l.startswith("#")]
    for r in rows:
        v = [int(x, 16) for x in r]
        out = philox4x32_10(v[0:4], v[4:6])
        assert [int(o) for o in out] == v[6:10]


def test_noise_counter_layout_and_box_muller():
    # element 0 of (X=0, j=0, seed=0) uses counter (0,0,0,0): the first KAT vector
    z = gaussian_noise(0, 0, 0, 8)
    u1 = (0x6627E8D5 + 0.5) / 2 ** 32
    u2 = (0xE169C58D + 0.5) / 2 ** 32
    assert z[0] == pytest.approx(np.sqrt(-2 * np.log(u1)) * np.cos(2 * np.pi * u2), abs=0, rel=1e-15)
    assert z[1] == pytest.approx(np.sqrt(-2 * np.log(u1)) * np.sin(2 * np.pi * u2), abs=0, rel=1e-15)
    # statistics: standard normal, independent of (X, j)
    big = gaussian_noise(12345, 7, 3, 400_000)
    assert abs(big.mean()) < 0.01 and abs(big.std() - 1) < 0.01
    other = gaussian_noise(12345, 7, 2, 400_000)
    assert abs(np.corrcoef(big, other)[0, 1]) < 0.01


# ------------------------------------------------------------------ P4 motion
def test_motion_intensity_closed_forms():
    r = np.random.default_rng(0)
    f = r.standard_normal((4, 8, 8))
    assert C.motion_intensity(f, f) == 0.0
    assert C.motion_intensity(f + 0.37, f) == pytest.approx(0.37, rel=1e-12)
    g = r.standard_normal((4, 8, 8))
    naive = 0.0
    for c in range(4):
        for y in range(8):
            for x in range(8):
                naive += (f[c, y, x] - g[c, y, x]) ** 2
    assert C.motion_intensity(f, g) == pytest.approx(np.sqrt(naive / 256), rel=1e-12)


def test_motion_spec_examples(golden_dir):
    ex = _golden(golden_dir, "spec_examples.json")
    for e in ex["normalized_motion"]:
        assert C.normalized_motion(e["ds"], e["sigma"]) == pytest.approx(e["expect"], abs=1e-12)
    for e in ex["ema_rate"]:
        assert C.ema_rate(e["d_hat"], e["s_prev"], e["s_min"], e["s_max"], e["lam"]) == pytest.approx(e["expect"], abs=1e-12)
    assert C.normalized_motion([0.0, 0.0], 0.3) == 0.0
    assert C.normalized_motion([0.6, 0.1], 0.3) == 1.0       # max d = 2 sigma -> clipped


def test_motion_invariants_random():
    """S:360-363 / S:580: bounds, EMA step bound, antitone, scale consistency."""
    r = np.random.default_rng(1)
    smin, smax = 0.4, 0.9
    for _ in range(2000):
        lam = r.uniform(0.01, 0.99)
        s = r.uniform(smin, smax)
        s2 = s
        for _ in range(5):
            dh = r.uniform(0, 1)
            dh2 = min(1.0, dh + r.uniform(0, 0.5))       # pointwise larger motion
            ns = C.ema_rate(dh, s, smin, smax, lam)
            ns2 = C.ema_rate(dh2, s2, smin, smax, lam)
            assert smin - 1e-12 <= ns <= smax + 1e-12
            assert abs(ns - s) <= lam * (smax - smin) + 1e-12
            assert ns2 <= ns + 1e-12
            s, s2 = ns, ns2
        ds = r.uniform(0, 2, size=9)
        sig = r.uniform(0.1, 2)
        assert C.normalized_motion(ds, sig) == pytest.approx(C.normalized_motion(2 * ds, 2 * sig), abs=1e-15)


def test_motion_controller_window_and_initial_state():
    sd = sg.StreamDesc((1000.0, 500.0), rope_reset_frames=4, motion_k=2, motion_sigma=0.5)
    mc = C.MotionController(sd)
    z = np.zeros((4, 1, 8, 8), np.float32)
    rec = mc.admit(z)                       # frame 0: d = 0 (Q15), s_{-1} = s_max
    assert rec["d"] == [0.0] and rec["d_hat"] == 0.0
    assert rec["s"] == pytest.approx(sd.s_max)
    seq = [0.0, 0.3, 0.0, 0.0, 0.0]         # a single jump
    prev = 0.0
    outs = []
    for d in seq[1:]:
        prev = prev + d                     # uniform shift => d exactly
        outs.append(mc.admit(z + np.float32(prev))["d_hat"])
    # window holds k+1 = 3 values: the jump is seen for 3 chunks then forgotten
    assert outs == pytest.approx([0.6, 0.6, 0.6, 0.0], abs=1e-6)
    assert rec["sigmas"][1] == pytest.approx(rec["s"] * 0.5, rel=1e-7)


# ------------------------------------------------------------ P2 RoPE / reset
def test_rope_position_examples(golden_dir):
    for e in _golden(golden_dir, "spec_examples.json")["rope_position"]:
        t = e["t_mult"] * e["T_reset"] + e["t_add"]
        assert C.rope_position(t, e["T_reset"]) == e["expect"]
    for t in range(0, 9):
        assert C.rope_position(t, 8) == t


def test_rope_identity_and_relative_invariance():
    hd = 64
    r = np.random.default_rng(2)
    x = r.standard_normal((5, hd))
    phi0 = M.rope_angles(hd, np.zeros(5), np.zeros(5), np.zeros(5))
    assert np.array_equal(M.rope_apply(x, phi0), x)
    q = r.standard_normal((1, hd))
    k = r.standard_normal((1, hd))
    for (pq, pk, sh) in [((10, 3, 4), (7, 1, 2), 500), ((3, 0, 0), (0, 0, 0), 77)]:
        a = M.rope_apply(q, M.rope_angles(hd, [pq[0]], [pq[1]], [pq[2]])) @ \
            M.rope_apply(k, M.rope_angles(hd, [pk[0]], [pk[1]], [pk[2]])).T
        b = M.rope_apply(q, M.rope_angles(hd, [pq[0] + sh], [pq[1]], [pq[2]])) @ \
            M.rope_apply(k, M.rope_angles(hd, [pk[0] + sh], [pk[1]], [pk[2]])).T
        assert a == pytest.approx(b, abs=1e-12)
    # group split (Wan: temporal d-4(d//6) dims, height/width 2(d//6)) -> pairs
    assert M.rope_split(128) == (22, 21, 21) and M.rope_split(64) == (12, 10, 10)
    # re-base: R(-D) R(p) k == R(p-D) k
    p, D = 300, 256
    rk = M.rope_apply(k, M.rope_angles(hd, [p], [1], [2]))
    rb = M.rope_apply(rk, M.rope_angles(hd, [-D], [0], [0]))
    assert rb == pytest.approx(M.rope_apply(k, M.rope_angles(hd, [p - D], [1], [2])), abs=1e-12)


# -------------------------------------------------------- P5 sink refresh
def test_sink_refresh_cases():
    h = np.array([1.0, 2.0, 3.0])
    sinks = [h.copy(), h.copy()]
    new, mask = C.sink_refresh(sinks, h, 0.95)
    assert mask == [False, False]
    new, mask = C.sink_refresh([np.array([1.0, 0, 0]), np.array([0, 1.0, 0])], np.array([0, 0, 5.0]), 0.1)
    assert mask == [True, True] and all(np.array_equal(s, [0, 0, 5.0]) for s in new)
    r = np.random.default_rng(3)
    hh = r.standard_normal(6)
    ss = [r.standard_normal(6) for _ in range(8)] + [hh * 2.0, hh + 0.01 * r.standard_normal(6)]
    new, mask = C.sink_refresh(ss, hh, 0.9)
    for s, mk in zip(ss, mask):
        c = sum(a * b for a, b in zip(s, hh)) / (np.sqrt(sum(a * a for a in s)) * np.sqrt(sum(b * b for b in hh)))
        assert mk == (c < 0.9)
    again, mask2 = C.sink_refresh(new, hh, 0.9)      # idempotent for repeated h
    assert mask2 == [False] * len(new)
    # tie alpha == tau keeps ("if alpha_i >= tau")
    _, m3 = C.sink_refresh([np.array([1.0, 0.0])], np.array([1.0, 0.0]), 1.0)
    assert m3 == [False]


# ------------------------------------------------- P3 metadata (Appendix A)
def _replay(geom, T_reset, tau, hs):
    ctl = C.ControlPlane(geom, T_reset, tau)
    lane = C.LaneCache(geom.sink_chunks, geom.window_chunks, T_reset)
    rows = []
    for X, h in enumerate(hs):
        act = ctl.admit(X, h)
        ev0 = lane.evictions
        lane.apply(act, None, None, geom.chunk_frames)
        st = lane.state()
        rows.append({"act": act, "state": st, "attended": [(e.tag, e.pos[0]) for e in lane.attended()],
                     "evict": lane.evictions, "new_evict": lane.evictions - ev0})
    return rows


def test_appendix_a_trace(golden_dir):
    g = _golden(golden_dir, "appendixA_trace.json")
    p = g["params"]
    geom = sg.Geometry(8, 8, p["T"], 2, p["m"], p["W"])
    hs = [p["h_before_6"] if X < 6 else p["h_from_6"] for X in range(8)]
    rows = _replay(geom, p["T_reset"], p["tau"], hs)
    for exp, got in zip(g["rows"], rows):
        act, st = got["act"], got["state"]
        assert act["pos"][0] == exp["qpos"] and act["r"] == exp["r"]
        assert act["rebase"] == exp["rebase"] and act["refresh"] == exp["refresh"]
        assert [list((st[i][0], st[i][1][0])) for i in range(p["m"])] == exp["sinks"]
        ring = [list((st[p["m"] + i][0], st[p["m"] + i][1][0])) if (p["m"] + i) in st else None for i in range(p["W"])]
        assert ring == exp["ring"]
        assert sorted(got["attended"], key=lambda t: (t[1], t[0])) == \
            sorted([tuple(a) for a in exp["attended"]], key=lambda t: (t[1], t[0]))
        assert got["evict"] == exp["evict"]


def test_kv_append_spec_example(golden_dir):
    e = _golden(golden_dir, "spec_examples.json")["kv_append"][0]
    geom = sg.Geometry(8, 8, 1, 1, e["m"], e["W"])
    rows = _replay(geom, 10 ** 6, -1.0, [np.array([1.0, 0.0])] * e["chunks"])
    st = rows[-1]["state"]
    assert sorted(st[i][0] for i in range(e["m"])) == e["expect_sinks"]
    assert sorted(st[i][0] for i in range(e["m"], e["m"] + e["W"])) == e["expect_ring"]
    assert rows[-1]["evict"] == e["expect_evictions"]
    # sinks never evicted; eviction count = max(0, inserted - free)
    for X, rw in enumerate(rows):
        assert [rw["state"][i][0] for i in range(e["m"]) if i in rw["state"]] == list(range(min(X + 1, e["m"])))
        assert rw["evict"] == max(0, (X + 1 - e["m"]) - e["W"])


# ----------------------------------------------- P1 ring path == brute force
def test_window_equals_bruteforce_definition():
    """The cache's attended set/positions == the definition: sinks = chunks 0..m-1 at
    their anchors, window = last W chunks at Y T' + f - r(X) T_reset (R3: relative
    distance to the query unchanged by resets)."""
    for (m, W, T, T_reset) in [(1, 2, 1, 4), (2, 3, 2, 6), (0, 4, 1, 5), (1, 4, 1, 240)]:
        geom = sg.Geometry(8, 8, T, 1, m, W)
        rows = _replay(geom, T_reset, -1.0, [np.array([1.0])] * 40)
        for X, rw in enumerate(rows):
            r = rw["act"]["r"]
            exp = [(i, i * T) for i in range(min(m, X + 1))]
            exp += [(Y, Y * T - r * T_reset) for Y in range(max(m, X - W + 1), X + 1) if Y >= m]
            assert sorted(rw["attended"]) == sorted(exp)
            # positions stay bounded for unbounded streams
            assert all(p <= T_reset + T - 1 for _, p in rw["attended"])


def test_streaming_attention_equals_full_attention():
    """window covering history == full attention; after eviction == full
    attention restricted to surviving tokens (masked)."""
    r = np.random.default_rng(4)
    hd, L = 16, 3
    ks = [r.standard_normal((L, hd)) for _ in range(7)]
    vs = [r.standard_normal((L, hd)) for _ in range(7)]
    q = r.standard_normal((L, hd))
    full = M.attention(q, np.concatenate(ks), np.concatenate(vs))
    geom = sg.Geometry(8, 8, 1, 1, 1, 8)
    ctl = C.ControlPlane(geom, 10 ** 6, -1.0)
    lane = C.LaneCache(1, 8, 10 ** 6)
    for X in range(7):
        lane.apply(ctl.admit(X, np.ones(1)), ks[X], vs[X], 1)
    ent = lane.attended()
    out = M.attention(q, np.concatenate([e.k for e in ent]), np.concatenate([e.v for e in ent]))
    assert out == pytest.approx(full, rel=1e-12, abs=1e-12)
    lane2 = C.LaneCache(1, 3, 10 ** 6)
    ctl2 = C.ControlPlane(sg.Geometry(8, 8, 1, 1, 1, 3), 10 ** 6, -1.0)
    for X in range(7):
        lane2.apply(ctl2.admit(X, np.ones(1)), ks[X], vs[X], 1)
    ent = lane2.attended()
    out2 = M.attention(q, np.concatenate([e.k for e in ent]), np.concatenate([e.v for e in ent]))
    s = q @ np.concatenate(ks).T / np.sqrt(hd)
    keep = np.zeros(7 * L, bool)
    for Y in (0, 4, 5, 6):
        keep[Y * L:(Y + 1) * L] = True
    s[:, ~keep] = -np.inf
    p = np.exp(s - s.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    assert out2 == pytest.approx(p @ np.concatenate(vs), rel=1e-12, abs=1e-12)


# ------------------------------------------------- P7 norms / activations
def test_norms_activations_attention_vs_torch():
    r = np.random.default_rng(5)
    x = r.standard_normal((6, 32))
    tx = torch.from_numpy(x)
    assert M.rms_norm(x, 1e-6) == pytest.approx(torch.nn.functional.rms_norm(tx, (32,), eps=1e-6).numpy(), rel=1e-12)
    assert M.layer_norm(x, 1e-6) == pytest.approx(torch.nn.functional.layer_norm(tx, (32,), eps=1e-6).numpy(), rel=1e-10, abs=1e-12)
    assert M.gelu_tanh(x) == pytest.approx(torch.nn.functional.gelu(tx, approximate="tanh").numpy(), rel=1e-12, abs=1e-15)
    assert M.silu(x) == pytest.approx(torch.nn.functional.silu(tx).numpy(), rel=1e-12, abs=1e-15)
    q, k, v = r.standard_normal((5, 16)), r.standard_normal((9, 16)), r.standard_normal((9, 16))
    ref = torch.nn.functional.scaled_dot_product_attention(torch.from_numpy(q)[None], torch.from_numpy(k)[None],
                                                           torch.from_numpy(v)[None])[0].numpy()
    out = M.attention(q, k, v)
    assert out == pytest.approx(ref, rel=1e-10, abs=1e-12)
    assert np.abs(M.attention(q, k[:1], v[:1]) - v[:1]).max() < 1e-15          # single key
    assert M.attention(np.zeros((2, 16)), k, v) == pytest.approx(np.tile(v.mean(0), (2, 1)), rel=1e-12)


# --------------------------------------------------------- P8 layouts
def test_patchify_is_conv3d_and_unpatchify_is_einsum():
    md = sg.TINY_MODEL
    r = np.random.default_rng(6)
    v = r.standard_normal((4, 1, 8, 8))
    w = r.standard_normal((md.dim, 16))
    b = r.standard_normal(md.dim)
    x = M.linear(M.patchify(v, md), w, b)
    conv = torch.nn.functional.conv3d(torch.from_numpy(v)[None], torch.from_numpy(w).reshape(md.dim, 4, 1, 2, 2),
                                      torch.from_numpy(b), stride=(1, 2, 2))[0]          # [d, 1, 4, 4]
    assert x == pytest.approx(conv.reshape(md.dim, -1).T.numpy(), rel=1e-10, abs=1e-12)
    y = r.standard_normal((16, 16))
    ref = torch.einsum("fhwpqrc->cfphqwr", torch.from_numpy(y).reshape(1, 4, 4, 1, 2, 2, 4)).reshape(4, 1, 8, 8)
    assert np.array_equal(M.unpatchify(y, md, 1, 8, 8), ref.numpy())


# ------------------------------------------------------ P11 time embedding
def test_time_embedding_t0():
    e = M.sinusoid(0.0, 256)
    assert np.array_equal(e, np.concatenate([np.ones(128), np.zeros(128)]))
    e = M.sinusoid(1000.0, 256)
    assert e[0] == pytest.approx(np.cos(1000.0)) and e[128] == pytest.approx(np.sin(1000.0))
    assert e[127] == pytest.approx(np.cos(1000.0 * 10000 ** (-127 / 128)))


# ---------------------------------------------------------- tiny fixtures
def _tiny():
    cfg = sg.CONFIGS["tiny"]
    W = sg.gen_weights(cfg.model, seed=0)
    ls = sg.LatentStream(4, 8, 8, seed=1, segment=3)
    chunks = [ls.chunk(X, 1) for X in range(cfg.num_chunks)]
    prompts = [sg.gen_prompt(cfg.model, 0), sg.gen_prompt(cfg.model, 1)]
    return cfg, W, chunks, prompts


# ------------------------------------------------------ P9 sampler wiring
def test_sampler_perfect_denoiser():
    cfg, W, chunks, prompts = _tiny()

    class Stub(StreamOracle):
        def dit(self, x_lat, sigma, j, act, taps=None):
            X = act["X"]
            eps = gaussian_noise(self.sd.seed, X, j, x_lat.size).reshape(x_lat.shape)
            return eps - self._v[X]

    o = Stub(cfg.model, cfg.geom, cfg.stream, W)
    o._v = chunks
    o.set_prompt(prompts[0])
    for X, v in enumerate(chunks):
        out = o.step_chunk(X, v)["out"]
        assert out == pytest.approx(v.astype(np.float64), abs=1e-12)


# --------------------------------------------------- P12 residual wiring
def test_identity_block():
    cfg, W, chunks, prompts = _tiny()
    W = dict(W)
    W["tp_w"] = np.zeros_like(W["tp_w"]); W["tp_b"] = np.zeros_like(W["tp_b"])
    for b in range(cfg.model.num_blocks):
        W[f"blocks.{b}.mod"] = W[f"blocks.{b}.mod"].copy()
        W[f"blocks.{b}.mod"][[2, 5]] = 0.0
        W[f"blocks.{b}.wco"] = np.zeros_like(W[f"blocks.{b}.wco"])
        W[f"blocks.{b}.bco"] = np.zeros_like(W[f"blocks.{b}.bco"])
    o = StreamOracle(cfg.model, cfg.geom, cfg.stream, W, tap=True)
    o.set_prompt(prompts[0])
    rec = o.step_chunk(0, chunks[0])
    e0 = rec["entries"][0]
    x_emb = M.linear(M.patchify(e0["x_in"], cfg.model), W["patch_w"].astype(np.float64), W["patch_b"].astype(np.float64))
    for t in e0["taps"]:
        assert np.array_equal(t, x_emb)


# ---------------------------------------------------------- P14 causality
def test_causality_and_determinism():
    cfg, W, chunks, prompts = _tiny()
    a = run_stream(cfg, W, chunks[:5], prompts)
    ch2 = [c.copy() for c in chunks[:5]]
    ch2[4] = ch2[4] + 1.0
    b = run_stream(cfg, W, ch2, prompts)
    for X in range(4):
        assert np.array_equal(a[X]["out"], b[X]["out"])
    assert not np.array_equal(a[4]["out"], b[4]["out"])
    c = run_stream(cfg, W, chunks[:5], prompts)
    for X in range(5):
        assert np.array_equal(a[X]["out"], c[X]["out"])


# --------------------------------------------- P6 order independence (O6)
def test_pipelined_order_equals_sequential():
    """Run entries in the R2 micro-batch order (K stages, mu = {(mu - jK, j)}) on the
    oracle components: per-entry math depends only on (X, j-1) and lane j's history,
    so results are bit-identical to the sequential order (O6)."""
    cfg, W, chunks, prompts = _tiny()
    seq = run_stream(cfg, W, chunks, prompts)
    n = cfg.geom.steps
    for K in (1, 2, 3):
        o = StreamOracle(cfg.model, cfg.geom, cfg.stream, W)
        acts, sig, xs, outs = {}, {}, {}, {}
        starts = [0, *cfg.prompt_switch]
        num = len(chunks)
        mu = 0
        while len(outs) < num:
            for j in range(n):
                X = mu - j * K
                if X < 0 or X >= num:
                    continue
                if j == 0:
                    if X in starts:
                        o.set_prompt(prompts[starts.index(X)])
                    mot = o.motion.admit(chunks[X])
                    acts[X] = o.admit_control(X)
                    sig[X] = mot["sigmas"]
                    s0 = np.float64(sig[X][0])
                    xs[X] = (1 - s0) * chunks[X].astype(np.float64) + s0 * gaussian_noise(
                        cfg.stream.seed, X, 0, chunks[X].size).reshape(chunks[X].shape)
                sj = np.float64(sig[X][j])
                vhat = o.dit(xs[X], sig[X][j], j, acts[X])
                x0 = xs[X] - sj * vhat
                if j < n - 1:
                    sn = np.float64(sig[X][j + 1])
                    xs[X] = (1 - sn) * x0 + sn * gaussian_noise(cfg.stream.seed, X, j + 1,
                                                                x0.size).reshape(x0.shape)
                else:
                    outs[X] = x0
            mu += 1
        for X in range(num):
            assert np.array_equal(outs[X], seq[X]["out"]), (K, X)


def test_tiny_stream_runs_and_refreshes():
    cfg, W, chunks, prompts = _tiny()
    recs = run_stream(cfg, W, chunks, prompts, tap=True)
    assert [r["act"]["refresh"] for r in recs][6] == [True]        # prompt switch at 6 (cos < tau)
    assert [r["act"]["rebase"] for r in recs] == [False] * 5 + [True, False, False]
    for r in recs:
        assert np.all(np.isfinite(r["out"]))
        assert 0.4 - 1e-12 <= r["motion"]["s"] <= 0.9 + 1e-12
