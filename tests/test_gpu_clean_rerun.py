"""GPU path of the clean-context re-run (sdv2_geometry.kv_mode = 1; reading Q5-clean,
SURVEY §8(f) N4) vs the CPU oracle (oracle/stream.py, pinned in
tests/test_oracle_clean_rerun.py): per-block rel-L2 <= 1e-4 (fp32) / 2e-2 (bf16),
outputs likewise, cache metadata bit-exact."""
import dataclasses

import numpy as np
import pytest

import synthgen as sg
from oracle.stream import run_stream
from paper_2511_07399_b200.sdv2 import SDV2_BF16, SDV2_FP32

from gpu_harness import rel_l2, run_gpu, tiny_inputs

TOL = {SDV2_FP32: 1e-4, SDV2_BF16: 2e-2}


def _clean(cfg, kv_mode=1, s=None, **geom):
    g = dataclasses.replace(cfg.geom, steps=1, kv_mode=kv_mode, **geom)
    sd = dataclasses.replace(cfg.stream, timesteps=sg.SCHEDULES[1])
    if s is not None:
        sd = dataclasses.replace(sd, s_min=s, s_max=s)
    return dataclasses.replace(cfg, geom=g, stream=sd)


def _check(cfg, recs, outs, taps, meta, tol):
    worst = 0.0
    for (X, j), tl in taps.items():
        for b in range(cfg.model.num_blocks):
            err = rel_l2(tl[b], recs[X]["entries"][j]["taps"][b])
            worst = max(worst, err)
            assert err <= tol, (X, j, b, err)
    for X in range(cfg.num_chunks):
        assert rel_l2(outs[X], recs[X]["out"]) <= tol, X
    for (X, j), (slots, _, _) in meta.items():
        assert slots == {s: (t, p[0]) for s, (t, p) in recs[X]["lane_state"][(0, j)].items()}, (X, j)
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [SDV2_FP32, SDV2_BF16])
def test_tiny_clean_rerun_parity(prec):
    cfg = _clean(sg.CONFIGS["tiny"])
    W, chunks, prompts = tiny_inputs(cfg)
    recs = run_stream(cfg, W, chunks, prompts, dtype=np.float64, tap=True)
    assert any(r["act"]["rebase"] for r in recs) and any(any(r["act"]["refresh"]) for r in recs)
    outs, taps, meta = run_gpu(cfg, W, chunks, prompts, prec)
    worst = _check(cfg, recs, outs, taps, meta, TOL[prec])
    # the variant is not a no-op: the step-lane (R1) stream differs from chunk 1 on
    r1 = run_stream(_clean(sg.CONFIGS["tiny"], kv_mode=0), W, chunks, prompts, dtype=np.float64)
    assert rel_l2(recs[3]["out"], r1[3]["out"]) > 1e-3        # 10x the fp32 parity bar
    print(f"clean re-run prec={prec}: worst block rel-L2 {worst:.3e}")


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [SDV2_FP32, SDV2_BF16])
def test_clean_rerun_at_zero_noise_is_bitwise_step_lanes(prec):
    """sigma = 0: the re-run repeats the denoising pass (same input, t = 0, same slots and
    key range), so the library's clean-mode outputs equal its step-lane outputs bit for bit."""
    base = sg.CONFIGS["tiny"]
    W, chunks, prompts = tiny_inputs(base)
    a, _, _ = run_gpu(_clean(base, kv_mode=0, s=0.0), W, chunks, prompts, prec, tap=False)
    b, _, _ = run_gpu(_clean(base, kv_mode=1, s=0.0), W, chunks, prompts, prec, tap=False)
    assert sorted(a) == sorted(b)
    for X in a:
        assert np.array_equal(a[X], b[X]), X


@pytest.mark.gpu
def test_clean_rerun_graph_replay_equals_eager():
    cfg = _clean(sg.CONFIGS["tiny"])
    W, chunks, prompts = tiny_inputs(cfg)
    g, _, _ = run_gpu(cfg, W, chunks, prompts, SDV2_BF16, tap=False, graphs=True)
    e, _, _ = run_gpu(cfg, W, chunks, prompts, SDV2_BF16, tap=False, graphs=False)
    assert sorted(g) == sorted(e)
    for X in g:
        assert np.array_equal(g[X], e[X]), X


@pytest.mark.gpu
def test_clean_rerun_full_width_bf16():
    """1.3B-shaped blocks at 480p (L = 1560), 2 blocks, prompt switch + RoPE re-base inside."""
    base = sg.CONFIGS["wan13_480p_1step"]
    cfg = dataclasses.replace(_clean(base), model=dataclasses.replace(base.model, num_blocks=2), num_chunks=6,
                              prompt_switch=(3,))
    cfg = dataclasses.replace(cfg, stream=dataclasses.replace(cfg.stream, rope_reset_frames=4))
    W, ch, prompts = tiny_inputs(cfg, segment=2)
    recs = run_stream(cfg, W, ch, prompts, dtype=np.float32, tap=True)
    outs, taps, meta = run_gpu(cfg, W, ch, prompts, SDV2_BF16)
    worst = _check(cfg, recs, outs, taps, meta, 2e-2)
    print(f"clean re-run 1.3B 480p: worst block rel-L2 {worst:.3e}")


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [SDV2_FP32, SDV2_BF16])
def test_clean_rerun_multi_stream(prec):
    """kv_mode 1 with B = 2 streams batched per call (each with its own prompts and switch):
    the clean pass re-runs both streams' previous chunks; each stream equals its own oracle."""
    from gpu_harness import multi_inputs, run_gpu_streams, stream_oracles
    cfg = _clean(sg.CONFIGS["tiny"])
    switches = [(4,), ()]
    W, chunks, prompts = multi_inputs(cfg, 2, 8, switches)
    recs = stream_oracles(cfg, W, chunks, prompts, switches)
    outs, _, meta = run_gpu_streams(cfg, W, chunks, prompts, switches, prec, tap=False)
    for b in range(2):
        assert len(outs[b]) == 8
        for X, o in outs[b].items():
            assert rel_l2(o, recs[b][X]["out"]) <= TOL[prec], (b, X)
        for (X, j), (slots, _, _) in meta[b].items():
            assert slots == {s: (t, p[0]) for s, (t, p) in recs[b][X]["lane_state"][(0, j)].items()}, (b, X)
