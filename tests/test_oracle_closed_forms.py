"""Closed-form pins of the oracle's model-card functions (SURVEY.md §8(c) C.2–C.7) and
the stream-level RoPE-reset invariance pin P2(iii) (no GPU).

Every pin builds its weights from zeros, ones, identities and one-hot selectors so
the expected value is derivable by hand from the stated wiring; the only library
routines on the expected side are torch's ``rms_norm`` / ``gelu`` / ``silu`` (pinned
against the oracle's own norms in ``test_oracle_pins.py::test_norms_activations_attention_vs_torch``)
and ``math``.  ``tests/test_oracle_mutations.py`` re-runs these pins against
deliberately broken oracle functions and requires each to fail.

Citations: P:n = PAPER.md line n; C.k = SURVEY.md §8(c) model card item k.
"""
import dataclasses
import math

import numpy as np
import pytest
import torch

import synthgen as sg
from oracle import control as C
from oracle import model as M
from oracle.stream import StreamOracle, run_stream

F = torch.nn.functional
EPS = 1e-6


def _rms(x):
    return F.rms_norm(torch.from_numpy(np.asarray(x, np.float64)), (np.shape(x)[-1],), eps=EPS).numpy()


def _gelu(x):
    return F.gelu(torch.from_numpy(np.asarray(x, np.float64)), approximate="tanh").numpy()


def _silu(z):
    return float(F.silu(torch.tensor(float(z), dtype=torch.float64)))


def _zero_weights(md):
    W = sg.gen_weights(md, seed=0)
    return {k: np.zeros_like(v, dtype=np.float64) for k, v in W.items()}


def _pm_rows(L, d, seed=11):
    """x[t, c] = +-s_t: every row has mean(x^2) = s_t^2, so N(x) = x / sqrt(s_t^2 + eps)."""
    r = np.random.default_rng(seed)
    s = 0.5 + np.arange(L, dtype=np.float64) / L
    sign = np.where(r.random((L, d)) < 0.5, -1.0, 1.0)
    return sign * s[:, None], sign * (s / np.sqrt(s * s + EPS))[:, None]


# ----------------------------------------------------- C.2 time embedding
def pin_time_embed():
    """e = W_t2 SiLU(W_t1 sinusoid(1000 sigma) + b_t1) + b_t2, e0 = W_tp SiLU(e) + b_tp,
    e0 viewed as [6, d] row-major (C.2; Wan time_embedding / time_projection)."""
    md = sg.TINY_MODEL
    d, half = md.dim, md.freq_dim // 2
    W = _zero_weights(md)
    W["t1_w"][0, 0] = 1.0            # hidden 0 <- cos(t * 10000^0)       (cos first)
    W["t1_w"][1, half] = 1.0         # hidden 1 <- sin(t * 10000^0)
    W["t1_b"][0] = 0.25
    W["t2_w"][0, 0] = 1.0
    W["t2_w"][1, 1] = -2.0
    W["t2_b"][2] = 0.7
    W["tp_w"][2 * d + 3, 0] = 1.0    # e0[2, 3] <- SiLU(e[0])
    W["tp_w"][5 * d + 0, 1] = 1.0    # e0[5, 0] <- SiLU(e[1])
    W["tp_b"][4 * d + 7] = -0.5      # e0[4, 7] = -0.5
    sigma = 0.25                     # timestep t = 1000 sigma = 250
    e, e0 = M.time_embed(np.float32(sigma), W, md, np.float64)
    h0 = _silu(math.cos(250.0) + 0.25)
    h1 = _silu(math.sin(250.0))
    exp_e = np.zeros(d)
    exp_e[0], exp_e[1], exp_e[2] = h0, -2.0 * h1, 0.7
    assert e == pytest.approx(exp_e, abs=1e-14)
    exp_e0 = np.zeros((6, d))
    exp_e0[2, 3] = _silu(h0)
    exp_e0[5, 0] = _silu(-2.0 * h1)
    exp_e0[4, 7] = -0.5
    assert e0.shape == (6, d)
    assert e0 == pytest.approx(exp_e0, abs=1e-14)


def test_time_embed_closed_form():
    pin_time_embed()


# ------------------------------------------------ C.3 prompt embedding / K, V
def pin_text_embed_and_prompt_kv():
    """ctx = W_x2 GELU_tanh(W_x1 P + b_x1) + b_x2; K_c = g_ck * RMS_full_d(ctx W_ck^T + b_ck),
    V_c = ctx W_cv^T + b_cv (C.3)."""
    md = sg.TINY_MODEL
    d, Dt = md.dim, md.text_dim
    W = _zero_weights(md)
    for c in range(Dt):
        W["txt1_w"][c, c] = 1.0
    W["txt1_b"][:] = 0.1
    W["txt2_w"][:] = 2.0 * np.eye(d)
    W["txt2_b"][:] = -0.3
    P = np.random.default_rng(7).standard_normal((md.text_len, Dt))
    ctx = M.text_embed(P, W, np.float64)
    hid = np.full((md.text_len, d), 0.1)
    hid[:, :Dt] += P
    exp_ctx = 2.0 * _gelu(hid) - 0.3
    assert ctx == pytest.approx(exp_ctx, abs=1e-14)
    W["blocks.0.wck"][:] = np.eye(d)
    W["blocks.0.gck"][:] = 1.5
    W["blocks.0.wcv"][:] = 0.5 * np.eye(d)
    W["blocks.0.bcv"][:] = 0.2
    K, V = M.prompt_kv(ctx, W, 0, md, np.float64)
    assert K == pytest.approx(1.5 * _rms(exp_ctx), abs=1e-13)
    assert V == pytest.approx(0.5 * exp_ctx + 0.2, abs=1e-14)


def test_text_embed_and_prompt_kv_closed_form():
    pin_text_embed_and_prompt_kv()


# ------------------------------------------------------ C.4 qk-norm over d
def pin_rms_g_full_dim():
    """RMS_g normalises over the full model dim d (Wan qk-norm), not per head: with
    head 0 all ones and head 1 all threes, mean(y^2) = 5 over d."""
    d = 128
    y = np.concatenate([np.ones(64), 3.0 * np.ones(64)])[None, :]
    g = 1.0 + np.arange(d) / d
    r = 1.0 / math.sqrt(5.0 + EPS)
    exp = g * np.concatenate([np.full(64, r), np.full(64, 3.0 * r)])
    assert M.rms_g(y, g, EPS) == pytest.approx(exp[None, :], abs=1e-15)


def test_rms_g_full_dim():
    pin_rms_g_full_dim()


# ---------------------------------------------------------- C.6 RoPE law
def pin_rope_frequency_law():
    """hd = 64: pairs split (12, 10, 10) = (t, h, w); group g with c_g pairs rotates
    pair i by pos_g * 10000^(-i / c_g).  The half-way pair of each group has
    10000^(-1/2) = 1/100 exactly; interleaved pairs (2i, 2i+1) rotate as complex numbers."""
    hd = 64
    exp = np.zeros((4, 32))
    exp[0, 0], exp[0, 6] = 1.0, 0.01                 # pos_t = 1
    exp[1, 12], exp[1, 17] = 1.0, 0.01               # pos_h = 1
    exp[2, 22], exp[2, 27] = 2.0, 0.02               # pos_w = 2
    exp[3, 0], exp[3, 12], exp[3, 22] = 3.0, 1.0, 2.0
    exp[3, 6], exp[3, 17], exp[3, 27] = 0.03, 0.01, 0.02
    phi = M.rope_angles(hd, [1, 0, 0, 3], [0, 1, 0, 1], [0, 0, 2, 2])
    for row in range(4):
        for i in (0, 6, 12, 17, 22, 27):
            assert phi[row, i] == pytest.approx(exp[row, i], rel=1e-14, abs=0), (row, i)
    assert phi[0, 12:].max() == 0.0 and phi[1, :12].max() == 0.0 and phi[1, 22:].max() == 0.0
    assert phi[2, :22].max() == 0.0
    # monotone decreasing inside each group
    assert np.all(np.diff(phi[0, :12]) < 0) and np.all(np.diff(phi[1, 12:22]) < 0)
    # complex rotation of the pair (2i, 2i+1): e_0 -> (cos phi, sin phi), e_1 -> (-sin, cos)
    x = np.zeros((2, hd))
    x[0, 0] = 1.0
    x[1, 13] = 1.0                                   # pair 6, second component
    out = M.rope_apply(x, M.rope_angles(hd, [1, 1], [0, 0], [0, 0]))
    assert out[0, 0] == pytest.approx(math.cos(1.0), abs=1e-15)
    assert out[0, 1] == pytest.approx(math.sin(1.0), abs=1e-15)
    assert out[1, 12] == pytest.approx(-math.sin(0.01), abs=1e-15)
    assert out[1, 13] == pytest.approx(math.cos(0.01), abs=1e-15)
    assert np.count_nonzero(out) == 4


def test_rope_frequency_law():
    pin_rope_frequency_law()


# -------------------------------------------------- C.1 / C.6 token positions
def pin_token_positions():
    """Token tau = f (h/2)(w/2) + i (w/2) + jj covers latent rows 2i.., columns 2jj..
    (patchify, C.1) and carries RoPE positions (frame_pos[f], i, jj) (C.6): height
    first, width second, on a non-square 4 x 8 latent with T' = 2."""
    md = sg.TINY_MODEL
    geom = sg.Geometry(4, 8, 2, 1, 1, 2)
    pt, ph, pw = M.token_positions(md, geom, [10, 11])
    assert len(pt) == 16
    assert (pt[6], ph[6], pw[6]) == (10, 1, 2)
    assert (pt[3], ph[3], pw[3]) == (10, 0, 3)
    assert (pt[13], ph[13], pw[13]) == (11, 1, 1)
    # the token that patchify fills from v[:, f, 2i+a, 2jj+b] has positions (f, i, jj)
    for (f, y, x) in [(0, 2, 5), (1, 3, 1), (1, 0, 7)]:
        v = np.zeros((4, 2, 4, 8))
        v[2, f, y, x] = 1.0
        u = M.patchify(v, md)
        tau = int(np.nonzero(u.any(axis=1))[0][0])
        assert (pt[tau], ph[tau], pw[tau]) == ([10, 11][f], y // 2, x // 2)


def test_token_positions_height_width():
    pin_token_positions()


# --------------------------------------------- C.5 / C.7 block wiring
def pin_block_wiring():
    """One block with: q = k = 0 (uniform attention over the chunk's own keys), V = O = I,
    cross-out = 0 with bias b_co, FFN = GELU (W1 = [I; 0], W2 = [I 0]), e0 = 0 and
    mod rows (sh1, sc1, g1, sh2, sc2, g2) = distinct constants (C.5, Wan modulation order).
        x1 = x + g1 * mean_tokens(N(x)(1 + sc1) + sh1)
        x2 = x1 + b_co
        x3 = x2 + g2 * GELU(N(x2)(1 + sc2) + sh2)"""
    cfg = sg.CONFIGS["tiny"]
    md, d, Fd = cfg.model, cfg.model.dim, cfg.model.ffn_dim
    W = _zero_weights(md)
    rows = [0.11, 0.23, 0.37, -0.41, 0.53, 0.67]
    p = "blocks.0."
    for r, val in enumerate(rows):
        W[p + "mod"][r, :] = val
    W[p + "wv"][:] = np.eye(d)
    W[p + "wo"][:] = np.eye(d)
    W[p + "bco"][:] = 0.05
    W[p + "n3_g"][:] = 1.0
    W[p + "gq"][:] = 1.0
    W[p + "gk"][:] = 1.0
    W[p + "w1"][:d, :] = np.eye(d)
    W[p + "w2"][:, :d] = np.eye(d)
    o = StreamOracle(md, cfg.geom, cfg.stream, W, blocks=[0])
    o.set_prompt(sg.gen_prompt(md, 0))
    act = o.admit_control(0)
    L = cfg.geom.tokens_per_chunk(md)
    x, nx = _pm_rows(L, d)
    out = o.block(x, np.zeros((6, d)), 0, o.lanes[(0, 0)], act)
    sh1, sc1, g1, sh2, sc2, g2 = rows
    x1 = x + g1 * np.mean(nx * (1 + sc1) + sh1, axis=0, keepdims=True)
    x2 = x1 + 0.05
    x3 = x2 + g2 * _gelu(_rms(x2) * (1 + sc2) + sh2)
    assert out == pytest.approx(x3, abs=1e-12)


def test_block_modulation_row_order():
    pin_block_wiring()


def pin_head():
    """(sh, sc) = head_mod + e (row 0 shift, row 1 scale), y = (N(x)(1 + sc) + sh) W_h^T + b_h (C.7)."""
    md = sg.TINY_MODEL
    d = md.dim
    P = md.latent_channels * md.patch_t * md.patch_h * md.patch_w
    W = _zero_weights(md)
    W["head_mod"][0, :] = 0.3
    W["head_mod"][1, :] = -0.2
    W["head_w"][:, :P] = np.eye(P)
    W["head_b"][:] = 0.01
    x, nx = _pm_rows(16, d, seed=5)
    e = np.full(d, 0.05)
    y = M.head(x, e, W, md, np.float64)
    assert y == pytest.approx(nx[:, :P] * (1 + (-0.2 + 0.05)) + (0.3 + 0.05) + 0.01, abs=1e-14)


def test_head_closed_form():
    pin_head()


# ------------------------------------- P2(iii): stream-level reset invariance
def _no_sink_cfg(T_reset):
    cfg = sg.CONFIGS["tiny"]
    return dataclasses.replace(cfg, geom=dataclasses.replace(cfg.geom, sink_chunks=0, window_chunks=2),
                               stream=dataclasses.replace(cfg.stream, rope_reset_frames=T_reset))


def pin_reset_invariance():
    """P:191, "RoPE relative-position invariance holds under offset reset": with no
    sinks (m = 0) every attended key is re-based with the query, so a stream with
    T_reset = 4 (resets at chunks 5, 9, ...) equals the same stream with no reset."""
    cfg_r, cfg_inf = _no_sink_cfg(4), _no_sink_cfg(10 ** 9)
    W = sg.gen_weights(cfg_r.model, seed=0)
    ls = sg.LatentStream(4, 8, 8, seed=1, segment=3)
    n = 11
    chunks = [ls.chunk(X, 1) for X in range(n)]
    prompts = [sg.gen_prompt(cfg_r.model, 0), sg.gen_prompt(cfg_r.model, 1)]
    a = run_stream(cfg_r, W, chunks, prompts)
    b = run_stream(cfg_inf, W, chunks, prompts)
    assert sum(r["act"]["rebase"] for r in a) == 2 and a[-1]["act"]["r"] == 2
    assert not any(r["act"]["rebase"] for r in b)
    for X in range(n):
        err = np.abs(a[X]["out"] - b[X]["out"]).max() / np.abs(b[X]["out"]).max()
        assert err <= 1e-12, (X, err)


def test_stream_rope_reset_invariance():
    pin_reset_invariance()


def test_reset_changes_output_with_sinks():
    """Counter-check: with a sink (m = 1, anchored, not re-based) the reset does change the
    output once the query's position has wrapped (the invariance above is not vacuous)."""
    cfg = sg.CONFIGS["tiny"]
    cfg_inf = dataclasses.replace(cfg, stream=dataclasses.replace(cfg.stream, rope_reset_frames=10 ** 9))
    W = sg.gen_weights(cfg.model, seed=0)
    ls = sg.LatentStream(4, 8, 8, seed=1, segment=3)
    chunks = [ls.chunk(X, 1) for X in range(7)]
    prompts = [sg.gen_prompt(cfg.model, 0), sg.gen_prompt(cfg.model, 1)]
    a = run_stream(cfg, W, chunks, prompts)
    b = run_stream(cfg_inf, W, chunks, prompts)
    assert np.array_equal(a[4]["out"], b[4]["out"])
    assert np.abs(a[6]["out"] - b[6]["out"]).max() > 1e-6


def pin_cross_wiring():
    """Cross-attention sub-block (C.5): a3 = N(x) * n3_g + n3_b (affine, no modulation),
    q_c = g_cq * RMS_full_d(a3 W_cq^T + b_cq), o_c = softmax(q_c K_c^T / sqrt(hd)) V_c per
    head, x <- x + o_c W_co^T + b_co (ungated).  Self-attention and FFN are zeroed
    (W_v = W_o = 0, W_1 = W_2 = 0, biases 0), so the block output is x + o_c."""
    cfg = sg.CONFIGS["tiny"]
    md = cfg.model
    d, H, hd = md.dim, md.num_heads, md.head_dim
    W = _zero_weights(md)
    p = "blocks.0."
    W[p + "mod"][:] = 0.3                       # gates != 0: a gated cross residual would show
    W[p + "n3_g"][:] = 1.0 + np.arange(d) / d
    W[p + "n3_b"][:] = 0.2
    W[p + "wcq"][:] = np.eye(d)
    W[p + "gcq"][:] = 1.0
    W[p + "wco"][:] = np.eye(d)
    r = np.random.default_rng(21)
    Kc, Vc = r.standard_normal((2, d)), r.standard_normal((2, d))
    o = StreamOracle(md, cfg.geom, cfg.stream, W, blocks=[0])
    o.set_prompt(sg.gen_prompt(md, 0))
    act = o.admit_control(0)
    act["ctx_kv"] = {0: (Kc, Vc)}
    L = cfg.geom.tokens_per_chunk(md)
    x = r.standard_normal((L, d))
    out = o.block(x, np.zeros((6, d)), 0, o.lanes[(0, 0)], act)
    a3 = _rms(x) * W[p + "n3_g"] + 0.2
    qc = torch.from_numpy(_rms(a3))
    exp = x.copy()
    for h in range(H):
        cs = slice(h * hd, (h + 1) * hd)
        s = qc[:, cs] @ torch.from_numpy(Kc[:, cs]).T / math.sqrt(hd)
        exp[:, cs] += (torch.softmax(s, dim=1) @ torch.from_numpy(Vc[:, cs])).numpy()
    assert out == pytest.approx(exp, abs=1e-12)


def test_cross_attention_wiring():
    pin_cross_wiring()
