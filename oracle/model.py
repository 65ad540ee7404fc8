"""Causal-DiT model card C.1–C.8 (oracle side, plain NumPy).

Test infrastructure only (see oracle/__init__.py).

The paper only says the model "is built on Wan 2.1 and CausVid" (§5.1
"Models"); BASELINE.json's north star lists the ops ("adaLN-modulated RMSNorm,
QKV/out/FFN projections, 3D RoPE ... attention of the chunk's queries over a
[sink tokens || rolling-window] KV cache").  The block definition below is the
external Wan2.1 reading written down in SURVEY.md §8(c) C.1–C.8 (readings
Q1–Q4, Q19, Q29, Q31 in DESIGN.md).  Every step is written in its plainest
form; matmuls are library calls, nothing is fused, blocked or reordered.
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------- C.4 norms
def rms_norm(x, eps):
    """N(x) = x / sqrt(mean(x^2) + eps)   (C.4, BJ "RMSNorm")."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def layer_norm(x, eps):
    """N(x) = (x - mu) / sqrt(var + eps)   (C.4, Wan affine-free LayerNorm, norm_center=1)."""
    mu = np.mean(x, axis=-1, keepdims=True)
    xc = x - mu
    return xc / np.sqrt(np.mean(xc * xc, axis=-1, keepdims=True) + eps)


def norm(x, md):
    return layer_norm(x, md.eps) if md.norm_center else rms_norm(x, md.eps)


def rms_g(y, g, eps):
    """RMS_g(y) = g * y / sqrt(mean(y^2) + eps) over the full dim (C.4, Wan qk-norm)."""
    return g * rms_norm(y, eps)


def gelu_tanh(z):
    """0.5 z (1 + tanh(sqrt(2/pi) (z + 0.044715 z^3)))   (C.4)."""
    return 0.5 * z * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (z + 0.044715 * z ** 3)))


def silu(z):
    """z / (1 + exp(-z))   (C.2)."""
    return z / (1.0 + np.exp(-z))


def linear(x, w, b):
    """nn.Linear: x W^T + b."""
    return x @ w.T + b


# ------------------------------------------------------- C.1 / C.7 layouts
def patchify(v, md):
    """v [C, T', h, w] -> u [L, C*pt*ph*pw]; token tau = f*(h/2)(w/2) + i*(w/2) + jj,
    u[tau, c*4 + a*2 + b] = v[c, f, 2i+a, 2jj+b]  (C.1, conv3d weight flattening order)."""
    C, T, h, w = v.shape
    pt, ph, pw = md.patch_t, md.patch_h, md.patch_w
    Tn, hn, wn = T // pt, h // ph, w // pw
    u = np.zeros((Tn * hn * wn, C * pt * ph * pw), dtype=v.dtype)
    for f in range(Tn):
        for i in range(hn):
            for jj in range(wn):
                tau = f * hn * wn + i * wn + jj
                for c in range(C):
                    for t in range(pt):
                        for a in range(ph):
                            for b in range(pw):
                                u[tau, ((c * pt + t) * ph + a) * pw + b] = v[c, f * pt + t, i * ph + a, jj * pw + b]
    return u


def unpatchify(y, md, T, h, w):
    """y [L, pt*ph*pw*C] -> v [C, T', h, w]; per-token layout (pt, ph, pw, c), channel
    innermost: v[c, f, 2i+a, 2jj+b] = y[tau, (a*2+b)*C + c]   (C.7)."""
    C = md.latent_channels
    pt, ph, pw = md.patch_t, md.patch_h, md.patch_w
    Tn, hn, wn = T // pt, h // ph, w // pw
    v = np.zeros((C, T, h, w), dtype=y.dtype)
    for f in range(Tn):
        for i in range(hn):
            for jj in range(wn):
                tau = f * hn * wn + i * wn + jj
                for t in range(pt):
                    for a in range(ph):
                        for b in range(pw):
                            for c in range(C):
                                v[c, f * pt + t, i * ph + a, jj * pw + b] = y[tau, ((t * ph + a) * pw + b) * C + c]
    return v


# --------------------------------------------------------- C.2 time embedding
def sinusoid(t, dim):
    """emb[k] = cos(t 10000^(-k/half)), emb[half+k] = sin(...), fp64, cos first (C.2)."""
    half = dim // 2
    k = np.arange(half, dtype=np.float64)
    arg = float(t) * np.power(10000.0, -k / half)
    return np.concatenate([np.cos(arg), np.sin(arg)])


def time_embed(sigma, W, md, dt):
    """sigma (fp32 noise level) -> e [d], e0 [6, d]   (C.2; timestep t = 1000 sigma)."""
    t = 1000.0 * float(sigma)
    emb = sinusoid(t, md.freq_dim).astype(dt)
    e = linear(silu(linear(emb, W["t1_w"].astype(dt), W["t1_b"].astype(dt))),
               W["t2_w"].astype(dt), W["t2_b"].astype(dt))
    e0 = linear(silu(e), W["tp_w"].astype(dt), W["tp_b"].astype(dt))
    return e, e0.reshape(6, md.dim)


# --------------------------------------------------------------- C.3 prompt
def text_embed(P, W, dt):
    """ctx = W_x2 GELU_tanh(W_x1 P + b_x1) + b_x2   (C.3)."""
    return linear(gelu_tanh(linear(P.astype(dt), W["txt1_w"].astype(dt), W["txt1_b"].astype(dt))),
                  W["txt2_w"].astype(dt), W["txt2_b"].astype(dt))


def prompt_kv(ctx, W, b, md, dt):
    """Per block: K_c = RMS_{g_ck}(ctx W_ck^T + b_ck), V_c = ctx W_cv^T + b_cv   (C.3)."""
    p = f"blocks.{b}."
    K = rms_g(linear(ctx, W[p + "wck"].astype(dt), W[p + "bck"].astype(dt)), W[p + "gck"].astype(dt), md.eps)
    V = linear(ctx, W[p + "wcv"].astype(dt), W[p + "bcv"].astype(dt))
    return K, V


# ------------------------------------------------------------------ C.6 RoPE
def rope_split(hd):
    """Pair groups (temporal, height, width) = (c - 2 floor(c/3), floor(c/3), floor(c/3)), c = hd/2."""
    c = hd // 2
    return c - 2 * (c // 3), c // 3, c // 3


def rope_angles(hd, pos_t, pos_h, pos_w):
    """phi[token, pair] in fp64: temporal pairs use pos_t * 10000^(-i/c_t), then height, then width."""
    ct, ch, cw = rope_split(hd)
    wt = np.power(10000.0, -np.arange(ct, dtype=np.float64) / ct)
    wh = np.power(10000.0, -np.arange(ch, dtype=np.float64) / ch)
    ww = np.power(10000.0, -np.arange(cw, dtype=np.float64) / cw)
    pt = np.asarray(pos_t, dtype=np.float64)[:, None]
    ph = np.asarray(pos_h, dtype=np.float64)[:, None]
    pw = np.asarray(pos_w, dtype=np.float64)[:, None]
    return np.concatenate([pt * wt[None], ph * wh[None], pw * ww[None]], axis=1)


def rope_apply(x, phi):
    """x [L, hd] (one head), interleaved pairs (2i, 2i+1) rotated by phi[:, i] (C.6)."""
    x64 = x.astype(np.float64)
    x0, x1 = x64[:, 0::2], x64[:, 1::2]
    c, s = np.cos(phi), np.sin(phi)
    out = np.empty_like(x64)
    out[:, 0::2] = x0 * c - x1 * s
    out[:, 1::2] = x0 * s + x1 * c
    return out.astype(x.dtype)


def token_positions(md, geom, frame_pos):
    """(temporal, height, width) RoPE positions of the L tokens of one chunk whose
    frame f sits at temporal position frame_pos[f]  (C.6)."""
    hn, wn = geom.latent_h // md.patch_h, geom.latent_w // md.patch_w
    pt, ph, pw = [], [], []
    for f in range(geom.chunk_frames // md.patch_t):
        for i in range(hn):
            for jj in range(wn):
                pt.append(frame_pos[f]); ph.append(i); pw.append(jj)
    return np.array(pt), np.array(ph), np.array(pw)


# ------------------------------------------------------------- attention
def attention(q, k, v):
    """softmax(q k^T / sqrt(hd)) v for one head; q [Lq, hd], k/v [Lk, hd]  (C.5, Q31)."""
    s = (q @ k.T) / np.sqrt(q.shape[1]).astype(q.dtype)
    s = s - np.max(s, axis=1, keepdims=True)
    p = np.exp(s)
    p = p / np.sum(p, axis=1, keepdims=True)
    return p @ v


# ---------------------------------------------------------------- C.7 head
def head(x, e, W, md, dt):
    """(sh, sc) = mod_h + e; y = (N(x)(1+sc) + sh) W_h^T + b_h   (C.7)."""
    mod = W["head_mod"].astype(dt) + e[None, :]
    sh, sc = mod[0], mod[1]
    return linear(norm(x, md) * (1 + sc) + sh, W["head_w"].astype(dt), W["head_b"].astype(dt))
