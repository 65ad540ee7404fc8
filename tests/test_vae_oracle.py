"""Pins of the Stream-VAE stand-in oracle:
the causal conv vs torch.conv3d with explicit causal padding, streamed == full sequence for
chunk sizes {1, 2, 4, 8} and for the whole encoder / decoder, causality, the kt = 1
special case, and the norm / pool / upsample steps vs torch routines (no GPU)."""
import dataclasses

import numpy as np
import pytest
import torch

import synthgen as sg
from oracle import vae as V

F = torch.nn.functional


def _conv_torch(x, w, b):
    """x [T,H,W,C] -> torch conv3d on NCDHW with 2 zero frames in front and 1 px each side."""
    xt = torch.from_numpy(x).permute(3, 0, 1, 2)[None]
    xt = F.pad(xt, (1, 1, 1, 1, 2, 0))
    wt = torch.from_numpy(w).permute(0, 4, 1, 2, 3)          # [co, ci, kt, kh, kw]
    y = F.conv3d(xt, wt, torch.from_numpy(b))
    return y[0].permute(1, 2, 3, 0).numpy()


def test_causal_conv_is_torch_conv3d_with_causal_padding():
    r = np.random.default_rng(0)
    x = r.standard_normal((5, 6, 7, 4))
    w = r.standard_normal((3, 3, 3, 3, 4))
    b = r.standard_normal(3)
    assert V.causal_conv3d(x, w, b) == pytest.approx(_conv_torch(x, w, b), rel=1e-10, abs=1e-10)


@pytest.mark.parametrize("chunk", [1, 2, 4, 8])
def test_streamed_conv_equals_full(chunk):
    """16 frames in chunks == one pass, exactly up to summation order (same here)."""
    r = np.random.default_rng(chunk)
    x = r.standard_normal((16, 5, 6, 3))
    w = r.standard_normal((4, 3, 3, 3, 3))
    b = r.standard_normal(4)
    full = V.causal_conv3d(x, w, b)
    cache = np.zeros((2, 5, 6, 3))
    outs = []
    for t0 in range(0, 16, chunk):
        y, cache = V.conv_with_cache(x[t0:t0 + chunk], cache, w, b)
        outs.append(y)
    assert np.array_equal(np.concatenate(outs), full)


def test_kernel_t1_is_per_frame_conv_and_causal():
    r = np.random.default_rng(3)
    x = r.standard_normal((6, 4, 5, 2))
    w = np.zeros((2, 3, 3, 3, 2))
    w[:, 2] = r.standard_normal((2, 3, 3, 2))                 # only the current frame's tap
    b = r.standard_normal(2)
    y = V.causal_conv3d(x, w, b)
    for t in range(6):
        assert np.allclose(y[t], V.causal_conv3d(x[t:t + 1], w, b)[0], atol=1e-12)
    w2 = r.standard_normal((2, 3, 3, 3, 2))
    x2 = x.copy()
    x2[4] += 1.0
    a, c = V.causal_conv3d(x, w2, b), V.causal_conv3d(x2, w2, b)
    assert np.array_equal(a[:4], c[:4]) and not np.array_equal(a[4], c[4])


def test_norm_pool_up_vs_torch():
    r = np.random.default_rng(4)
    x = r.standard_normal((4, 6, 8, 5))
    g = 1 + 0.1 * r.standard_normal(5)
    ref = F.silu(F.rms_norm(torch.from_numpy(x), (5,), torch.from_numpy(g), eps=1e-6)).numpy()
    assert V.rms_silu(x, g, 1e-6) == pytest.approx(ref, rel=1e-10, abs=1e-12)
    xt = torch.from_numpy(x).permute(3, 0, 1, 2)[None]
    p = F.avg_pool3d(xt, (2, 2, 2))[0].permute(1, 2, 3, 0).numpy()
    assert V.pool(x, 2) == pytest.approx(p, rel=1e-12)
    u = F.interpolate(xt, scale_factor=(2, 2, 2), mode="nearest")[0].permute(1, 2, 3, 0).numpy()
    assert np.array_equal(V.up(x, 2), u)


def _small():
    vd = dataclasses.replace(sg.VAE, dims=(8, 12, 16), latent_channels=4)
    return vd, sg.gen_vae_weights(vd)


def test_stream_vae_equals_full_sequence():
    """the chunked encoder / decoder with per-conv feature caches reproduce the
    full-sequence causal VAE (3 chunks = 12 frames, shapes multiples of 8)."""
    vd, W = _small()
    video = sg.gen_video(vd, 12, 16, 24)
    full = V.encode_full(video, W, vd)
    sv = V.StreamVAE(W, vd)
    chunked = np.concatenate([sv.encode_chunk(video[:, 4 * i:4 * i + 4]) for i in range(3)], axis=1)
    assert full.shape == (4, 3, 2, 3)
    assert chunked == pytest.approx(full, rel=1e-12, abs=1e-12)
    dfull = V.decode_full(full, W, vd)
    dch = np.concatenate([sv.decode_chunk(full[:, i:i + 1]) for i in range(3)], axis=1)
    assert dfull.shape == (3, 12, 16, 24)
    assert dch == pytest.approx(dfull, rel=1e-12, abs=1e-12)


def test_stream_vae_causality():
    vd, W = _small()
    video = sg.gen_video(vd, 12, 16, 24)
    v2 = video.copy()
    v2[:, 9] += 0.5                                           # chunk 2 only
    a, b = V.encode_full(video, W, vd), V.encode_full(v2, W, vd)
    assert np.array_equal(a[:, :2], b[:, :2]) and not np.array_equal(a[:, 2], b[:, 2])
