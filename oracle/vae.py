"""Stream-VAE stand-in (oracle side).

Test infrastructure only (see oracle/__init__.py).

PAPER.md P:235-236 (§3.3 "Stream-VAE"): "processes short video chunks (e.g., 4 frames)
and caches intermediate features within each 3D convolution to maintain temporal
coherence".  The stand-in has Wan2.1-VAE shapes (synthgen.vae_layers): 3x3x3 convs that are
causal in time (two zero frames in front of the sequence), RMS-normalised SiLU residual
blocks, 2x2 (x2 in time) average pooling in the encoder, nearest 2x2 (x2 in time)
upsampling in the decoder; 4 video frames <-> 1 latent frame.

Plain NumPy, channels-last arrays [T, H, W, C], fp64 unless the caller picks fp32.  The
full-sequence functions (*_full) are the definition; StreamVAE runs the same layers chunk
by chunk with a two-frame cache per convolution (chunked == full).
"""
from __future__ import annotations

import numpy as np


def causal_conv3d(x, w, b):
    """y[t,h,w,co] = b[co] + sum_{kt,kh,kw,ci} w[co,kt,kh,kw,ci] xp[t+kt, h+kh, w+kw, ci] with xp =
    x zero-padded by 2 frames in front (causal) and 1 pixel on each spatial side."""
    T, H, W, C = x.shape
    xp = np.zeros((T + 2, H + 2, W + 2, C), dtype=x.dtype)
    xp[2:, 1:-1, 1:-1] = x
    y = np.zeros((T, H, W, w.shape[0]), dtype=x.dtype) + b
    for kt in range(3):
        for kh in range(3):
            for kw in range(3):
                y += xp[kt:kt + T, kh:kh + H, kw:kw + W] @ w[:, kt, kh, kw, :].T
    return y


def conv_with_cache(x, cache, w, b):
    """One chunk of a streamed causal conv: the cache holds the previous chunk's last two
    input frames (zeros at stream start).  Returns (y, new cache)."""
    T, H, W, C = x.shape
    xc = np.concatenate([cache, x], axis=0)          # [T + 2, ...]
    xp = np.zeros((T + 2, H + 2, W + 2, C), dtype=x.dtype)
    xp[:, 1:-1, 1:-1] = xc
    y = np.zeros((T, H, W, w.shape[0]), dtype=x.dtype) + b
    for kt in range(3):
        for kh in range(3):
            for kw in range(3):
                y += xp[kt:kt + T, kh:kh + H, kw:kw + W] @ w[:, kt, kh, kw, :].T
    return y, xc[-2:].copy()


def rms_silu(x, g, eps):
    """SiLU(g * x / sqrt(mean_c x^2 + eps)) over the channel axis."""
    z = g * x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return z / (1.0 + np.exp(-z))


def pool(x, tf):
    """Average of 2x2 pixels (and of tf consecutive frames)."""
    T, H, W, C = x.shape
    return x.reshape(T // tf, tf, H // 2, 2, W // 2, 2, C).mean(axis=(1, 3, 5))


def up(x, tf):
    """Nearest upsampling: every pixel to 2x2, every frame repeated tf times."""
    return np.repeat(np.repeat(np.repeat(x, tf, axis=0), 2, axis=1), 2, axis=2)


class _Runner:
    """Walks a layer list; `conv(name, x)` is either the full-sequence conv or the cached one."""

    def __init__(self, W, vd, dt, conv):
        self.W, self.vd, self.dt, self.conv = W, vd, dt, conv

    def w(self, n):
        return self.W[n].astype(self.dt)

    def run(self, layers, x):
        eps = self.vd.eps
        for name, kind, ci, co in layers:
            p = f"vae.{name}."
            if kind == "conv":
                x = self.conv(name, x, self.w(p + "w"), self.w(p + "b"))
            elif kind == "res":
                h = rms_silu(x, self.w(p + "n1"), eps)
                h = self.conv(name + ".c1", h, self.w(p + "c1.w"), self.w(p + "c1.b"))
                h = rms_silu(h, self.w(p + "n2"), eps)
                h = self.conv(name + ".c2", h, self.w(p + "c2.w"), self.w(p + "c2.b"))
                x = x + h
            elif kind == "norm":
                x = rms_silu(x, self.w(p + "g"), eps)
            elif kind == "pool_s":
                x = pool(x, 1)
            elif kind == "pool_st":
                x = pool(x, 2)
            elif kind == "up_s":
                x = up(x, 1)
            elif kind == "up_st":
                x = up(x, 2)
        return x


def encode_full(video, W, vd, dt=np.float64):
    """video [3, F, H, W] (F a multiple of 4) -> latent [16, F / 4, H / 8, W / 8]."""
    import synthgen as sg
    enc, _ = sg.vae_layers(vd)
    x = np.transpose(np.asarray(video, dt), (1, 2, 3, 0))
    y = _Runner(W, vd, dt, lambda n, x, w, b: causal_conv3d(x, w, b)).run(enc, x)
    return np.transpose(y, (3, 0, 1, 2))


def decode_full(latent, W, vd, dt=np.float64):
    """latent [16, T, h, w] -> video [3, 4 T, 8 h, 8 w]."""
    import synthgen as sg
    _, dec = sg.vae_layers(vd)
    x = np.transpose(np.asarray(latent, dt), (1, 2, 3, 0))
    y = _Runner(W, vd, dt, lambda n, x, w, b: causal_conv3d(x, w, b)).run(dec, x)
    return np.transpose(y, (3, 0, 1, 2))


class StreamVAE:
    """Chunked encoder / decoder: every causal conv keeps its last two input frames."""

    def __init__(self, W, vd, dt=np.float64):
        import synthgen as sg
        self.enc, self.dec = sg.vae_layers(vd)
        self.caches = {}
        self.runner = _Runner(W, vd, dt, self._conv)
        self.dt = dt

    def _conv(self, name, x, w, b):
        cache = self.caches.get(name)
        if cache is None:
            cache = np.zeros((2,) + x.shape[1:], dtype=x.dtype)
        y, self.caches[name] = conv_with_cache(x, cache, w, b)
        return y

    def encode_chunk(self, video_chunk):
        """[3, 4, H, W] -> [16, 1, H / 8, W / 8]."""
        x = np.transpose(np.asarray(video_chunk, self.dt), (1, 2, 3, 0))
        return np.transpose(self.runner.run(self.enc, x), (3, 0, 1, 2))

    def decode_chunk(self, latent_chunk):
        """[16, 1, h, w] -> [3, 4, 8 h, 8 w]."""
        x = np.transpose(np.asarray(latent_chunk, self.dt), (1, 2, 3, 0))
        return np.transpose(self.runner.run(self.dec, x), (3, 0, 1, 2))
