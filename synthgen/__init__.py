"""Seeded synthetic inputs shared by the oracle-side tests and the product driver.

This module holds NO arithmetic of the method (no norms, attention, RoPE,
controller or sampler math).  It only defines:

* the BASELINE.json configurations as plain shape records (``CONFIGS``);
* the weight list of the Wan2.1-shaped causal DiT (names, shapes, init law,
  SURVEY.md §8(c) O2) and a per-tensor seeded generator;
* prompts and the synthetic moving latent stream (SURVEY.md §8(d)
  "Synthetic inputs").

Every value it produces is deterministic in (seed, tensor name) so the oracle
and the GPU path receive bit-identical inputs.  Weights are rounded once to
bf16-representable fp32 (round-to-nearest-even) so the bf16 and fp32 GPU paths
and the oracle all use the same numbers.
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, Iterator, List, Tuple

import numpy as np


# ---------------------------------------------------------------------------
# Configurations (BASELINE.json configs[0..4]; SURVEY.md §8(d) per-config table)
# ---------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class ModelDesc:
    num_blocks: int
    dim: int
    num_heads: int
    ffn_dim: int
    latent_channels: int
    patch_t: int = 1
    patch_h: int = 2
    patch_w: int = 2
    text_len: int = 512
    text_dim: int = 4096
    freq_dim: int = 256
    eps: float = 1e-6
    norm_center: int = 0          # 0 = RMSNorm (BJ wording), 1 = affine-free LayerNorm (Wan)

    @property
    def head_dim(self) -> int:
        return self.dim // self.num_heads


@dataclasses.dataclass(frozen=True)
class Geometry:
    latent_h: int
    latent_w: int
    chunk_frames: int             # T'
    steps: int                    # n = B (stream batch = in-flight denoising steps)
    sink_chunks: int              # m
    window_chunks: int            # W
    streams: int = 1              # B: independent streams batched per call (SLO batch, N2)
    kv_mode: int = 0              # 0: step-j K/V cached in lane j (R1); 1: clean re-run (Q5, N4; n = 1)

    def tokens_per_chunk(self, md: ModelDesc) -> int:
        return (self.chunk_frames // md.patch_t) * (self.latent_h // md.patch_h) * (self.latent_w // md.patch_w)


@dataclasses.dataclass(frozen=True)
class StreamDesc:
    timesteps: Tuple[float, ...]  # strictly decreasing, t_0 in (0, 1000]
    rope_reset_frames: int        # T_reset
    motion_k: int = 8             # window holds k+1 values (Q13)
    motion_sigma: float = 1.0     # sigma_m (Q14: fixed constant)
    s_min: float = 0.4            # Q17
    s_max: float = 0.9
    ema_lambda: float = 0.4
    sink_tau: float = 0.95        # Q18
    seed: int = 3                 # Philox key for the injected noise (Q21)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    model: ModelDesc
    geom: Geometry
    stream: StreamDesc
    num_chunks: int
    prompt_switch: Tuple[int, ...] = ()   # chunk indices where a new prompt takes effect


SCHEDULES = {1: (1000.0,), 2: (1000.0, 500.0), 4: (1000.0, 750.0, 500.0, 250.0)}   # Q20

TINY_MODEL = ModelDesc(num_blocks=2, dim=128, num_heads=2, ffn_dim=512, latent_channels=4,
                       text_len=8, text_dim=32)
WAN13_MODEL = ModelDesc(num_blocks=30, dim=1536, num_heads=12, ffn_dim=8960, latent_channels=16)
WAN14_MODEL = ModelDesc(num_blocks=40, dim=5120, num_heads=40, ffn_dim=13824, latent_channels=16)

CONFIGS: Dict[str, Config] = {
    # configs[0]: tiny causal DiT, oracle in seconds
    "tiny": Config("tiny", TINY_MODEL,
                   Geometry(8, 8, 1, 2, 1, 2),
                   StreamDesc(SCHEDULES[2], rope_reset_frames=4, motion_k=2, motion_sigma=0.5),
                   num_chunks=8, prompt_switch=(6,)),
    # configs[1]: 1.3B 480p, 1 step, single B200 (the N=1 bench workload)
    "wan13_480p_1step": Config("wan13_480p_1step", WAN13_MODEL,
                               Geometry(60, 104, 1, 1, 1, 4),
                               StreamDesc(SCHEDULES[1], rope_reset_frames=240), num_chunks=1024),
    # configs[2]: 1.3B 512x512, stream batch of 4 steps
    "wan13_512_4step": Config("wan13_512_4step", WAN13_MODEL,
                              Geometry(64, 64, 1, 4, 1, 4),
                              StreamDesc(SCHEDULES[4], rope_reset_frames=240), num_chunks=2048),
    # configs[3]: 14B 480p, 4 steps
    "wan14_480p_4step": Config("wan14_480p_4step", WAN14_MODEL,
                               Geometry(60, 104, 1, 4, 1, 4),
                               StreamDesc(SCHEDULES[4], rope_reset_frames=240), num_chunks=1024),
    # configs[4]: long-horizon 1.3B 480p, 10k chunks
    "long_horizon": Config("long_horizon", WAN13_MODEL,
                           Geometry(60, 104, 1, 4, 1, 4),
                           StreamDesc(SCHEDULES[4], rope_reset_frames=240), num_chunks=10000,
                           prompt_switch=(2500, 5000, 7500)),
}


# ---------------------------------------------------------------------------
# Weights
# ---------------------------------------------------------------------------
# init kinds: ("linear_w", fan_in) U(+-1/sqrt(fan_in)); ("linear_b", fan_in) same law;
# ("mod", d) N(0,1)/sqrt(d); ("gain",) 1+0.1 N(0,1); ("shift",) 0.1 N(0,1)
GLOBAL_TENSORS = ("patch_w", "patch_b", "txt1_w", "txt1_b", "txt2_w", "txt2_b",
                  "t1_w", "t1_b", "t2_w", "t2_b", "tp_w", "tp_b", "head_mod", "head_w", "head_b")
BLOCK_TENSORS = ("mod", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "gq", "gk",
                 "n3_g", "n3_b", "wcq", "bcq", "wck", "bck", "wcv", "bcv", "wco", "bco", "gcq", "gck",
                 "w1", "b1", "w2", "b2")


def tensor_spec(md: ModelDesc, name: str) -> Tuple[Tuple[int, ...], tuple]:
    """Shape and init law of one named tensor (nn.Linear weights are [out, in])."""
    d, F, C = md.dim, md.ffn_dim, md.latent_channels
    P = C * md.patch_t * md.patch_h * md.patch_w
    base = name.split(".")[-1]
    g = {
        "patch_w": ((d, P), ("u", P)), "patch_b": ((d,), ("u", P)),
        "txt1_w": ((d, md.text_dim), ("u", md.text_dim)), "txt1_b": ((d,), ("u", md.text_dim)),
        "txt2_w": ((d, d), ("u", d)), "txt2_b": ((d,), ("u", d)),
        "t1_w": ((d, md.freq_dim), ("u", md.freq_dim)), "t1_b": ((d,), ("u", md.freq_dim)),
        "t2_w": ((d, d), ("u", d)), "t2_b": ((d,), ("u", d)),
        "tp_w": ((6 * d, d), ("u", d)), "tp_b": ((6 * d,), ("u", d)),
        "head_mod": ((2, d), ("mod", d)),
        "head_w": ((P, d), ("u", d)), "head_b": ((P,), ("u", d)),
        "mod": ((6, d), ("mod", d)),
        "wq": ((d, d), ("u", d)), "bq": ((d,), ("u", d)),
        "wk": ((d, d), ("u", d)), "bk": ((d,), ("u", d)),
        "wv": ((d, d), ("u", d)), "bv": ((d,), ("u", d)),
        "wo": ((d, d), ("u", d)), "bo": ((d,), ("u", d)),
        "gq": ((d,), ("gain",)), "gk": ((d,), ("gain",)),
        "n3_g": ((d,), ("gain",)), "n3_b": ((d,), ("shift",)),
        "wcq": ((d, d), ("u", d)), "bcq": ((d,), ("u", d)),
        "wck": ((d, d), ("u", d)), "bck": ((d,), ("u", d)),
        "wcv": ((d, d), ("u", d)), "bcv": ((d,), ("u", d)),
        "wco": ((d, d), ("u", d)), "bco": ((d,), ("u", d)),
        "gcq": ((d,), ("gain",)), "gck": ((d,), ("gain",)),
        "w1": ((F, d), ("u", d)), "b1": ((F,), ("u", d)),
        "w2": ((d, F), ("u", F)), "b2": ((d,), ("u", F)),
    }
    if base not in g:
        raise KeyError(name)
    return g[base]


def block_tensor_names(b: int) -> List[str]:
    return [f"blocks.{b}.{t}" for t in BLOCK_TENSORS]


def all_tensor_names(md: ModelDesc) -> List[str]:
    names = list(GLOBAL_TENSORS)
    for b in range(md.num_blocks):
        names += block_tensor_names(b)
    return names


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed, zlib.crc32(name.encode())]))


def gen_tensor(md: ModelDesc, name: str, seed: int = 0) -> np.ndarray:
    shape, law = tensor_spec(md, name)
    r = _rng(seed, name)
    if law[0] == "u":
        bound = 1.0 / np.sqrt(law[1])
        a = r.uniform(-bound, bound, size=shape)
    elif law[0] == "mod":
        a = r.standard_normal(size=shape) / np.sqrt(law[1])
    elif law[0] == "gain":
        a = 1.0 + 0.1 * r.standard_normal(size=shape)
    elif law[0] == "shift":
        a = 0.1 * r.standard_normal(size=shape)
    else:  # pragma: no cover
        raise ValueError(law)
    return round_to_bf16(a.astype(np.float32))


def gen_weights(md: ModelDesc, seed: int = 0, blocks=None) -> Dict[str, np.ndarray]:
    """All global tensors plus the per-block tensors of ``blocks`` (default: all)."""
    out = {n: gen_tensor(md, n, seed) for n in GLOBAL_TENSORS}
    for b in (range(md.num_blocks) if blocks is None else blocks):
        for n in block_tensor_names(b):
            out[n] = gen_tensor(md, n, seed)
    return out


# ---------------------------------------------------------------------------
# Prompts and the latent stream
# ---------------------------------------------------------------------------
def gen_prompt(md: ModelDesc, k: int) -> np.ndarray:
    """Prompt k: N(0,1) [text_len, text_dim] fp32, seed 100+k."""
    r = np.random.Generator(np.random.PCG64(100 + k))
    return r.standard_normal((md.text_len, md.text_dim)).astype(np.float32)


def prompt_index_for_chunk(cfg: Config, X: int) -> int:
    return sum(1 for s in cfg.prompt_switch if X >= s)


class LatentStream:
    """Moving multi-sinusoid latent field + per-frame noise.

    Per channel: sum of R random 2D sinusoids (wavenumbers U(-0.6,0.6) rad per
    latent px, random phases, amplitudes N(0,1)/sqrt(R)), normalised to unit RMS,
    translated by u(g) latent px along x at frame g (exact sub-pixel via phase),
    plus ``noise`` * N(0,1) per frame.  The speed profile cycles through
    ``speeds`` in segments of ``segment`` frames.
    """

    def __init__(self, C: int, h: int, w: int, seed: int = 1, R: int = 8,
                 speeds=(0.0, 0.25, 2.0, 6.0), segment: int = 256, noise: float = 0.05):
        r = np.random.Generator(np.random.PCG64(seed))
        self.C, self.h, self.w = C, h, w
        self.kx = r.uniform(-0.6, 0.6, size=(C, R))
        self.ky = r.uniform(-0.6, 0.6, size=(C, R))
        self.ph = r.uniform(0, 2 * np.pi, size=(C, R))
        self.amp = r.standard_normal((C, R)) / np.sqrt(R)
        self.speeds = tuple(speeds)
        self.segment = segment
        self.noise = noise
        self.seed = seed
        base = self._field(0.0)
        self.scale = 1.0 / np.sqrt(np.mean(base * base, axis=(1, 2), keepdims=True))

    def _field(self, shift: float) -> np.ndarray:
        y = np.arange(self.h)[:, None]
        x = np.arange(self.w)[None, :]
        out = np.zeros((self.C, self.h, self.w))
        for c in range(self.C):
            for k in range(self.kx.shape[1]):
                out[c] += self.amp[c, k] * np.cos(self.kx[c, k] * (x - shift) + self.ky[c, k] * y + self.ph[c, k])
        return out

    def speed(self, g: int) -> float:
        return self.speeds[(g // self.segment) % len(self.speeds)]

    def shift(self, g: int) -> float:
        # cumulative translation before frame g
        full, rem = divmod(g, self.segment)
        s = 0.0
        for i in range(full):
            s += self.segment * self.speeds[i % len(self.speeds)]
        return s + rem * self.speeds[full % len(self.speeds)]

    def frame(self, g: int) -> np.ndarray:
        f = self._field(self.shift(g)) * self.scale
        r = np.random.Generator(np.random.PCG64([self.seed, 7, g]))
        f = f + self.noise * r.standard_normal(f.shape)
        return f.astype(np.float32)

    def chunk(self, X: int, T: int) -> np.ndarray:
        """Chunk X as [C, T', h, w] fp32."""
        return np.stack([self.frame(X * T + f) for f in range(T)], axis=1)

    def chunks(self, n: int, T: int) -> Iterator[np.ndarray]:
        for X in range(n):
            yield self.chunk(X, T)


# ---------------------------------------------------------------------------
# Stream-VAE stand-in: Wan-VAE-shaped causal 3D-conv encoder /
# decoder, shapes and init law only (no arithmetic).  Channels per stage (Wan2.1 VAE:
# base 96, multipliers 1, 2, 4), 3x3x3 causal convs, RMS gains.
# ---------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class VaeDesc:
    dims: Tuple[int, int, int] = (96, 192, 384)
    latent_channels: int = 16
    video_channels: int = 3
    frames_per_chunk: int = 4     # video frames per latent frame (temporal factor 4)
    eps: float = 1e-6


VAE = VaeDesc()


def vae_layers(vd: VaeDesc = VAE):
    """Ordered layer list: (name, kind, cin, cout) with kind in {conv, res, norm, pool_s,
    pool_st, up_s, up_st}.  res = RMS-SiLU-conv-RMS-SiLU-conv + skip (channels c)."""
    c1, c2, c3 = vd.dims
    enc = [("enc.conv_in", "conv", vd.video_channels, c1), ("enc.res1", "res", c1, c1), ("enc.p1", "pool_s", c1, c1),
           ("enc.conv2", "conv", c1, c2), ("enc.res2", "res", c2, c2), ("enc.p2", "pool_st", c2, c2),
           ("enc.conv3", "conv", c2, c3), ("enc.res3", "res", c3, c3), ("enc.p3", "pool_st", c3, c3),
           ("enc.res4", "res", c3, c3), ("enc.norm_out", "norm", c3, c3),
           ("enc.conv_out", "conv", c3, vd.latent_channels)]
    dec = [("dec.conv_in", "conv", vd.latent_channels, c3), ("dec.res1", "res", c3, c3), ("dec.u1", "up_st", c3, c3),
           ("dec.conv2", "conv", c3, c3), ("dec.res2", "res", c3, c3), ("dec.u2", "up_st", c3, c3),
           ("dec.conv3", "conv", c3, c2), ("dec.res3", "res", c2, c2), ("dec.u3", "up_s", c2, c2),
           ("dec.conv4", "conv", c2, c1), ("dec.res4", "res", c1, c1), ("dec.norm_out", "norm", c1, c1),
           ("dec.conv_out", "conv", c1, vd.video_channels)]
    return enc, dec


def vae_tensor_specs(vd: VaeDesc = VAE):
    """name -> (shape, law); conv weights [cout, 3, 3, 3, cin] and biases U(+-1/sqrt(27 cin)),
    RMS gains 1 + 0.1 N(0, 1)."""
    out = {}
    enc, dec = vae_layers(vd)
    for name, kind, ci, co in enc + dec:
        if kind == "conv":
            out[f"vae.{name}.w"] = ((co, 3, 3, 3, ci), ("u", 27 * ci))
            out[f"vae.{name}.b"] = ((co,), ("u", 27 * ci))
        elif kind == "res":
            for k in ("1", "2"):
                out[f"vae.{name}.n{k}"] = ((ci,), ("gain",))
                out[f"vae.{name}.c{k}.w"] = ((ci, 3, 3, 3, ci), ("u", 27 * ci))
                out[f"vae.{name}.c{k}.b"] = ((ci,), ("u", 27 * ci))
        elif kind == "norm":
            out[f"vae.{name}.g"] = ((ci,), ("gain",))
    return out


def gen_vae_weights(vd: VaeDesc = VAE, seed: int = 0) -> Dict[str, np.ndarray]:
    out = {}
    for name, (shape, law) in vae_tensor_specs(vd).items():
        r = _rng(seed, name)
        if law[0] == "u":
            bound = 1.0 / np.sqrt(law[1])
            a = r.uniform(-bound, bound, size=shape)
        else:
            a = 1.0 + 0.1 * r.standard_normal(size=shape)
        out[name] = round_to_bf16(a.astype(np.float32))
    return out


def gen_video(vd: VaeDesc, frames: int, H: int, W: int, seed: int = 5) -> np.ndarray:
    """A moving synthetic video [3, frames, H, W] fp32 (sinusoid field, translation + noise)."""
    ls = LatentStream(vd.video_channels, H, W, seed=seed, speeds=(0.0, 1.0, 3.0), segment=4)
    return np.stack([ls.frame(g) for g in range(frames)], axis=1)
