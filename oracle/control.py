"""Control plane of the stream (oracle side): motion-aware noise controller, RoPE
phase reset, adaptive sink refresh, rolling KV cache bookkeeping, and the
DiT-block partition.

Test infrastructure only (see oracle/__init__.py).  Integer / fp64 throughout.
"""
from __future__ import annotations

import itertools
from typing import List, Optional, Sequence

import numpy as np


# ------------------------------------------------ O4: motion-aware noise
def motion_intensity(v_cur, v_prev):
    """d_t = sqrt( ||v_t - v_{t-1}||^2 / (C H W) )   (fp64)."""
    a = np.asarray(v_cur, dtype=np.float64)
    b = np.asarray(v_prev, dtype=np.float64)
    return float(np.sqrt(np.sum((a - b) ** 2) / a.size))


def normalized_motion(window: Sequence[float], sigma: float) -> float:
    """d_hat = clip(max_{i in window} d_i / sigma, 0, 1)   (window = k+1 values, Q13)."""
    return float(min(max(max(window) / sigma, 0.0), 1.0))


def ema_rate(d_hat: float, s_prev: float, s_min: float, s_max: float, lam: float) -> float:
    """s_t = lam [s_max - (s_max - s_min) d_hat] + (1 - lam) s_{t-1}."""
    return lam * (s_max - (s_max - s_min) * d_hat) + (1.0 - lam) * s_prev


class MotionController:
    """Per-frame d, window of the last k+1 values, d_hat at the chunk's last frame,
    EMA noise rate s_X with s_{-1} = s_max (Q15); sigma_{X,j} = s_X t_j / t_0 (R5/Q16)."""

    def __init__(self, sd):
        self.sd = sd
        self.ds: List[float] = []
        self.prev_frame = None
        self.s = sd.s_max

    def admit(self, chunk) -> dict:
        """chunk [C, T', h, w] -> {d (per frame), d_hat, s, sigmas (fp32 per step)}."""
        sd = self.sd
        dlist = []
        for f in range(chunk.shape[1]):
            fr = chunk[:, f]
            d = 0.0 if self.prev_frame is None else motion_intensity(fr, self.prev_frame)
            self.ds.append(d)
            dlist.append(d)
            self.prev_frame = fr
        window = self.ds[-(sd.motion_k + 1):]
        d_hat = normalized_motion(window, sd.motion_sigma)
        self.s = ema_rate(d_hat, self.s, sd.s_min, sd.s_max, sd.ema_lambda)
        t0 = float(sd.timesteps[0])
        sigmas = [np.float32(self.s * float(t) / t0) for t in sd.timesteps]
        return {"d": dlist, "d_hat": d_hat, "s": self.s, "sigmas": sigmas}


# -------------------------------------------- RoPE phase reset (R3/Q11)
def rope_position(t: int, T_reset: int) -> int:
    """Repeated wrap of theta_t = theta_{t - T_reset} for t > T_reset."""
    while t > T_reset:
        t -= T_reset
    return t


# ------------------------------------- visual chunk embedding (N4 / Q8-visual)
def visual_embedding(chunk) -> np.ndarray:
    """h_X[c] = mean over (T', h, w) of latent channel c, fp64 (the visual reading of the
    paper's "chunk embedding h_t"; the default reading Q8 is the mean-pooled prompt)."""
    a = np.asarray(chunk, dtype=np.float64)
    return a.reshape(a.shape[0], -1).mean(axis=1)


# ----------------------------------------------- sink refresh (R4/Q9)
def cosine(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b)))


def sink_refresh(sinks: List[np.ndarray], h, tau: float):
    """alpha_i = cos(h, s_i); keep s_i if alpha_i >= tau, else s_i <- h.  Returns (new sinks, mask)."""
    mask = [cosine(h, s) < tau for s in sinks]
    return [np.asarray(h, dtype=np.float64) if r else s for s, r in zip(sinks, mask)], mask


# ------------------------------------------ per-chunk control record (O3)
class ControlPlane:
    """Chunk admission (O3): reset count r, temporal positions, sink fill / refresh
    decisions and the ring slot.  Actions are recorded once per chunk and replayed
    by every (block, lane) when it processes entry (X, j)."""

    def __init__(self, geom, T_reset: int, tau: float):
        self.g = geom
        self.T_reset = T_reset
        self.tau = tau
        self.r = 0
        self.sink_emb: List[Optional[np.ndarray]] = [None] * geom.sink_chunks

    def admit(self, X: int, h) -> dict:
        T, m, W = self.g.chunk_frames, self.g.sink_chunks, self.g.window_chunks
        rebase = False
        while X * T - self.r * self.T_reset > self.T_reset:
            self.r += 1
            rebase = True
        pos = [X * T + f - self.r * self.T_reset for f in range(T)]
        act = {"X": X, "pos": pos, "r": self.r, "rebase": rebase,
               "sink_fill": -1, "refresh": [False] * m, "ring_slot": -1}
        if X < m:
            act["sink_fill"] = X
            self.sink_emb[X] = np.asarray(h, dtype=np.float64)
        else:
            self.sink_emb, act["refresh"] = sink_refresh(self.sink_emb, h, self.tau)
            act["ring_slot"] = (X - m) % W
        return act


class CacheEntry:
    __slots__ = ("tag", "pos", "k", "v", "slot")

    def __init__(self, tag, pos, k, v, slot):
        self.tag, self.pos, self.k, self.v, self.slot = tag, list(pos), k, v, slot


class LaneCache:
    """Explicit temporal list for one (block, lane): m sink entries + a window of at
    most W chunks, oldest first (P:472 rolling KV cache; Q6/Q7).  Keys are stored
    un-rotated (post qk-norm) with their temporal positions; RoPE is applied at
    attention time, so a re-base is a position shift (R3)."""

    def __init__(self, m: int, W: int, T_reset: int):
        self.m, self.W, self.T_reset = m, W, T_reset
        self.sinks: List[Optional[CacheEntry]] = [None] * m
        self.window: List[CacheEntry] = []
        self.evictions = 0

    def apply(self, act: dict, k, v, T: int):
        # 1. re-base every ring entry (sinks keep their anchors, R3)
        if act["rebase"]:
            for e in self.window:
                e.pos = [p - self.T_reset for p in e.pos]
        # 2. write or refresh
        if act["sink_fill"] >= 0:
            i = act["sink_fill"]
            self.sinks[i] = CacheEntry(act["X"], act["pos"], k, v, i)
        else:
            for i, r in enumerate(act["refresh"]):
                if r:
                    self.sinks[i] = CacheEntry(act["X"], [i * T + f for f in range(T)], k, v, i)
            self.window.append(CacheEntry(act["X"], act["pos"], k, v, self.m + act["ring_slot"]))
            if len(self.window) > self.W:
                self.window.pop(0)
                self.evictions += 1

    def overwrite(self, act: dict, k, v):
        """Clean-context re-run (reading Q5-clean, N4): chunk act["X"]'s K/V are replaced
        in place -- its sink fill, or its window entry and the sinks it refreshed -- with
        tags, positions and slots unchanged (no admission, no eviction, no re-base)."""
        X = act["X"]
        if act["sink_fill"] >= 0:
            targets = [self.sinks[act["sink_fill"]]]
        else:
            targets = [self.sinks[i] for i, r in enumerate(act["refresh"]) if r] + [self.window[-1]]
        for e in targets:
            if e is None or e.tag != X:
                raise ValueError(f"clean re-run of chunk {X}: cache entry is not chunk {X}")
            e.k, e.v = k, v

    def attended(self) -> List[CacheEntry]:
        """[sinks || window] in temporal order, current chunk included."""
        return [s for s in self.sinks if s is not None] + list(self.window)

    def state(self) -> dict:
        """Slot metadata: physical slot -> (tag, positions) (bit-exact observable, O7)."""
        slots = {}
        for s in self.sinks:
            if s is not None:
                slots[s.slot] = (s.tag, tuple(s.pos))
        for e in self.window:
            slots[e.slot] = (e.tag, tuple(e.pos))
        return slots


# ------------------------------------- DiT block partition (a14)
def stage_times(costs, bounds, e_first=0.0, e_last=0.0):
    K = len(bounds) - 1
    out = []
    for s in range(K):
        t = sum(costs[bounds[s]:bounds[s + 1]])
        if s == 0:
            t += e_first
        if s == K - 1:
            t += e_last
        out.append(t)
    return out


def brute_force_partition(costs, K, e_first=0.0, e_last=0.0):
    """Exhaustive min-max over all contiguous splits; returns the optimum value."""
    B = len(costs)
    if K > B:
        raise ValueError("more stages than blocks")
    best = None
    for cuts in itertools.combinations(range(1, B), K - 1):
        bounds = [0, *cuts, B]
        v = max(stage_times(costs, bounds, e_first, e_last))
        best = v if best is None or v < best else best
    return best
