"""Sequential stream algorithm O1–O7 (oracle side).

Test infrastructure only (see oracle/__init__.py).

Order: for chunk X: admit (motion controller P:205–219, control record P:190–191),
then for step j = 0..n-1 run entry (X, j) on lane j (R1): DiT forward with the
lane's explicit [sink || window] list, flow-matching x0 prediction, re-noise
(O5).  By O6 any order that respects (X, j-1) -> (X, j) and per-lane chunk
order yields the same per-entry math; this sequential order is the reference
for the stream-batched and pipelined GPU executions.

kv_mode 1 (reading Q5-clean; n = 1 only): before chunk X is admitted, the
finished chunk X-1 is re-run through the DiT on its prediction x0 at sigma = 0 (t = 0,
CausVid's clean-context pass, EXT) and the K/V of that pass replace its step-0 K/V in the
cache (LaneCache.overwrite): later chunks attend to clean K/V of earlier chunks.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional

import numpy as np

from . import model as M
from .control import ControlPlane, LaneCache, MotionController
from .philox import gaussian_noise


class StreamOracle:
    def __init__(self, md, geom, sd, W: Dict[str, np.ndarray], dtype=np.float64,
                 blocks: Optional[List[int]] = None, tap: bool = False):
        self.md, self.g, self.sd, self.W, self.dt = md, geom, sd, W, dtype
        self.blocks = list(range(md.num_blocks)) if blocks is None else list(blocks)
        self.L = geom.tokens_per_chunk(md)
        self.ctl = ControlPlane(geom, sd.rope_reset_frames, sd.sink_tau)
        self.motion = MotionController(sd)
        self.lanes = {(b, j): LaneCache(geom.sink_chunks, geom.window_chunks, sd.rope_reset_frames)
                      for b in self.blocks for j in range(geom.steps)}
        self.tap = tap
        self.clean = getattr(geom, "kv_mode", 0) == 1
        if self.clean and geom.steps != 1:
            raise ValueError("the clean re-run (kv_mode 1) is defined for n = 1")
        self.prompt = None
        self.ctx_kv = None
        self.h = None
        self.records: List[dict] = []

    # -------------------------------------------------------------- prompt
    def set_prompt(self, P):
        """C.3: text embedding and per-block cross K/V; h = mean-pooled prompt (fp64, Q8)."""
        dt = self.dt
        h = np.mean(np.asarray(P, dtype=np.float64), axis=0)
        if np.linalg.norm(h) == 0.0:
            raise ValueError("zero-norm prompt mean")
        ctx = M.text_embed(P, self.W, dt)
        self.ctx_kv = {b: M.prompt_kv(ctx, self.W, b, self.md, dt) for b in self.blocks}
        self.h = h

    def admit_control(self, X):
        """Control record of chunk X; it also pins the prompt version (cross K/V) in effect."""
        act = self.ctl.admit(X, self.h)
        act["ctx_kv"] = self.ctx_kv
        return act

    # ------------------------------------------------------------- one block
    def block(self, x, e0, b, lane: LaneCache, act, rerun: bool = False):
        md, dt, W = self.md, self.dt, self.W
        p = f"blocks.{b}."
        w = lambda n: W[p + n].astype(dt)
        H, hd = md.num_heads, md.head_dim
        mod = w("mod") + e0                              # [6, d]
        sh1, sc1, g1, sh2, sc2, g2 = mod
        # 1. adaLN norm1 + modulate
        a = M.norm(x, md) * (1 + sc1) + sh1
        # 2. projections + qk RMSNorm over the full dim
        q = M.rms_g(M.linear(a, w("wq"), w("bq")), w("gq"), md.eps)
        k = M.rms_g(M.linear(a, w("wk"), w("bk")), w("gk"), md.eps)
        v = M.linear(a, w("wv"), w("bv"))
        # 4. cache update (re-base, write/refresh) then attention over all valid entries
        if rerun:
            lane.overwrite(act, k, v)
        else:
            lane.apply(act, k, v, self.g.chunk_frames)
        pt_q, ph_q, pw_q = M.token_positions(md, self.g, act["pos"])
        R = x.shape[0]          # a chunk, or a row prefix of one (bench sample only)
        phi_q = M.rope_angles(hd, pt_q[:R], ph_q[:R], pw_q[:R])
        ents = lane.attended()
        keys, vals = [], []
        for e in ents:
            pt, ph, pw = M.token_positions(md, self.g, e.pos)
            nk = e.k.shape[0]
            phi = M.rope_angles(hd, pt[:nk], ph[:nk], pw[:nk])
            keys.append((e.k, phi))
            vals.append(e.v)
        o = np.zeros_like(x)
        for hh in range(H):
            cs = slice(hh * hd, (hh + 1) * hd)
            qh = M.rope_apply(q[:, cs], phi_q)
            kh = np.concatenate([M.rope_apply(kk[:, cs], phi) for kk, phi in keys], axis=0)
            vh = np.concatenate([vv[:, cs] for vv in vals], axis=0)
            o[:, cs] = M.attention(qh, kh, vh)
        # 5. out projection, gated residual
        x = x + g1 * M.linear(o, w("wo"), w("bo"))
        # 6–7. cross-attention (affine norm3, RMS q, ungated residual)
        a3 = M.norm(x, md) * w("n3_g") + w("n3_b")
        qc = M.rms_g(M.linear(a3, w("wcq"), w("bcq")), w("gcq"), md.eps)
        Kc, Vc = act["ctx_kv"][b]
        oc = np.zeros_like(x)
        for hh in range(H):
            cs = slice(hh * hd, (hh + 1) * hd)
            oc[:, cs] = M.attention(qc[:, cs], Kc[:, cs], Vc[:, cs])
        x = x + M.linear(oc, w("wco"), w("bco"))
        # 8. FFN, gated residual
        a2 = M.norm(x, md) * (1 + sc2) + sh2
        x = x + g2 * M.linear(M.gelu_tanh(M.linear(a2, w("w1"), w("b1"))), w("w2"), w("b2"))
        return x

    # ------------------------------------------------------------ DiT forward
    def dit(self, x_lat, sigma, j, act, taps=None):
        md, dt, W = self.md, self.dt, self.W
        u = M.patchify(x_lat.astype(dt), md)
        x = M.linear(u, W["patch_w"].astype(dt), W["patch_b"].astype(dt))
        e, e0 = M.time_embed(sigma, W, md, dt)
        for b in self.blocks:
            x = self.block(x, e0, b, self.lanes[(b, j)], act)
            if taps is not None:
                taps.append(x.copy())
        y = M.head(x, e, W, md, dt)
        C, T, h, w_ = x_lat.shape
        return M.unpatchify(y, md, T, h, w_)

    def clean_rerun(self, rec: dict):
        """Re-run finished chunk rec["X"] on its prediction x0 at sigma = 0 (t = 0), with the
        control record it was admitted with; its K/V replace its step-0 K/V in every block's
        lane (Q5-clean).  The head is not evaluated (the pass only writes the cache)."""
        md, dt, W = self.md, self.dt, self.W
        act = rec["act"]
        u = M.patchify(rec["out"].astype(dt), md)
        x = M.linear(u, W["patch_w"].astype(dt), W["patch_b"].astype(dt))
        _, e0 = M.time_embed(np.float32(0.0), W, md, dt)
        for b in self.blocks:
            x = self.block(x, e0, b, self.lanes[(b, 0)], act, rerun=True)

    # ------------------------------------------------------------- one chunk
    def step_chunk(self, X: int, v_X, prompt=None) -> dict:
        """Admit chunk X, run its n entries sequentially; returns output x0 and records."""
        if prompt is not None:
            self.set_prompt(prompt)
        dt, sd, g = self.dt, self.sd, self.g
        if self.clean and self.records:
            self.clean_rerun(self.records[-1])
        mot = self.motion.admit(v_X)
        act = self.admit_control(X)
        sig = mot["sigmas"]
        numel = v_X.size
        eps = lambda j: gaussian_noise(sd.seed, X, j, numel).reshape(v_X.shape).astype(dt)
        s0 = dt(sig[0])
        x = (1 - s0) * v_X.astype(dt) + s0 * eps(0)
        taps = [] if self.tap else None
        entries = []
        out = None
        for j in range(g.steps):
            sj = dt(sig[j])
            et = [] if self.tap else None
            vhat = self.dit(x, sig[j], j, act, et)
            x0 = x - sj * vhat
            entries.append({"x_in": x, "vhat": vhat, "x0": x0, "taps": et})
            if j < g.steps - 1:
                sn = dt(sig[j + 1])
                x = (1 - sn) * x0 + sn * eps(j + 1)
            else:
                out = x0
        rec = {"X": X, "act": act, "motion": mot, "out": out, "entries": entries,
               "lane_state": {bj: ln.state() for bj, ln in self.lanes.items()}}
        self.records.append(rec)
        return rec


def run_stream(cfg, W, chunks, prompts, dtype=np.float64, blocks=None, tap=False) -> List[dict]:
    """Run the whole stream: chunks is a list of [C,T',h,w]; prompts[k] takes effect at
    cfg.prompt_switch[k-1] (prompt 0 from chunk 0)."""
    o = StreamOracle(cfg.model, cfg.geom, cfg.stream, W, dtype=dtype, blocks=blocks, tap=tap)
    starts = [0, *cfg.prompt_switch]
    recs = []
    for X, v in enumerate(chunks):
        P = None
        if X in starts:
            P = prompts[starts.index(X)]
        recs.append(o.step_chunk(X, v, P))
    return recs
