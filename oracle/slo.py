"""SLO-aware batching scheduler (oracle side).

Test infrastructure only (see oracle/__init__.py).

Paper (§3.1 "SLO-aware batching scheduler"): given a target frame
rate f_SLO, the system processes T frames per iteration with latency L(T, B); "the
product B.T must not exceed the number of frames already collected from the input
stream"; the scheduler "adaptively converges to an optimal batch size B*" and
"continuously adapts B to the observed end-to-end latency so that the per-stream rate
satisfies f_SLO".  SPEC.md S:120-147 (module slo_batcher) fixes the interface used
here: select_batch = exhaustive search over the measured L(T, B) table; adapt = AIMD.

Units (reading N2-a in DESIGN.md): T = latent frames per chunk (T'), each latent frame
is `px_per_latent` output frames (Wan VAE temporal factor 4, reading Q23); one call of
the library emits one clean chunk per stream per call in steady state, so a stream's
output rate is px_per_latent * T / L and the batch's throughput is B times that.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple


def select_batch(table: Dict[Tuple[int, int], float], f_slo: float, deadline_s: float, buffered_frames: int,
                 b_max: int, px_per_latent: int = 4) -> dict:
    """Exhaustive search over the measured table {(T, B): latency seconds}.

    Feasible (T, B): B <= b_max, B T <= buffered_frames, per-stream rate
    px T / L >= f_slo, and chunk latency L <= deadline_s * px T (per-frame deadline).
    Objective: throughput px B T / L; ties -> smaller B, then smaller T.
    No feasible pair -> the smallest-latency pair with B T <= buffered (B = 1 if
    possible), flagged infeasible (never silently relaxed).
    buffered_frames < min T -> error."""
    if not table:
        raise ValueError("empty latency table")
    min_t = min(t for t, _ in table)
    if buffered_frames < min_t:
        raise ValueError("not enough input: buffered frames < T")
    best = None
    for (t, b), lat in sorted(table.items()):
        if b > b_max or b * t > buffered_frames or lat <= 0:
            continue
        rate = px_per_latent * t / lat
        if rate < f_slo or lat > deadline_s * px_per_latent * t:
            continue
        thr = b * rate
        key = (-thr, b, t)
        if best is None or key < best[0]:
            best = (key, t, b, lat)
    if best is not None:
        _, t, b, lat = best
        return {"T": t, "B": b, "latency": lat, "fps": px_per_latent * b * t / lat, "feasible": True}
    # infeasible: B = 1 at the fastest T that fits the buffer
    cands = [(lat, t, b) for (t, b), lat in table.items() if b * t <= buffered_frames and b <= b_max]
    ones = [c for c in cands if c[2] == 1]
    lat, t, b = min(ones or cands)
    return {"T": t, "B": b, "latency": lat, "fps": px_per_latent * b * t / lat, "feasible": False}


class AimdState:
    """SPEC S:136-146 adapt: multiplicative decrease (halve, floor 1) on an SLO violation,
    additive increase (+1, cap b_max) after `streak` consecutive compliant iterations."""

    def __init__(self, B: int, T: int, b_max: int, streak: int):
        self.B, self.T, self.b_max, self.streak = B, T, b_max, streak
        self.ok_run = 0
        self.infeasible = False

    def adapt(self, observed_latency: float, f_slo: float, deadline_s: float, px_per_latent: int = 4) -> dict:
        if observed_latency <= 0:
            raise ValueError("observed latency must be positive")
        rate = px_per_latent * self.T / observed_latency
        violated = rate < f_slo or observed_latency > deadline_s * px_per_latent * self.T
        if violated:
            self.infeasible = self.B == 1
            self.B = max(1, self.B // 2)
            self.ok_run = 0
        else:
            self.infeasible = False
            self.ok_run += 1
            if self.ok_run >= self.streak:
                self.B = min(self.b_max, self.B + 1)
                self.ok_run = 0
        return {"B": self.B, "infeasible": self.infeasible}


def fit_latency_model(table: Dict[Tuple[int, int], float]) -> Tuple[float, float]:
    """in the memory-bound regime L(T, B) ~ (A(T, B) + P_model) / (eta BW) with the
    activation footprint A linear in B T, i.e. L = a + b (B T).  Ordinary least squares
    over the table points (plain sums)."""
    pts: List[Tuple[float, float]] = [(float(b * t), lat) for (t, b), lat in table.items()]
    n = len(pts)
    sx = sum(x for x, _ in pts)
    sy = sum(y for _, y in pts)
    sxx = sum(x * x for x, _ in pts)
    sxy = sum(x * y for x, y in pts)
    den = n * sxx - sx * sx
    if n < 2 or den == 0:
        raise ValueError("need two distinct B T values")
    b = (n * sxy - sx * sy) / den
    a = (sy - b * sx) / n
    return a, b
