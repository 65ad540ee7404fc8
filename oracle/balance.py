"""Online DiT-block rebalancing (oracle side).

Test infrastructure only (see oracle/__init__.py).

PAPER.md P:231-233 (§3.3 "DiT Block Scheduler"): "dynamically reallocates blocks between
devices based on measured execution time ... searches for an optimal partition that
minimizes per-stage latency".  SPEC.md S:201-209 (rebalance_online): re-run balance on
EMA-smoothed measured times; adopt the new partition only if the predicted max-stage
improvement exceeds a hysteresis.  The optimum is the brute-force one (control.py).
"""
from __future__ import annotations

from . import control as C


def rebalance_online(measured, stages, cur_bounds, ema, extra_first=0.0, extra_last=0.0, alpha=0.5,
                     hysteresis=0.05):
    """Returns (new_ema, changed, pred_cur, pred_opt): ema_b = alpha m_b + (1 - alpha) ema_b
    (first sample when ema_b == 0); pred_cur = max stage of cur_bounds on the EMA; pred_opt =
    brute-force optimum; changed iff pred_cur - pred_opt > (hysteresis + 1e-9) pred_cur."""
    new_ema = [m if e <= 0.0 else alpha * m + (1.0 - alpha) * e for m, e in zip(measured, ema)]
    cur = max(C.stage_times(new_ema, cur_bounds, extra_first, extra_last))
    opt = C.brute_force_partition(new_ema, stages, extra_first, extra_last)
    changed = cur - opt > (hysteresis + 1e-9) * cur      # 1e-9: rounding ties never move blocks
    return new_ema, changed, cur, (opt if changed else cur)
