"""SLO-aware batch choice from MEASURED bench lines.

  python tools/slo_table.py out.json bench_B1.json bench_B2.json ...

Each bench line (bench.py --streams B) gives one point of L(T', B): the device time of
one call (ms_per_step) with B streams batched.  The library's scheduler
(sdv2_slo_select) picks (T', B) for a few per-stream output-frame-rate SLOs, the
deadline = 1 / f_SLO per frame; the memory-bound latency model of P:178 is fitted too."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_07399_b200.sdv2 import slo_fit, slo_select  # noqa: E402

out = sys.argv[1]
table, src = {}, {}
for f in sys.argv[2:]:
    d = json.load(open(f))
    B = d["config"].get("streams", 1)
    T = d["config"]["latent"][1]
    table[(T, B)] = d["ms_per_step"] / 1e3
    src[f"T{T}_B{B}"] = {"ms_per_call": d["ms_per_step"], "aggregate_fps": d["value"],
                         "per_stream_fps": d.get("per_stream_fps"), "gemm_frac": d["roofline"]["frac"],
                         "sm_mhz": d["clocks"]["sm_mhz"], "file": os.path.basename(f)}
a, b = slo_fit(table)
res = {"table": src, "model_L_eq_a_plus_b_BT": {"a_s": a, "b_s_per_latent_frame": b},
       "decisions": {}}
bmax = max(B for _, B in table)
for f_slo in (16.0, 30.0, 60.0, 120.0, 240.0):
    for buffered in (1, 4, 8):
        res["decisions"][f"f_slo={f_slo:g} buffered={buffered}"] = slo_select(table, f_slo, 1.0 / f_slo, buffered,
                                                                              bmax)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res["decisions"], indent=0)[:1500])
