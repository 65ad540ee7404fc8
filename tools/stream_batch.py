"""E10 (Fig. 10 "Stream Batch substantially improves throughput"): time per
clean chunk with Stream Batch (n = 4 entries batched in one tick) vs without (the same
4 denoising passes run one per tick, M = L each: 4 ticks of an n = 1 handle).

  python tools/stream_batch.py out.json on.json off_n1.json
on.json = bench.py --config wan13_512_4step; off_n1.json = the same with --denoise-steps 1."""
import json
import sys

out, on_f, off_f = sys.argv[1:4]
on, off = json.load(open(on_f)), json.load(open(off_f))
n = on["config"]["steps_n"]
on_ms = on["ms_per_step"]                 # one tick emits one clean chunk in steady state
off_ms = n * off["ms_per_step"]           # n sequential passes of one entry each
px = on["config"]["px_frames_per_chunk"]
res = {"workload": on["config"]["workload"], "steps_n": n,
       "stream_batch_on": {"ms_per_clean_chunk": on_ms, "fps": px * 1e3 / on_ms, "gemm_frac": on["roofline"]["frac"],
                           "sm_mhz": on["clocks"]["sm_mhz"]},
       "stream_batch_off": {"ms_per_clean_chunk": off_ms, "fps": px * 1e3 / off_ms,
                            "gemm_frac": off["roofline"]["frac"], "sm_mhz": off["clocks"]["sm_mhz"],
                            "note": f"{n} x the n = 1 tick (one entry, M = L rows per pass)"},
       "speedup": off_ms / on_ms}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
