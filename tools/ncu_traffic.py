"""Per-launch DRAM traffic and tensor-pipe use of the tensor-core kernels of one DiT block,
from one `ncu --set full` capture (tools/ncu_block.sh) -> profiles/<tag>_ncu_traffic.json,
which bench.py reads for roofline.traffic (GEMM class: mean bytes per launch).
  python tools/ncu_traffic.py <prof.ncu-rep> <out.json> <workload>"""
import csv
import json
import subprocess
import sys

rep, out, workload = sys.argv[1:4]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units = rows[0], rows[1]


def val(r, k):
    i = hdr.index(k)
    v = float(r[i].replace(",", ""))
    u = units[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
                "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(u, 1.0)


UTC = "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"
launches = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("sdv2::", "")
    launches.append({"kernel": name, "duration_us": val(r, "gpu__time_duration.sum"),
                     "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                     "tensor_pipe_pct": float(r[hdr.index(UTC)]) if UTC in hdr else None})
g = [x for x in launches if x["kernel"].startswith("gemm_tc")]
res = {"workload": workload, "source": rep.split("/")[-1], "launches": launches,
       "gemm_mean_dram_bytes_per_launch": sum(x["dram_bytes"] for x in g) / max(1, len(g)),
       "note": "ncu --set full --clock-control none, caches flushed between kernels (cold): traffic is an upper "
               "bound on the in-step (L2-warm) value"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res)[:600])
