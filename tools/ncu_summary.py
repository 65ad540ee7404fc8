"""Summarise an ncu launch list (gpu__time_duration per launch) and a full capture into
a markdown file under profiles/.   python tools/ncu_summary.py <tag> <launches.csv> <prof.ncu-rep> <out.md>"""
import collections
import csv
import subprocess
import sys


def launch_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    iN, iV, iU, iM = (hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"),
                      hdr.index("Metric Name"))
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = r[iN].split("(")[0].replace("void ", "").replace("sdv2::", "")[:48]
        v = float(r[iV].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(r[iU], 1e-3)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = ["| kernel | launches | total µs | avg µs | share |", "|---|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {v:.1f} | {v / n:.2f} | {100 * v / tot:.1f}% |")
    return out, tot, sum(a[0] for a in agg.values())


KEYS = [("gpu__time_duration.sum", "duration"), ("launch__grid_size", "grid"),
        ("launch__registers_per_thread", "regs"), ("dram__bytes_read.sum", "DRAM rd"),
        ("dram__bytes_write.sum", "DRAM wr"),
        ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
         "tensor pipe (UTC bf16 HMMA ops) % of peak"),
        ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "TMEM/UTC active %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %")]


def full_table(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(n for _, n in KEYS) + " |", "|---|" + "---|" * len(KEYS)]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("sdv2::", "")[:40]
        vals = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
    return out


if __name__ == "__main__":
    tag, lcsv, rep, dst = sys.argv[1:5]
    lt, tot, n = launch_table(lcsv)
    lines = [f"# ncu summary {tag}", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over the bench's timed",
             f"region (NVTX range `timed`, 2 steps). Cold-cache, serialised: compare shares, not absolutes.",
             f"Total {tot:.1f} µs over {n} launches.", ""] + lt + ["", "Full capture (`--set full`):", ""] + full_table(rep)
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
