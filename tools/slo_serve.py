"""Online SLO-aware batching ("continuously adapts B to the observed
end-to-end latency so that the per-stream rate satisfies f_SLO"): a serving loop over
handles with B = 1..Bmax batched streams (1.3B 480p, n = 1); each iteration runs one call
of the current B, observes its latency (CUDA events), and the library's AIMD controller
(sdv2_slo_adapt) picks the next B.  Also the offline choice (sdv2_slo_select) from the
latencies measured here.

  python tools/slo_serve.py out.json [f_slo_per_stream] [iterations] [Bmax]"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen as sg  # noqa: E402


def main():
    import torch
    from bench import gen_weights_parallel
    from paper_2511_07399_b200.sdv2 import SDV2_BF16, SloAdapter, Stage, slo_select
    out = sys.argv[1]
    f_slo = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 80
    bmax = int(sys.argv[4]) if len(sys.argv) > 4 else 6
    cfg = sg.CONFIGS["wan13_480p_1step"]
    md, g, sd = cfg.model, cfg.geom, cfg.stream
    W = gen_weights_parallel(md)
    ls = [sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1 + b) for b in range(bmax)]
    chunks = torch.from_numpy(np.stack([np.stack([l.chunk(X, 1) for l in ls]) for X in range(8)])).cuda()
    stages, outs = {}, {}
    for B in range(1, bmax + 1):
        st = Stage(md, dataclasses.replace(g, streams=B), W, precision=SDV2_BF16)
        st.reset_stream(sd, [sg.gen_prompt(md, b) for b in range(B)])
        stages[B] = st
        outs[B] = torch.empty((B,) + tuple(chunks.shape[2:]), device="cuda")
    calls = {B: 0 for B in stages}

    def run(B):
        st = stages[B]
        x = chunks[calls[B] % 8, :B].contiguous()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st.stream)
        st.denoise_chunk(x.data_ptr(), outs[B].data_ptr())
        b.record(st.stream)
        b.synchronize()
        calls[B] += 1
        return a.elapsed_time(b) / 1e3

    table = {}
    for B in stages:                      # measured L(1, B) (after 3 warm-up calls)
        for _ in range(3):
            run(B)
        table[(1, B)] = float(np.median([run(B) for _ in range(5)]))
    deadline = 1.0 / f_slo
    offline = slo_select(table, f_slo, deadline, bmax, bmax)
    ad = SloAdapter(1, 1, bmax, 3, f_slo, deadline)
    traj = []
    for it in range(iters):
        B = ad.st.streams
        lat = run(B)
        r = ad.adapt(lat)
        traj.append({"B": B, "latency_ms": lat * 1e3, "per_stream_fps": 4 / lat, "next_B": r["B"],
                     "infeasible": r["infeasible"]})
    tail = [t["B"] for t in traj[-30:]]
    res = {"workload": "wan13_480p_1step, B streams per call, n = 1", "f_slo_per_stream": f_slo,
           "frame_deadline_s": deadline, "table_ms": {f"B{B}": v * 1e3 for (_, B), v in table.items()},
           "offline_choice": offline, "aimd_trajectory": traj, "aimd_tail_B": tail,
           "aimd_tail_mean_B": float(np.mean(tail)),
           "aimd_tail_fps": float(np.mean([4 * t["B"] / (t["latency_ms"] / 1e3) for t in traj[-30:]]))}
    for st in stages.values():
        st.close()
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "aimd_trajectory"}))


if __name__ == "__main__":
    main()
