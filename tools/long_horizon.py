"""configs[4] long-horizon run: 1.3B 480p, n = 4, m = 1, W = 4, T_reset = 240,
10,000 chunks, prompt switch every 2500 chunks, scene cut every 2048 chunks.  Reports the
output FPS per 500-chunk window (device events, one per call), the whole-run FPS, and the
cache metadata sampled every 250 chunks against the oracle control-plane replay
(oracle/control.py: resets, positions, evictions of lane 0).

  python tools/long_horizon.py out.json [num_chunks]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthgen as sg  # noqa: E402


def main():
    import torch
    from bench import ClockSampler, gen_weights_parallel
    from oracle import control as C
    from paper_2511_07399_b200.sdv2 import SDV2_BF16, Stage
    out = sys.argv[1]
    cfg = sg.CONFIGS["long_horizon"]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.num_chunks
    debug = os.environ.get("LH_DEBUG") == "1"     # sync + print every call from 2990 on
    md, g, sd = cfg.model, cfg.geom, cfg.stream
    n = g.steps
    W = gen_weights_parallel(md)
    stage = Stage(md, g, W, precision=SDV2_BF16)
    torch.cuda.set_stream(stage.stream)
    prompts = [sg.gen_prompt(md, k) for k in range(1 + len(cfg.prompt_switch))]
    seg = 256
    scenes = {}

    def chunk(X):          # scene k = X // 2048 (a cut: new field), 256 consecutive frames cycled
        k = X // 2048
        if k not in scenes:
            ls = sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1 + k)
            scenes[k] = torch.from_numpy(np.stack([ls.chunk(i, g.chunk_frames) for i in range(seg)])).cuda()
        return scenes[k][X % seg]

    for k in range((N + 2047) // 2048):
        chunk(k * 2048)
    out_dev = torch.empty(tuple(chunk(0).shape), dtype=torch.float32, device="cuda")
    stage.reset_stream(sd, prompts[0])
    # oracle control-plane replay (metadata only)
    octl = C.ControlPlane(g, sd.rope_reset_frames, sd.sink_tau)
    olane = C.LaneCache(g.sink_chunks, g.window_chunks, sd.rope_reset_frames)
    pidx = [sum(1 for s in cfg.prompt_switch if X >= s) for X in range(N + n)]
    hs = [np.mean(np.asarray(p, np.float64), axis=0) for p in prompts]
    evs, outs = [], []
    meta_checked, meta_ok = 0, True
    clk = ClockSampler(0)
    clk.start()
    t0 = time.time()
    start = torch.cuda.Event(enable_timing=True)
    start.record(stage.stream)
    for c in range(N + n - 1):
        if debug and c == 3130:
            import ctypes
            stage.L.sdv2_debug_sync.argtypes = [ctypes.c_void_p, ctypes.c_int32]
            stage.L.sdv2_debug_sync(stage.h, 1)
        if c % 1000 == 0 or (debug and c >= 2990):
            if debug:
                torch.cuda.synchronize()
            print(f"call {c} t={time.time() - t0:.1f}s", file=sys.stderr, flush=True)
        if c in cfg.prompt_switch:
            stage.set_prompt(prompts[pidx[c]])
        X = min(c, N - 1)
        oc = stage.denoise_chunk(chunk(X).data_ptr(), out_dev.data_ptr())
        e = torch.cuda.Event(enable_timing=True)
        e.record(stage.stream)
        evs.append(e)
        outs.append(oc)
        if c < N:
            act = octl.admit(c, hs[pidx[c]])
            olane.apply(act, None, None, g.chunk_frames)
            if c % 250 == 0 or act["rebase"] or any(act["refresh"]):
                st = stage.cache_state(0, 0)            # lane 0 holds chunk c after this call
                ost = olane.state()
                got = {s: (st.tag[s], st.pos[s]) for s in range(st.num_slots) if st.tag[s] >= 0}
                exp = {s: (t, p[0]) for s, (t, p) in ost.items()}
                meta_ok &= got == exp and st.resets == act["r"] and st.evictions == olane.evictions
                meta_checked += 1
    torch.cuda.synchronize()
    wall = time.time() - t0
    clocks = clk.stop()
    px = 4 * g.chunk_frames
    t_end = [start.elapsed_time(e) for e in evs]
    emit = [(c, oc) for c, oc in enumerate(outs) if oc >= 0]
    windows = []
    for w0 in range(0, N, 500):
        cs = [c for c, oc in emit if w0 <= oc < w0 + 500]
        if len(cs) < 2:
            continue
        dt = (t_end[cs[-1]] - t_end[cs[0] - 1]) / 1e3 if cs[0] > 0 else t_end[cs[-1]] / 1e3
        windows.append({"chunks": [w0, w0 + 500], "fps": px * len(cs) / dt})
    total = px * len(emit) / (t_end[-1] / 1e3)
    res = {"workload": "long_horizon (configs[4])", "chunks": N, "steps_n": n, "prompt_switches": list(cfg.prompt_switch),
           "scene_cut_every": 2048, "fps_total": total, "fps_windows": windows,
           "fps_window_min_max": [min(w["fps"] for w in windows), max(w["fps"] for w in windows)],
           "resets": int(octl.r), "evictions_lane0": int(olane.evictions),
           "metadata_vs_oracle": {"checked": meta_checked, "bit_exact": bool(meta_ok)},
           "wall_s": wall, "clocks": clocks}
    stage.close()
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "fps_windows"}))


if __name__ == "__main__":
    main()
