"""Helpers for the GPU parity tests: run the library on a seeded stream, collect
per-(chunk, step, block) block outputs, clean outputs and lane metadata."""
import numpy as np

import synthgen as sg
from paper_2511_07399_b200.sdv2 import Stage


def tiny_inputs(cfg, extra=0, segment=3):
    W = sg.gen_weights(cfg.model, seed=0)
    ls = sg.LatentStream(cfg.model.latent_channels, cfg.geom.latent_h, cfg.geom.latent_w, seed=1, segment=segment)
    chunks = [ls.chunk(X, cfg.geom.chunk_frames) for X in range(cfg.num_chunks + extra)]
    prompts = [sg.gen_prompt(cfg.model, k) for k in range(1 + len(cfg.prompt_switch))]
    return W, chunks, prompts


def run_gpu(cfg, W, chunks, prompts, prec, tap=True, blocks=None, stream_desc=None, graphs=True):
    import torch
    md, g = cfg.model, cfg.geom
    stage = Stage(md, g, W, precision=prec)
    stage.set_graphs(graphs)
    sd = stream_desc or cfg.stream
    stage.reset_stream(sd, prompts[0])
    L = g.tokens_per_chunk(md)
    n = g.steps
    tap_t = torch.zeros((md.num_blocks, n * L, md.dim), dtype=torch.float32, device="cuda") if tap else None
    if tap:
        stage.set_block_tap(tap_t)
    starts = [0, *cfg.prompt_switch]
    out_buf = torch.zeros(chunks[0].shape, dtype=torch.float32, device="cuda")
    outs, taps, meta = {}, {}, {}
    for c, v in enumerate(chunks):
        if c in starts and c > 0:
            stage.set_prompt(prompts[starts.index(c)])
        vin = torch.from_numpy(v).cuda()
        oc = stage.denoise_chunk(vin.data_ptr(), out_buf.data_ptr())
        torch.cuda.synchronize()
        info = stage.tick_info()
        if oc >= 0:
            outs[oc] = out_buf.cpu().numpy().copy()
        if tap:
            tp = tap_t.cpu().numpy()
            for j in range(n):
                X = info["chunk"][j]
                if X >= 0:
                    taps[(X, j)] = [tp[b, j * L:(j + 1) * L].copy() for b in range(md.num_blocks)]
        for j in range(n):
            X = info["chunk"][j]
            if X >= 0:
                st = stage.cache_state(0, j)
                meta[(X, j)] = ({s: (st.tag[s], st.pos[s]) for s in range(st.num_slots) if st.tag[s] >= 0},
                                st.noise_rate, st.d_hat)
    stage.close()
    return outs, taps, meta


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
