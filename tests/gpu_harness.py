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


def multi_inputs(cfg, B, n_chunks, switches):
    """Per-stream inputs for a B-stream handle: stream b has its own latent stream
    (seed 1 + b), its own prompts and prompt switches (switches[b] = chunk indices)."""
    md, g = cfg.model, cfg.geom
    W = sg.gen_weights(md, seed=0)
    chunks, prompts = [], []
    for b in range(B):
        ls = sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1 + b, segment=2 + b)
        chunks.append([ls.chunk(X, g.chunk_frames) for X in range(n_chunks)])
        prompts.append([sg.gen_prompt(md, 10 * b + k) for k in range(1 + len(switches[b]))])
    return W, chunks, prompts


def stream_oracles(cfg, W, chunks, prompts, switches, dtype=np.float64, n_oracle=None):
    """Stream b through its own oracle with Philox key (seed_lo, seed_hi + b)."""
    import dataclasses
    from oracle.stream import StreamOracle
    recs = []
    for b in range(len(chunks)):
        sd = dataclasses.replace(cfg.stream, seed=cfg.stream.seed + (b << 32))
        o = StreamOracle(cfg.model, cfg.geom, sd, W, dtype=dtype, tap=True)
        starts = [0, *switches[b]]
        rb = []
        for X, v in enumerate(chunks[b][:n_oracle]):
            P = prompts[b][starts.index(X)] if X in starts else None
            rb.append(o.step_chunk(X, v, P))
        recs.append(rb)
    return recs


def run_gpu_streams(cfg, W, chunks, prompts, switches, prec, tap=True):
    """B streams batched in one handle (geometry.streams = B)."""
    import dataclasses
    import torch
    md = cfg.model
    B = len(chunks)
    g = dataclasses.replace(cfg.geom, streams=B)
    stage = Stage(md, g, W, precision=prec)
    stage.reset_stream(cfg.stream, [p[0] for p in prompts])
    L = g.tokens_per_chunk(md)
    NE = g.steps * B
    tap_t = torch.zeros((md.num_blocks, NE * L, md.dim), dtype=torch.float32, device="cuda") if tap else None
    if tap:
        stage.set_block_tap(tap_t)
    out_buf = torch.zeros((B,) + chunks[0][0].shape, dtype=torch.float32, device="cuda")
    outs, taps, meta = [{} for _ in range(B)], [{} for _ in range(B)], [{} for _ in range(B)]
    for c in range(len(chunks[0])):
        for b in range(B):
            if c in switches[b]:
                stage.set_prompt(prompts[b][1 + list(switches[b]).index(c)], stream=b)
        vin = torch.from_numpy(np.stack([chunks[b][c] for b in range(B)])).cuda()
        oc = stage.denoise_chunk(vin.data_ptr(), out_buf.data_ptr())
        torch.cuda.synchronize()
        info = stage.tick_info()
        if oc >= 0:
            ob = out_buf.cpu().numpy()
            for b in range(B):
                outs[b][oc] = ob[b].copy()
        tp = tap_t.cpu().numpy() if tap else None
        for j in range(g.steps):
            X = info["chunk"][j]
            if X < 0:
                continue
            for b in range(B):
                e = j * B + b
                if tap:
                    taps[b][(X, j)] = [tp[blk, e * L:(e + 1) * L].copy() for blk in range(md.num_blocks)]
                st = stage.cache_state(0, e)
                meta[b][(X, j)] = ({s: (st.tag[s], st.pos[s]) for s in range(st.num_slots) if st.tag[s] >= 0},
                                   st.noise_rate, st.d_hat)
    stage.close()
    return outs, taps, meta
