"""Pipeline parallelism through the real library on one GPU: two processes (rank 0 =
block 0, rank 1 = block 1 of the tiny model) exchange stage packets with gloo through
host staging.  The last rank's clean outputs must equal a single-stage run bitwise
(fp32 hand-off, batch-invariant kernels; SURVEY.md §8(e) pin P6)."""
import os
import socket

import numpy as np
import pytest

import synthgen as sg

NCALL = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(kind="tiny"):
    """tiny (configs[0]) or a 1.3B-shaped 2-block model at 480p, n = 1 (configs[1] block shapes)."""
    import dataclasses
    cfg = sg.CONFIGS["tiny"]
    if kind == "wan13":
        base = sg.CONFIGS["wan13_480p_1step"]
        cfg = dataclasses.replace(base, model=dataclasses.replace(base.model, num_blocks=2),
                                  stream=dataclasses.replace(base.stream, rope_reset_frames=4))
    md, g = cfg.model, cfg.geom
    W = sg.gen_weights(md, seed=0)
    ls = sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1, segment=3)
    chunks = [ls.chunk(X, 1) for X in range(NCALL)]
    prompts = [sg.gen_prompt(md, 0), sg.gen_prompt(md, 1)]
    return cfg, W, chunks, prompts


def _run(prec, rank, world, q=None, port=None, kind="tiny"):
    import torch
    from paper_2511_07399_b200.pipeline import StageTransport, balanced_ranges, run_pipelined, stage_io_tensors
    from paper_2511_07399_b200.sdv2 import Stage
    torch.cuda.set_device(0)
    cfg, W, chunks, prompts = _inputs(kind)
    if world > 1:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ranges, _ = balanced_ranges(cfg.model.num_blocks, world, 1.0, 0.0, 0.0)
        pp = (world, rank, *ranges[rank])
    else:
        pp = None
    stage = Stage(cfg.model, cfg.geom, W, precision=prec, pipeline=pp)
    stage.reset_stream(cfg.stream, prompts[0])
    dev = [torch.from_numpy(c).cuda() for c in chunks]
    outs = torch.zeros((NCALL,) + chunks[0].shape, device="cuda")

    def on_call(c):
        if c == 6:
            stage.set_prompt(prompts[1])

    if world > 1:
        tr = StageTransport(rank, world, stage_io_tensors(stage, stage.workspace), host_staging=True, device=0)
        idx = run_pipelined(stage, tr, lambda c: dev[c].data_ptr(), lambda c: outs[c].data_ptr(), NCALL,
                            on_call=on_call)
    else:
        idx = []
        for c in range(NCALL):
            on_call(c)
            idx.append(stage.denoise_chunk(dev[c].data_ptr(), outs[c].data_ptr()))
    torch.cuda.synchronize()
    res = {X: outs[c].cpu().numpy() for c, X in enumerate(idx) if X >= 0}
    stage.close()
    if world > 1:
        import torch.distributed as dist
        if rank == world - 1:
            q.put((idx, {k: v.tolist() for k, v in res.items()}))
        dist.barrier()
        dist.destroy_process_group()
    return idx, res


def _worker(rank, world, port, q, prec, kind):
    _run(prec, rank, world, q, port, kind)


@pytest.mark.gpu
@pytest.mark.parametrize("prec,kind", [(0, "tiny"), (1, "tiny"), (1, "wan13")])
def test_two_stage_pipeline_bitwise(prec, kind):
    import torch.multiprocessing as mp
    from paper_2511_07399_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, prec, kind)) for r in range(2)]
    for p in ps:
        p.start()
    idx, got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_idx, ref = _run(prec, 0, 1, kind=kind)
    n = _inputs(kind)[0].geom.steps
    assert idx == [-1] * ((n - 1) * 2) + list(range(NCALL - (n - 1) * 2))
    assert set(got) and set(got) <= set(ref)
    for X, v in got.items():
        assert np.array_equal(np.array(v, dtype=np.float32), ref[X]), X
