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
    if kind == "tiny4":
        cfg = dataclasses.replace(cfg, model=dataclasses.replace(cfg.model, num_blocks=4))
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


def _rebalance_worker(rank, world, port, q, prec):
    """4-block tiny model on 2 stages, every block resident on both ranks: run 5 calls on
    the split [0,1) | [1,4), measure block times, move the boundary to [0,3) | [3,4) (the
    policy is forced by a made-up profile; the move is what is tested), run 7 more calls."""
    import dataclasses
    import torch
    import torch.distributed as dist
    from paper_2511_07399_b200.pipeline import StageTransport, migrate_blocks, run_pipelined, stage_io_tensors
    from paper_2511_07399_b200.sdv2 import Stage, rebalance
    torch.cuda.set_device(0)
    cfg, W, chunks, prompts = _inputs("tiny4")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nb = cfg.model.num_blocks
    bounds = [0, 1, nb]
    stage = Stage(cfg.model, cfg.geom, W, precision=prec, pipeline=(world, rank, bounds[rank], bounds[rank + 1], 0, nb))
    stage.reset_stream(cfg.stream, prompts[0])
    dev = [torch.from_numpy(c).cuda() for c in chunks]
    outs = torch.zeros((NCALL,) + chunks[0].shape, device="cuda")

    def on_call(c):
        if c == 6:
            stage.set_prompt(prompts[1])

    tr = StageTransport(rank, world, stage_io_tensors(stage, stage.workspace), host_staging=True, device=0)
    idx = []
    stage.profile_enable(True)
    idx += run_pipelined(stage, tr, lambda c: dev[c].data_ptr(), lambda c: outs[c].data_ptr(), 5, on_call=on_call)
    ms = stage.profile_block_ms()
    stage.profile_enable(False)
    assert all((m > 0) == (bounds[rank] <= b < bounds[rank + 1]) for b, m in enumerate(ms)), ms
    ema = [0.0] * nb
    new, changed, _, _ = rebalance([1.0, 0.2, 0.2, 3.0], world, bounds, ema, alpha=1.0)
    assert changed and new == [0, 3, 4]
    migrate_blocks(stage, rank, world, bounds, new, host_staging=True, device=0)
    off = 5
    idx += run_pipelined(stage, tr, lambda c: dev[c + off].data_ptr(), lambda c: outs[c + off].data_ptr(),
                         NCALL - off, on_call=lambda c: on_call(c + off))
    torch.cuda.synchronize()
    res = {X: outs[c].cpu().numpy() for c, X in enumerate(idx) if X >= 0}
    stage.close()
    if rank == world - 1:
        q.put((idx, {k: v.tolist() for k, v in res.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [0, 1])
def test_online_rebalance_kv_migration_bitwise(prec):
    """N3: blocks move between stages mid-stream with their KV lanes; the
    stream continues exactly: outputs equal a single-stage run bit for bit (tiny model with
    4 blocks, n = 2, prompt switch after the move, re-bases and evictions before and after)."""
    import torch.multiprocessing as mp
    from paper_2511_07399_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rebalance_worker, args=(r, 2, port, q, prec)) for r in range(2)]
    for p in ps:
        p.start()
    idx, got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_idx, ref = _run(prec, 0, 1, kind="tiny4")
    n = _inputs("tiny4")[0].geom.steps
    assert idx == [-1] * ((n - 1) * 2) + list(range(NCALL - (n - 1) * 2))
    assert set(got) and set(got) <= set(ref)
    for X, v in got.items():
        assert np.array_equal(np.array(v, dtype=np.float32), ref[X]), X
