"""Pipeline transport on CPU with gloo, world_size 2 and 3 (no GPU): grouped send/recv
per tick + ring closure + the library's R2 schedule reproduce the single-stage result
bit for bit (pin P6 on the host side)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_07399_b200 import build
from paper_2511_07399_b200.pipeline import StageTransport, run_pipelined, stage_io_tensors, balanced_ranges

from toy_stage import ToyStage

NBLK, NCALL = 6, 24


def _chunk(X):
    return np.sin(np.arange(6) * 0.3 + X)


def _reference(n):
    st = ToyStage(n, 1, 0, 0, NBLK)
    out = {}
    for c in range(NCALL):
        st.denoise_chunk(_chunk, out)
    return out


def _worker(rank, world, n, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges, _ = balanced_ranges(NBLK, world, 1.0, 0.0, 0.0)
    b0, b1 = ranges[rank]
    st = ToyStage(n, world, rank, b0, b1)
    io = stage_io_tensors(st, st.workspace)
    tr = StageTransport(rank, world, io)
    out = {}
    outs = run_pipelined(st, tr, lambda c: _chunk, lambda c: out, NCALL)
    if rank == world - 1:
        q.put((outs, {k: v.tolist() for k, v in out.items()}))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n", [(2, 1), (2, 4), (3, 2)])
def test_gloo_pipeline_equals_single_stage(world, n):
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, n, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs, got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _reference(n)
    # one clean chunk per call once the pipeline is full (first at call (n-1) K)
    assert outs[:(n - 1) * world] == [-1] * ((n - 1) * world)
    assert outs[(n - 1) * world:] == list(range(NCALL - (n - 1) * world))
    for X, v in got.items():
        assert np.array_equal(np.array(v), ref[X]), X
    assert len(got) == NCALL - (n - 1) * world


def _worker_split(rank, world, n, port, q, runs):
    """The bench's phase structure: several drained runs with a barrier between them."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges, _ = balanced_ranges(NBLK, world, 1.0, 0.0, 0.0)
    b0, b1 = ranges[rank]
    st = ToyStage(n, world, rank, b0, b1)
    tr = StageTransport(rank, world, stage_io_tensors(st, st.workspace))
    out, outs = {}, []
    for r in runs:
        outs += run_pipelined(st, tr, lambda c: _chunk, lambda c: out, r)
        dist.barrier()
    if rank == world - 1:
        q.put((outs, {k: v.tolist() for k, v in out.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1), (3, 1), (2, 4), (3, 2), (4, 3)])
def test_gloo_pipeline_split_runs(world, n):
    """Runs of odd lengths separated by barriers (bench phases, an online re-partition)
    neither deadlock nor mis-pair the parity-double-buffered packets, and the stream
    continues exactly: ring-closure packets whose consumer lies in the next run are
    stashed and delivered at the drain, so the output equals the single-stage stream bit
    for bit for every n (runs shorter than K included)."""
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    runs = [5, 2, 7, NCALL - 14]
    ps = [ctx.Process(target=_worker_split, args=(r, world, n, port, q, runs)) for r in range(world)]
    for p in ps:
        p.start()
    outs, got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[(n - 1) * world:] == list(range(NCALL - (n - 1) * world))
    ref = _reference(n)
    for X, v in got.items():
        assert np.array_equal(np.array(v), ref[X]), X
    assert len(got) == NCALL - (n - 1) * world
