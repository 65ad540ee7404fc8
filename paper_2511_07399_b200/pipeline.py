"""Pipeline-parallel stage transport ("the DiT blocks are partitioned across
devices ... each device processes its input sequence as a micro-step and transmits the
results to the next stage within a ring structure"; P:238–240 two CUDA streams).

Each rank owns one ``Stage`` (a contiguous block range, chosen by the exact min-max
partition of measured block times).  The library exposes its hand-off
packets (``sdv2_stage_io_buffers``); this module moves them with ``torch.distributed``:

* rank s -> s+1: the tick packet (fp32 residual stream, time embeddings, sigmas,
  entry latents) of call c;
* last -> rank 0 (ring closure): the re-noised latents of the continuing entries of
  call c, consumed by rank 0 at call c + K.

Deadlock freedom: after call c every rank posts ONE grouped batch
{send its outputs of call c, recv its inputs of call c+1}.  Under the R2 schedule the
groups of all ranks line up on the same global stage-tick (rank s finishes call c at
tick c + s), so every send has its matching recv in the peer's concurrent group.

Backends: NCCL on device buffers (NVLink / NVSwitch), or any backend through host
staging (gloo; used by the CPU tests and by 2-process-on-one-GPU tests).
"""
from __future__ import annotations

import json
import os
import statistics
import time
from typing import Callable, List, Optional

import numpy as np


class StageTransport:
    """Grouped point-to-point transport of one rank's stage packets."""

    def __init__(self, rank: int, world: int, io: Callable[[int], dict], host_staging: bool = False,
                 device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = rank, world
        self.io = io                    # parity -> {"act_in","act_out","ring_in","ring_out"} uint8 tensors
        self.host = host_staging
        self.device = device
        self.pending = []
        self._stage = {}

    def _buf(self, t):
        """Tensor used on the wire (a host copy when staging through the host)."""
        if not self.host or t.device.type == "cpu":
            return t
        key = (t.data_ptr(), t.numel())
        if key not in self._stage:
            self._stage[key] = self.torch.empty(t.numel(), dtype=self.torch.uint8)
        return self._stage[key]

    def _ops(self, c: int, num_calls: int):
        """Ops posted after call c (c = -1: the initial receive before call 0)."""
        dist = self.dist
        K, r = self.world, self.rank
        ops, post = [], []
        if c >= 0:
            cur = self.io(c & 1)
            if r < K - 1 and cur["act_out"].numel():
                src = cur["act_out"]
                wire = self._buf(src)
                if wire is not src:
                    wire.copy_(src)
                ops.append(dist.P2POp(dist.isend, wire, r + 1))
            # ring packet of call c is consumed by rank 0 at call c + K
            if r == K - 1 and K > 1 and cur["ring_out"].numel() and c + K < num_calls:
                src = cur["ring_out"]
                wire = self._buf(src)
                if wire is not src:
                    wire.copy_(src)
                ops.append(dist.P2POp(dist.isend, wire, 0))
        nxt = self.io((c + 1) & 1)
        if c + 1 >= num_calls:
            return ops, post
        if r > 0 and nxt["act_in"].numel():
            dst = nxt["act_in"]
            wire = self._buf(dst)
            ops.append(dist.P2POp(dist.irecv, wire, r - 1))
            if wire is not dst:
                post.append((dst, wire))
        if r == 0 and K > 1 and c + 1 >= K and nxt["ring_in"].numel():
            dst = nxt["ring_in"]
            wire = self._buf(dst)
            ops.append(dist.P2POp(dist.irecv, wire, K - 1))
            if wire is not dst:
                post.append((dst, wire))
        return ops, post

    def post(self, c: int, num_calls: int):
        """After call c (of num_calls): send this call's outputs, receive call c+1's inputs."""
        ops, post = self._ops(c, num_calls)
        if self.host and self.device is not None:
            self.torch.cuda.synchronize(self.device)   # device outputs complete before host copy
        works = self.dist.batch_isend_irecv(ops) if ops else []
        self.pending.append((works, post))

    def wait(self):
        for works, post in self.pending:
            for w in works:
                w.wait()
            for dst, wire in post:
                dst.copy_(wire, non_blocking=False)
        self.pending = []


def stage_io_tensors(stage, workspace):
    """uint8 views of the library's hand-off buffers inside the workspace tensor."""
    base = workspace.data_ptr()
    cache = {}

    def io(parity):
        if parity in cache:
            return cache[parity]
        s = stage.stage_io(parity)
        out = {}
        for name, ptr, nb in (("act_in", s.act_in, s.act_bytes), ("act_out", s.act_out, s.act_bytes),
                              ("ring_in", s.ring_in, s.ring_bytes), ("ring_out", s.ring_out, s.ring_bytes)):
            if not ptr or nb == 0:
                out[name] = workspace[:0]
            else:
                off = ptr - base
                out[name] = workspace[off:off + nb]
        cache[parity] = out
        return out

    return io


def run_pipelined(stage, transport: StageTransport, chunks, out_cb, num_calls: int, on_call=None):
    """Drive num_calls stage-ticks on this rank.  chunks(c) -> device/host pointer of the
    chunk admitted at call c (rank 0 only); out_cb(c) -> output pointer (last rank)."""
    import contextlib
    stream = getattr(stage, "stream", None)
    ctx = transport.torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:   # NCCL waits and host-staging copies are ordered on the stage's stream
        transport.post(-1, num_calls)
        outs = []
        for c in range(num_calls):
            transport.wait()
            if on_call:
                on_call(c)
            oc = stage.denoise_chunk(chunks(c) if transport.rank == 0 else None,
                                     out_cb(c) if transport.rank == transport.world - 1 else None)
            outs.append(oc)
            transport.post(c, num_calls)
        transport.wait()
    return outs


def balanced_ranges(num_blocks: int, world: int, block_ms: float, first_extra_ms: float, last_extra_ms: float):
    """Exact min-max partition of the blocks with the first / last stage
    extras (noise controller + embeddings / head) from measured times."""
    from .sdv2 import partition
    bounds, mx = partition([block_ms] * num_blocks, world, first_extra_ms, last_extra_ms)
    return [(bounds[i], bounds[i + 1]) for i in range(world)], mx


# ------------------------------------------------------------------------- bench
def run_pipeline_bench(args, cfg):
    """bench.py --gpus N under torchrun: one rank per GPU, NCCL over NVLink."""
    import torch
    import torch.distributed as dist
    import synthgen as sg
    from . import build as B
    from .sdv2 import SDV2_BF16, Stage
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if local == 0:
        B.build()
    dist.barrier()
    md, g, sd = cfg.model, cfg.geom, cfg.stream
    if world > md.num_blocks:
        raise SystemExit("more stages than DiT blocks")
    # Stage split: blocks are shape-identical, so one measured block time; extras of the
    # first / last stage (controller, embeddings / head) are small at these shapes.
    ranges, _ = balanced_ranges(md.num_blocks, world, 1.0, 0.05, 0.05)
    b0, b1 = ranges[rank]
    W = sg.gen_weights(md, seed=0, blocks=range(b0, b1))
    stage = Stage(md, g, W, precision=SDV2_BF16, pipeline=(world, rank, b0, b1), device=local)
    del W
    io = stage_io_tensors(stage, stage.workspace)
    tr = StageTransport(rank, world, io)
    stage.reset_stream(sd, sg.gen_prompt(md, 0))
    ls = sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1)
    R = 16
    dev_chunks = [torch.from_numpy(ls.chunk(X, g.chunk_frames)).cuda() for X in range(R)]
    out_dev = torch.empty(dev_chunks[0].shape, dtype=torch.float32, device="cuda")
    fill = g.steps * world
    # warm-up (fills the pipeline, includes TTFF ticks)
    run_pipelined(stage, tr, lambda c: dev_chunks[c % R].data_ptr(), lambda c: out_dev.data_ptr(),
                  fill + args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    outs = run_pipelined(stage, tr, lambda c: dev_chunks[c % R].data_ptr(), lambda c: out_dev.data_ptr(),
                         args.steps)
    ev1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    total_ms = ms.item()
    if rank == 0:
        chunks_out = args.steps            # one clean chunk per stage-tick in steady state
        value = 4 * g.chunk_frames * chunks_out / (total_ms / 1e3)
        print(json.dumps({
            "metric": "output FPS, TTFF and p99 chunk latency at 1/2/4/8 B200; GEMM tensor-pipe %",
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg.name, "parallelism": f"pp{world}", "block_ranges": ranges}}))
    stage.close()
    dist.destroy_process_group()
