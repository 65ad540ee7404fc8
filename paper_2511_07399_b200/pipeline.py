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
        self.base = 0                   # stage calls made before the current run (buffer parity)
        # ring-closure packets whose consumer call (producer + K) lies beyond the run that
        # produced them: kept by the last rank, shipped to rank 0 when the run drains and
        # copied into ring_in before the consuming call of a later run (exact chaining of
        # runs, e.g. around an online re-partition).  global producer call -> tensor
        self.ring_stash = {}

    def _buf(self, t, role="recv"):
        """Tensor used on the wire (a host copy when staging through the host).  Sends and
        receives of the same device buffer get separate host copies: ranks > 0 send from
        the buffer they received into (the packet is computed in place)."""
        if not self.host or t.device.type == "cpu":
            return t
        key = (t.data_ptr(), t.numel(), role)
        if key not in self._stage:
            self._stage[key] = self.torch.empty(t.numel(), dtype=self.torch.uint8)
        return self._stage[key]

    def _ops(self, c: int, num_calls: int):
        """Ops posted after call c (c = -1: the initial receive before call 0)."""
        dist = self.dist
        K, r = self.world, self.rank
        ops, post = [], []
        if c >= 0:
            cur = self.io((self.base + c) & 1)
            if r < K - 1 and cur["act_out"].numel():
                src = cur["act_out"]
                wire = self._buf(src, "send")
                if wire is not src:
                    wire.copy_(src)
                ops.append(dist.P2POp(dist.isend, wire, r + 1))
            # ring packet of call c is consumed by rank 0 at call c + K
            if r == K - 1 and K > 1 and cur["ring_out"].numel():
                src = cur["ring_out"]
                if c + K < num_calls:
                    wire = self._buf(src, "send")
                    if wire is not src:
                        wire.copy_(src)
                    ops.append(dist.P2POp(dist.isend, wire, 0))
                else:       # consumer in a later run: keep a copy (the parity buffer is reused)
                    self.ring_stash[self.base + c] = src.clone()
        nxt = self.io((self.base + c + 1) & 1)
        if c + 1 >= num_calls:
            return ops, post
        if r > 0 and nxt["act_in"].numel():
            dst = nxt["act_in"]
            wire = self._buf(dst)
            ops.append(dist.P2POp(dist.irecv, wire, r - 1))
            if wire is not dst:
                post.append((dst, wire))
        g = self.base + c + 1                       # global index of the next call
        if r == 0 and K > 1 and g >= K and nxt["ring_in"].numel():
            dst = nxt["ring_in"]
            if g - K < self.base:                   # produced in an earlier run: stashed here
                dst.copy_(self.ring_stash.pop(g - K).to(dst.device))
            else:
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
        kinds = ["recv" if o.op is self.dist.irecv else "send" for o in ops]
        if len(works) != len(ops):       # one coalesced work for the whole group (NCCL)
            kinds = ["recv"] * len(works)
        self.pending.append((works, kinds, post))

    def wait(self):
        """Before the next call c+1: only its INPUTS must have arrived (the
        communication stream overlaps local computation).  The sends of call c read the
        parity-(c % 2) output buffers, which call c+2 overwrites, so they are waited for
        one call later (all works of older posts here)."""
        last = len(self.pending) - 1
        keep = []
        for i, (works, kinds, post) in enumerate(self.pending):
            sends = []
            for w, k in zip(works, kinds):
                if k == "recv" or i < last:
                    w.wait()
                else:
                    sends.append(w)
            for dst, wire in post:
                dst.copy_(wire, non_blocking=False)
            if sends:
                keep.append((sends, ["send"] * len(sends), []))
        self.pending = keep

    def drain(self, num_calls: int):
        """Wait for every outstanding transfer (end of a run of num_calls), then move the
        ring packets whose consumers lie in a later run from the last rank to rank 0."""
        for works, _, post in self.pending:
            for w in works:
                w.wait()
            for dst, wire in post:
                dst.copy_(wire, non_blocking=False)
        self.pending = []
        K, r, dist = self.world, self.rank, self.dist
        if K < 2 or r not in (0, K - 1):
            return
        ring_bytes = self.io(0)["ring_in" if r == 0 else "ring_out"].numel()
        if not ring_bytes:
            return
        end = self.base + num_calls
        producers = list(range(max(self.base, end - K), end))   # produced in this run, consumed later
        ops, post = [], []
        for p in producers:
            if r == K - 1:
                src = self.ring_stash.pop(p)
                wire = self._buf(src, "send")
                if wire is not src:
                    wire.copy_(src)
                ops.append(dist.P2POp(dist.isend, wire, 0))
            else:
                dev = self.io(0)["ring_in"].device
                buf = self.torch.empty(ring_bytes, dtype=self.torch.uint8, device=dev)
                wire = self._buf(buf) if self.host else buf
                ops.append(dist.P2POp(dist.irecv, wire, K - 1))
                post.append((p, buf, wire))
        if self.host and self.device is not None:
            self.torch.cuda.synchronize(self.device)
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for p, buf, wire in post:
            if wire is not buf:
                buf.copy_(wire)
            self.ring_stash[p] = buf


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


def run_pipelined(stage, transport: StageTransport, chunks, out_cb, num_calls: int, on_call=None, after_call=None):
    """Drive num_calls stage-ticks on this rank.  chunks(c) -> device/host pointer of the
    chunk admitted at call c (rank 0 only); out_cb(c) -> output pointer (last rank).
    on_call(c) runs before call c (its inputs already ordered on the stage stream, no
    transport op outstanding); after_call(c, out_chunk) right after it is enqueued.

    Every transfer of a run is matched inside the run, so the pipeline is drained when
    it returns (a barrier between runs is safe; a barrier inside one would deadlock:
    rank s waits for rank s-1's call c before its own call c).  Ring-closure packets
    whose consumer call lies beyond the run are stashed and delivered when the run
    drains, so consecutive runs continue the stream exactly (tests/test_pipeline_cpu.py)."""
    import contextlib
    transport.base = getattr(stage, "calls", 0)
    if num_calls < 1:
        return []
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
            if after_call:
                after_call(c, oc)
            transport.post(c, num_calls)
        transport.drain(num_calls)
    return outs


def migrate_blocks(stage, rank: int, world: int, old_bounds, new_bounds, host_staging: bool = False, device=None):
    """Online re-partition: move the KV lanes of every block whose owner changes
    from its old stage to its new one (one grouped send/recv batch; the control-plane
    metadata and the prompt K/V of resident blocks are already on every rank), then switch
    this rank's active block range.  Called between drained runs (run_pipelined), so no
    call of either rank is in flight."""
    import torch
    import torch.distributed as dist
    owner = lambda bounds, b: next(s for s in range(world) if bounds[s] <= b < bounds[s + 1])
    ws = stage.workspace
    base = ws.data_ptr()
    if device is not None:
        torch.cuda.synchronize(device)
    ops, post = [], []
    for b in range(old_bounds[0], old_bounds[-1]):
        o, n = owner(old_bounds, b), owner(new_bounds, b)
        if o == n or rank not in (o, n):
            continue
        for which in (0, 1):
            ptr, nbytes = stage.block_kv(b, which)
            t = ws[ptr - base:ptr - base + nbytes]
            wire = t.cpu() if host_staging else t
            if rank == o:
                ops.append(dist.P2POp(dist.isend, wire, n))
            else:
                ops.append(dist.P2POp(dist.irecv, wire, o))
                if wire is not t:
                    post.append((t, wire))
    for w in (dist.batch_isend_irecv(ops) if ops else []):
        w.wait()
    for t, wire in post:
        t.copy_(wire)
    stage.set_block_range(new_bounds[rank], new_bounds[rank + 1])


def balanced_ranges(num_blocks: int, world: int, block_ms: float, first_extra_ms: float, last_extra_ms: float):
    """Exact min-max partition of the blocks with the first / last stage
    extras (noise controller + embeddings / head) from measured times."""
    from .sdv2 import partition
    bounds, mx = partition([block_ms] * num_blocks, world, first_extra_ms, last_extra_ms)
    return [(bounds[i], bounds[i + 1]) for i in range(world)], mx


# ------------------------------------------------------------------------- bench
def _pp_backend(args):
    """NCCL over NVLink for the real multi-GPU run.  ``bench.py --pp-backend gloo`` moves the
    same packets through host staging, so the bench logic runs with several ranks on one GPU."""
    return getattr(args, "pp_backend", "nccl")


def _gather(dist, vals, backend):
    """all_gather of a small float vector (one row per rank)."""
    import torch
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().tolist() for o in out]


def _stage_weights(md, blocks, device):
    """Seeded weights of the global tensors + this stage's blocks, generated straight onto
    the GPU tensor by tensor for large models (no full fp32 host copy)."""
    import torch
    import synthgen as sg
    from concurrent.futures import ThreadPoolExecutor
    names = [n for n in sg.all_tensor_names(md)
             if not n.startswith("blocks.") or int(n.split(".")[1]) in set(blocks)]
    big = md.dim >= 4096

    def one(n):
        a = sg.gen_tensor(md, n, 0)
        return torch.from_numpy(a).to(device) if big else a

    with ThreadPoolExecutor(max_workers=8) as ex:
        return dict(zip(names, ex.map(one, names)))


def run_pipeline_bench(args, cfg):
    """bench.py --gpus N under torchrun: one rank per GPU, blocks split by the exact
    min-max partition of MEASURED per-block and stage-extra times, stage
    packets moved with NCCL send/recv over NVLink.  One continuous stream of calls:
      calibration (provisional uniform split, per-class event profile) -> re-partition
      -> fill (TTFF) -> warm-up -> timed (device-resident inputs; barrier + sync on both
      sides; max over ranks) -> e2e (pinned host chunk in on rank 0, host out on the last
      rank) -> per-kernel-class profile."""
    import torch
    import torch.distributed as dist
    import synthgen as sg
    from . import build as B
    from .sdv2 import SDV2_BF16, Stage, rebalance
    sys_path_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    if sys_path_root not in sys.path:
        sys.path.insert(0, sys_path_root)
    from bench import ClockSampler, METRIC, chunk_frames_px, measured_peaks
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = _pp_backend(args)
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev_index}"))
    else:
        dist.init_process_group("gloo")
    host_staging = backend != "nccl"
    if local == 0:
        B.build()
    dist.barrier()
    md, g, sd = cfg.model, cfg.geom, cfg.stream
    if world > md.num_blocks:
        raise SystemExit("more stages than DiT blocks")
    n, K = g.steps, world
    ls = sg.LatentStream(md.latent_channels, g.latent_h, g.latent_w, seed=1)
    R = 16
    host_chunks = [ls.chunk(X, g.chunk_frames) for X in range(R)]
    dev_chunks = [torch.from_numpy(c).to(f"cuda:{dev_index}") for c in host_chunks]
    out_dev = torch.empty(dev_chunks[0].shape, dtype=torch.float32, device=f"cuda:{dev_index}")
    prompt = sg.gen_prompt(md, 0)
    fill = n * K

    # resident blocks: the whole model for 1.3B (online re-partition anywhere), +-2 blocks
    # around the provisional range for 14B (weights generated per rank)
    margin = md.num_blocks if md.dim < 4096 else 2

    def make_stage(ranges):
        b0, b1 = ranges[rank]
        r0, r1 = max(0, b0 - margin), min(md.num_blocks, b1 + margin)
        W = _stage_weights(md, range(r0, r1), f"cuda:{dev_index}")
        st = Stage(md, g, W, precision=SDV2_BF16, pipeline=(world, rank, b0, b1, r0, r1), device=dev_index)
        del W
        torch.cuda.empty_cache()
        st.reset_stream(sd, prompt)
        tr = StageTransport(rank, world, stage_io_tensors(st, st.workspace), host_staging=host_staging,
                            device=dev_index)
        return st, tr

    def ptr_in(c):
        return dev_chunks[c % R].data_ptr()

    # ---- calibration on a provisional uniform split (balance by measured time)
    ranges0, _ = balanced_ranges(md.num_blocks, world, 1.0, 0.0, 0.0)
    stage, tr = make_stage(ranges0)
    run_pipelined(stage, tr, ptr_in, lambda c: out_dev.data_ptr(), fill)
    ncal = 6
    stage.profile_enable(True)
    base = stage.calls
    run_pipelined(stage, tr, lambda c: ptr_in(base + c), lambda c: out_dev.data_ptr(), ncal)
    blk_res = stage.profile_block_ms()                 # per resident block, 0 where not run here
    prof = stage.profile_read()
    stage.profile_enable(False)
    ext = prof["stage_extras"]["ms"] / ncal
    # Stream-VAE stand-in on the first / last stage ("the first and last ranks handle
    # VAE encoding and decoding in addition to DiT blocks"): its measured time joins the
    # stage extras the partition balances
    vae = None
    if getattr(args, "vae", False) and rank in (0, world - 1):
        from .sdv2 import StreamVAE
        vd = sg.VAE
        H8, W8 = 8 * g.latent_h, 8 * g.latent_w
        vae_w = sg.gen_vae_weights(vd)
        vae = StreamVAE(vd, H8, W8, vae_w, device=dev_index, stream=stage.stream)
        vae.reset()
        vae_vid = torch.from_numpy(np.ascontiguousarray(sg.gen_video(vd, 4, H8, W8))).to(f"cuda:{dev_index}")
        vae_lat = torch.empty(tuple(dev_chunks[0].shape), dtype=torch.float32, device=f"cuda:{dev_index}")
        vae_lat.zero_()
        vae_out = torch.empty((3, 4, H8, W8), dtype=torch.float32, device=f"cuda:{dev_index}")
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(4):
            if i == 1:
                a_.record(stage.stream)
            if rank == 0:
                vae.encode_chunk(vae_vid.data_ptr(), vae_lat.data_ptr())
            if rank == world - 1:
                vae.decode_chunk(vae_lat.data_ptr(), vae_out.data_ptr())
        b_.record(stage.stream)
        torch.cuda.synchronize(dev_index)
        ext += a_.elapsed_time(b_) / 3
    r0 = stage.resident[0]
    mine = [0.0] * md.num_blocks
    for i, v in enumerate(blk_res):
        mine[r0 + i] = v
    rows = _gather(dist, mine + [ext], backend)
    measured = [sum(r[b] for r in rows) for b in range(md.num_blocks)]   # each block timed on its owner
    first_extra, last_extra = rows[0][-1], rows[-1][-1]
    bounds0 = [ranges0[0][0]] + [r[1] for r in ranges0]
    ema = [0.0] * md.num_blocks
    bounds, changed, pred_cur, pred_new = rebalance(measured, world, bounds0, ema, first_extra, last_extra,
                                                    alpha=1.0, hysteresis=0.02)
    ranges = [(bounds[s], bounds[s + 1]) for s in range(world)]
    balance = {"block_ms": measured, "first_extra_ms": first_extra, "last_extra_ms": last_extra,
               "provisional": ranges0, "predicted_stage_ms": pred_new, "predicted_stage_ms_provisional": pred_cur,
               "moved_online": False}
    if changed:
        fits = all(stage_res[0] <= b0 and b1 <= stage_res[1] for stage_res, (b0, b1) in
                   zip(_gather(dist, list(stage.resident), backend), ranges))
        if fits:      # online: move the KV lanes of the moved blocks, no re-creation (N3)
            migrate_blocks(stage, rank, world, bounds0, bounds, host_staging=host_staging, device=dev_index)
            balance["moved_online"] = True
        else:
            stage.close()
            del stage, tr
            torch.cuda.empty_cache()
            stage, tr = make_stage(ranges)
    stage.reset_stream(sd, prompt)
    tr = StageTransport(rank, world, stage_io_tensors(stage, stage.workspace), host_staging=host_staging,
                        device=dev_index)
    stream = stage.stream
    if vae is not None and vae.stream is not stream:     # stage re-created: the VAE follows its stream
        vae.close()
        vae = StreamVAE(vd, H8, W8, vae_w, device=dev_index, stream=stream)
    if vae is not None:
        vae.reset()
    dist.barrier()

    # ---- phases, each a drained run bracketed by sync + barrier:
    #      fill (TTFF) + warm-up | timed (device-resident inputs) | e2e (pinned host in /
    #      out) | per-kernel-class profile
    pin_in = [torch.from_numpy(h).pin_memory() for h in host_chunks]
    pin_out = torch.empty(host_chunks[0].shape, dtype=torch.float32).pin_memory()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def sync_barrier():
        torch.cuda.synchronize(dev_index)
        dist.barrier()

    def dev_out(c):
        return out_dev.data_ptr()

    T = {"first_out": None}

    def first_out(c, oc):
        if oc >= 0 and T["first_out"] is None:
            T["first_out"] = ev()

    sync_barrier()
    t0 = ev()
    run_pipelined(stage, tr, ptr_in, dev_out, fill + args.warmup, after_call=first_out)
    sync_barrier()
    ttff = t0.elapsed_time(T["first_out"]) if T["first_out"] is not None else -1.0

    base = stage.calls
    step_ev = []
    clk = ClockSampler(dev_index)
    clk.start()
    l0 = stage.tick_info()["kernel_launches"]
    sync_barrier()
    ta = ev()
    def vae_in(c):           # rank 0: encode the chunk's 4 video frames into the latent it admits
        if vae is not None and rank == 0:
            vae.encode_chunk(vae_vid.data_ptr(), vae_lat.data_ptr())

    def vae_out_cb(c, oc):    # last rank: decode the emitted clean latent
        if vae is not None and rank == world - 1 and oc >= 0:
            vae.decode_chunk(out_dev.data_ptr(), vae_out.data_ptr())
        step_ev.append(ev())

    outs = run_pipelined(stage, tr, (lambda c: vae_lat.data_ptr()) if (vae is not None and rank == 0)
                         else (lambda c: ptr_in(base + c)), dev_out, args.steps,
                         on_call=vae_in, after_call=vae_out_cb)
    tb = ev()
    sync_barrier()
    clocks = clk.stop()
    launches = stage.tick_info()["kernel_launches"] - l0
    timed_ms = ta.elapsed_time(tb)
    step_ms = [a.elapsed_time(b) for a, b in zip([ta] + step_ev[:-1], step_ev)]
    outs_timed = sum(1 for oc in outs if oc >= 0)

    e2e_steps = max(8, min(args.steps, 64))
    base = stage.calls
    sync_barrier()
    ea = ev()
    outs_e = run_pipelined(stage, tr, lambda c: pin_in[(base + c) % R].data_ptr(), lambda c: pin_out.data_ptr(),
                           e2e_steps)
    eb = ev()
    sync_barrier()
    e2e_ms = ea.elapsed_time(eb)
    outs_e2e = sum(1 for oc in outs_e if oc >= 0)

    prof_steps = max(4, min(args.steps, 32))
    base = stage.calls
    stage.profile_enable(True)
    run_pipelined(stage, tr, lambda c: ptr_in(base + c), dev_out, prof_steps)
    torch.cuda.synchronize(dev_index)
    prof = stage.profile_read()
    stage.profile_enable(False)
    # ---- stage hand-off link rate (SURVEY §8(d) NVLink): ranks 0 -> 1 send the act packet
    # size back to back; device time on the sending stream, vs 900 GB/s per direction
    link = None
    act_bytes = int(tr.io(0)["act_out"].numel()) if world > 1 else 0
    if world > 1 and act_bytes and rank in (0, 1):
        dev = f"cuda:{dev_index}" if backend == "nccl" else "cpu"
        buf = torch.empty(act_bytes, dtype=torch.uint8, device=dev)
        reps = 20
        with torch.cuda.stream(stream):
            for i in range(reps + 3):
                if i == 3:
                    l0 = ev()
                if rank == 0:
                    dist.send(buf, 1)
                else:
                    dist.recv(buf, 0)
            l1 = ev()
        torch.cuda.synchronize(dev_index)
        ms_link = l0.elapsed_time(l1)
        link = [act_bytes * reps / (ms_link / 1e3) / 1e9 if ms_link > 0 else 0.0, float(act_bytes)]
    reasons = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    mine = [timed_ms, e2e_ms, ttff, float(outs_timed), float(outs_e2e), float(launches),
            float(clocks.get("sm_mhz") or 0.0), float(clocks.get("sm_max_mhz") or 0.0),
            prof["gemm"]["ms"], prof["gemm"]["flops"], prof["gemm"]["launches"],
            prof["self_attn"]["ms"], prof["self_attn"]["flops"], prof["cross_attn"]["ms"],
            prof["cross_attn"]["flops"]] + [1.0 if r in clocks.get("reasons", []) else 0.0 for r in reasons] + \
           (link if link else [0.0, 0.0])
    allr = _gather(dist, mine, backend)
    steps_all = _gather(dist, step_ms, backend)
    dist.barrier()
    if rank == 0:
        max_ms = max(r[0] for r in allr)
        max_e2e = max(r[1] for r in allr)
        last = allr[-1]
        px = chunk_frames_px(cfg)
        value = px * last[3] / (max_ms / 1e3)
        # rank s starts s ticks late (pipeline refill after the barrier): per-tick time
        # = max over ranks, aligned on the global tick, the refill ticks dropped
        tick = [max(col) for col in zip(*[r[K - 1 - i:len(r) - i] for i, r in enumerate(steps_all)])]
        lat = [sum(tick[i:i + n * K]) for i in range(0, len(tick) - n * K + 1)]
        peaks, src = measured_peaks()
        gm = max(r[8] for r in allr)          # slowest rank's GEMM class (kernels only)
        gr = max(range(world), key=lambda i: allr[i][8])
        g_ms, g_fl, g_n = allr[gr][8], allr[gr][9], allr[gr][10]
        achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
        peak = peaks["bf16_tflops_sustained"]
        res = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg.name, "latent": [md.latent_channels, g.chunk_frames, g.latent_h, g.latent_w],
                       "tokens_per_chunk": g.tokens_per_chunk(md), "steps_n": n, "sink_chunks": g.sink_chunks,
                       "window_chunks": g.window_chunks, "blocks": md.num_blocks, "dim": md.dim,
                       "parallelism": f"pp{world}", "transport": backend, "block_ranges": ranges,
                       "balance": balance, "px_frames_per_chunk": px,
                       "stream_vae": bool(getattr(args, "vae", False)),
                       "l2": "per-step working set >> L2 (stage weights + KV lanes streamed each step)"},
            "latent_chunks_per_s": last[3] / (max_ms / 1e3),
            "steady_state": {"tick_ms_median": float(np.median(tick)) if tick else None,
                             "frames_per_s": px * 1e3 / float(np.median(tick)) if tick else None,
                             "note": f"value includes the {K - 1}-tick refill after the opening barrier"},
            "ttff_ms": last[2],
            "ttff_with_buffering_ms": {"16fps": last[2] + 1e3 * px / 16.0, "30fps": last[2] + 1e3 * px / 30.0},
            "latency_ms": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                           "max": float(np.max(lat)), "definition": f"sum of {n * K} consecutive stage-ticks "
                           "(per-tick time = max over ranks)"} if lat else None,
            "e2e": {"value": px * last[4] / (max_e2e / 1e3), "unit": "frames/s",
                    "h2d_bytes_per_step": host_chunks[0].nbytes, "d2h_bytes_per_step": host_chunks[0].nbytes},
            "gpu_launches": int(sum(r[5] for r in allr)),
            "roofline": {"bound": "tensor", "kernel": "gemm", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": f"{src} bf16_tflops_sustained",
                         "per_launch_ms": g_ms / max(1, g_n), "flops_per_launch": g_fl / max(1, g_n),
                         "rank": gr, "note": "projection GEMMs of the slowest stage, per-launch CUDA events"},
            "cpu_baseline": None,
            "stage_handoff": {"bytes_per_tick": allr[0][20], "GBps_rank0_to_1": allr[0][19], "peak_GBps": 900.0,
                              "frac": allr[0][19] / 900.0, "transport": backend,
                              "note": "back-to-back send of one act packet, device time on the sending stream"}
            if world > 1 else None,
            "clocks": {"sm_mhz": statistics.median([r[6] for r in allr]), "sm_max_mhz": max(r[7] for r in allr),
                       "reasons": [reasons[i] for i in range(4) if any(r[15 + i] for r in allr)],
                       "per_rank_sm_mhz": [r[6] for r in allr]},
        }
        del gm
        print(json.dumps(res))
    if vae is not None:
        vae.close()
    stage.close()
    dist.barrier()
    dist.destroy_process_group()
