"""Thin ctypes binding of libsdv2.so (include/sdv2.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  PyTorch provides the
device workspace and the CUDA stream.  There is no CPU fallback: importing the
binding without the built library raises."""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsdv2.so")
CTL_LIB_PATH = os.path.join(HERE, "libsdv2_ctl.so")

SDV2_FP32, SDV2_BF16 = 0, 1
STATUS = {0: "ok", -1: "invalid argument", -2: "invalid shape", -3: "invalid state",
          -4: "workspace too small", -5: "cuda error", -6: "unsupported shape"}

GLOBAL_ORDER = ("patch_w", "patch_b", "txt1_w", "txt1_b", "txt2_w", "txt2_b", "t1_w", "t1_b", "t2_w", "t2_b",
                "tp_w", "tp_b", "head_mod", "head_w", "head_b")
BLOCK_ORDER = ("mod", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "gq", "gk", "n3_g", "n3_b", "wcq", "bcq",
               "wck", "bck", "wcv", "bcv", "wco", "bco", "gcq", "gck", "w1", "b1", "w2", "b2")


class ModelDescC(ctypes.Structure):
    _fields_ = [("num_blocks", ctypes.c_int32), ("dim", ctypes.c_int32), ("num_heads", ctypes.c_int32),
                ("ffn_dim", ctypes.c_int32), ("latent_channels", ctypes.c_int32), ("patch_t", ctypes.c_int32),
                ("patch_h", ctypes.c_int32), ("patch_w", ctypes.c_int32), ("text_len", ctypes.c_int32),
                ("text_dim", ctypes.c_int32), ("freq_dim", ctypes.c_int32), ("eps", ctypes.c_float),
                ("norm_center", ctypes.c_int32)]


class GeometryC(ctypes.Structure):
    _fields_ = [("latent_h", ctypes.c_int32), ("latent_w", ctypes.c_int32), ("chunk_frames", ctypes.c_int32),
                ("steps", ctypes.c_int32), ("sink_chunks", ctypes.c_int32), ("window_chunks", ctypes.c_int32),
                ("streams", ctypes.c_int32), ("kv_mode", ctypes.c_int32)]


class PipelineC(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("block_begin", ctypes.c_int32),
                ("block_end", ctypes.c_int32), ("resident_begin", ctypes.c_int32), ("resident_end", ctypes.c_int32)]


class WeightsC(ctypes.Structure):
    _fields_ = [("tensors", ctypes.POINTER(ctypes.c_void_p)), ("count", ctypes.c_int32)]


class StreamDescC(ctypes.Structure):
    _fields_ = [("timesteps", ctypes.POINTER(ctypes.c_float)), ("num_timesteps", ctypes.c_int32),
                ("rope_reset_frames", ctypes.c_int32), ("motion_k", ctypes.c_int32),
                ("motion_sigma", ctypes.c_float), ("s_min", ctypes.c_float), ("s_max", ctypes.c_float),
                ("ema_lambda", ctypes.c_float), ("sink_tau", ctypes.c_float), ("seed", ctypes.c_uint64)]


class ExecOptionsC(ctypes.Structure):
    _fields_ = [("tune_gemms", ctypes.c_int32), ("pdl", ctypes.c_int32), ("graphs", ctypes.c_int32),
                ("l2_persist", ctypes.c_int32), ("gemm_table", ctypes.POINTER(ctypes.c_int32)),
                ("gemm_table_len", ctypes.c_int32)]


class StageIOC(ctypes.Structure):
    _fields_ = [("act_in", ctypes.c_void_p), ("act_out", ctypes.c_void_p), ("act_bytes", ctypes.c_size_t),
                ("ring_in", ctypes.c_void_p), ("ring_out", ctypes.c_void_p), ("ring_bytes", ctypes.c_size_t)]


class TickInfoC(ctypes.Structure):
    _fields_ = [("call", ctypes.c_int64), ("num_entries", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("chunk", ctypes.c_int64 * 8), ("out_chunk", ctypes.c_int64), ("kernel_launches", ctypes.c_int64)]


class ProfileC(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 6), ("ms", ctypes.c_double * 6), ("flops", ctypes.c_double * 6)]


class CacheStateC(ctypes.Structure):
    _fields_ = [("num_slots", ctypes.c_int32), ("num_valid", ctypes.c_int32), ("tag", ctypes.c_int64 * 64),
                ("pos", ctypes.c_int32 * 64), ("resets", ctypes.c_int32), ("evictions", ctypes.c_int64),
                ("noise_rate", ctypes.c_double), ("d_hat", ctypes.c_double)]


_EXPORTS = ["sdv2_workspace_bytes", "sdv2_create", "sdv2_reset_stream", "sdv2_set_prompt", "sdv2_denoise_chunk",
            "sdv2_stage_io_buffers", "sdv2_get_tick_info", "sdv2_destroy", "sdv2_status_string",
            "sdv2_last_error", "sdv2_get_cache_state", "sdv2_set_block_tap", "sdv2_kv_lane", "sdv2_partition"]


def _declare(lib):
    P = ctypes.c_void_p
    lib.sdv2_workspace_bytes.restype = ctypes.c_size_t
    lib.sdv2_workspace_bytes.argtypes = [ctypes.POINTER(ModelDescC), ctypes.POINTER(GeometryC),
                                         ctypes.POINTER(PipelineC), ctypes.c_int]
    lib.sdv2_create.argtypes = [ctypes.POINTER(ModelDescC), ctypes.POINTER(GeometryC), ctypes.POINTER(PipelineC),
                                ctypes.c_int, ctypes.POINTER(WeightsC), P, ctypes.c_size_t, ctypes.c_int, P,
                                ctypes.POINTER(ExecOptionsC), ctypes.POINTER(P)]
    lib.sdv2_reset_stream.argtypes = [P, ctypes.POINTER(StreamDescC), P]
    lib.sdv2_set_prompt.argtypes = [P, ctypes.c_int32, P]
    lib.sdv2_denoise_chunk.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_int64)]
    lib.sdv2_stage_io_buffers.argtypes = [P, ctypes.c_int32, ctypes.POINTER(StageIOC)]
    lib.sdv2_get_tick_info.argtypes = [P, ctypes.POINTER(TickInfoC)]
    lib.sdv2_destroy.argtypes = [P]
    lib.sdv2_gemm_configs.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    lib.sdv2_status_string.restype = ctypes.c_char_p
    lib.sdv2_status_string.argtypes = [ctypes.c_int]
    lib.sdv2_last_error.restype = ctypes.c_char_p
    lib.sdv2_last_error.argtypes = [P]
    lib.sdv2_get_cache_state.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(CacheStateC)]
    lib.sdv2_set_block_tap.argtypes = [P, P]
    lib.sdv2_kv_lane.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(P),
                                 ctypes.POINTER(ctypes.c_size_t)]
    lib.sdv2_partition.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_double)]
    lib.sdv2_profile_enable.argtypes = [P, ctypes.c_int32]
    lib.sdv2_set_graphs.argtypes = [P, ctypes.c_int32]
    lib.sdv2_set_graphs.restype = ctypes.c_int
    lib.sdv2_profile_read.argtypes = [P, ctypes.POINTER(ProfileC)]
    lib.sdv2_set_block_range.argtypes = [P, ctypes.c_int32, ctypes.c_int32]
    lib.sdv2_set_block_range.restype = ctypes.c_int
    lib.sdv2_block_kv.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t)]
    lib.sdv2_block_kv.restype = ctypes.c_int
    lib.sdv2_profile_block_ms.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.c_int32]
    lib.sdv2_profile_block_ms.restype = ctypes.c_int
    for f in ("sdv2_profile_enable", "sdv2_profile_read", "sdv2_create", "sdv2_reset_stream", "sdv2_set_prompt", "sdv2_denoise_chunk", "sdv2_stage_io_buffers",
              "sdv2_get_tick_info", "sdv2_destroy", "sdv2_get_cache_state", "sdv2_set_block_tap", "sdv2_kv_lane",
              "sdv2_partition"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


_LIB = None
_LIB_PATH = LIB_PATH


def load_library(path: str):
    """Use another build of the same library (A/B timing tools); must precede the first lib()."""
    global _LIB_PATH
    if _LIB is not None and path != _LIB_PATH:
        raise RuntimeError("libsdv2 already loaded from " + _LIB_PATH)
    _LIB_PATH = path


def lib():
    """Load libsdv2.so (raises if it has not been built: no fallback exists)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} is missing: run `python -m paper_2511_07399_b200.build` "
                               "(the hot path has no CPU fallback)")
        _LIB = _declare(ctypes.CDLL(_LIB_PATH))
    return _LIB


class SDV2Error(RuntimeError):
    pass


def _check(st, h=None):
    if st != 0:
        msg = STATUS.get(st, str(st))
        if h is not None:
            msg += ": " + lib().sdv2_last_error(h).decode()
        raise SDV2Error(msg)


def model_desc_c(md) -> ModelDescC:
    return ModelDescC(md.num_blocks, md.dim, md.num_heads, md.ffn_dim, md.latent_channels, md.patch_t, md.patch_h,
                      md.patch_w, md.text_len, md.text_dim, md.freq_dim, md.eps, md.norm_center)


def geometry_c(g) -> GeometryC:
    return GeometryC(g.latent_h, g.latent_w, g.chunk_frames, g.steps, g.sink_chunks, g.window_chunks,
                     getattr(g, "streams", 1), getattr(g, "kv_mode", 0))


def partition(costs: Sequence[float], stages: int, extra_first=0.0, extra_last=0.0):
    """Exact min-max contiguous block partition; returns (bounds, max_stage)."""
    L = lib() if os.path.exists(LIB_PATH) else ctl_lib()
    c = (ctypes.c_double * len(costs))(*costs)
    b = (ctypes.c_int32 * (stages + 1))()
    mx = ctypes.c_double()
    _check(L.sdv2_partition(c, len(costs), stages, extra_first, extra_last, b, ctypes.byref(mx)))
    return list(b), mx.value


_CTL = None


def ctl_lib():
    """Host control plane alone (no CUDA needed): libsdv2_ctl.so."""
    global _CTL
    if _CTL is None:
        if not os.path.exists(CTL_LIB_PATH):
            raise RuntimeError(f"{CTL_LIB_PATH} is missing: run `python -m paper_2511_07399_b200.build`")
        L = ctypes.CDLL(CTL_LIB_PATH)
        L.sdv2ctl_new.restype = ctypes.c_void_p
        L.sdv2ctl_new.argtypes = [ctypes.c_int32] * 7 + [ctypes.c_double, ctypes.c_int32]
        L.sdv2ctl_free.argtypes = [ctypes.c_void_p]
        L.sdv2ctl_set_prompt_mean.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                              ctypes.c_int32, ctypes.c_int32]
        L.sdv2ctl_call.restype = ctypes.c_int32
        L.sdv2ctl_call.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]
        L.sdv2ctl_lane_state.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(CacheStateC)]
        L.sdv2ctl_max_frames.restype = ctypes.c_int32
        L.sdv2_partition.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_double)]
        L.sdv2_partition.restype = ctypes.c_int
        _CTL = L
    return _CTL


class HostControl:
    """The library's host control plane driven without a GPU (tests)."""

    def __init__(self, T, m, W, n, K=1, rank=0, T_reset=4, tau=0.95, B=1):
        self.L = ctl_lib()
        self.n, self.B = n, B
        self.h = self.L.sdv2ctl_new(T, m, W, n, K, rank, T_reset, tau, B)
        if not self.h:
            raise SDV2Error("invalid control parameters")
        self.F = self.L.sdv2ctl_max_frames()

    def set_prompt_mean(self, h, pver, stream=0):
        a = np.ascontiguousarray(h, dtype=np.float64)
        st = self.L.sdv2ctl_set_prompt_mean(self.h, stream, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            a.size, pver)
        if st != 0:
            raise SDV2Error("stream out of range")

    def call(self):
        """One call; entries e = j B + b."""
        w = 10 + self.F
        out = (ctypes.c_int32 * (self.n * self.B * w))()
        oc = ctypes.c_int64()
        na = self.L.sdv2ctl_call(self.h, out, ctypes.byref(oc))
        ents = []
        for i in range(self.n * self.B):
            o = out[i * w:(i + 1) * w]
            ents.append({"X": o[0], "j": o[1], "active": o[2], "write_slot": o[3], "nvalid": o[4],
                         "refresh_mask": o[5], "rebase": o[6], "pver": o[7], "stream": o[8], "xslot": o[9],
                         "pos": list(o[10:])})
        return na, ents, oc.value

    def lane_state(self, lane):
        st = CacheStateC()
        self.L.sdv2ctl_lane_state(self.h, lane, ctypes.byref(st))
        return st

    def __del__(self):
        try:
            self.L.sdv2ctl_free(self.h)
        except Exception:
            pass


class Stage:
    """One pipeline stage (or the whole model when pipeline=None) of the hot path."""

    def __init__(self, md, geom, weights: Dict[str, np.ndarray], precision=SDV2_BF16, pipeline=None,
                 device=0, stream=None, tune_gemms=True, pdl=True, graphs=True, l2_persist=True,
                 gemm_table=None):
        import torch
        self.torch = torch
        self.md, self.geom = md, geom
        self.precision = precision
        self.L = lib()
        self._mdc = model_desc_c(md)
        self._gc = geometry_c(geom)
        if pipeline is None:
            self._pp = None
            b0, b1 = 0, md.num_blocks
            r0, r1 = b0, b1
        else:
            # (world, rank, block_begin, block_end[, resident_begin, resident_end])
            pl = tuple(pipeline) + ((0, 0) if len(pipeline) == 4 else ())
            self._pp = PipelineC(*pl)
            b0, b1 = pl[2], pl[3]
            r0, r1 = (pl[4], pl[5]) if pl[4:6] != (0, 0) else (b0, b1)
        self.block_range = (b0, b1)
        self.resident = (r0, r1)
        ppp = ctypes.byref(self._pp) if self._pp is not None else None
        nbytes = self.L.sdv2_workspace_bytes(ctypes.byref(self._mdc), ctypes.byref(self._gc), ppp, precision)
        if nbytes == 0:
            raise SDV2Error("invalid model / geometry descriptor")
        self.device = device
        self.workspace = torch.empty(nbytes + 1024, dtype=torch.uint8, device=f"cuda:{device}")
        # a dedicated (capturable) stream: per-call device work is replayed from CUDA graphs
        self.stream = stream if stream is not None else torch.cuda.Stream(device)
        names = list(GLOBAL_ORDER) + [f"blocks.{b}.{t}" for b in range(r0, r1) for t in BLOCK_ORDER]
        keep = []
        ptrs = (ctypes.c_void_p * len(names))()
        for i, nme in enumerate(names):
            a = weights[nme]
            if isinstance(a, np.ndarray):
                a = np.ascontiguousarray(a, dtype=np.float32)
                ptrs[i] = a.ctypes.data
            else:   # torch tensor (host or device), fp32 contiguous
                a = a.contiguous().float()
                ptrs[i] = a.data_ptr()
            keep.append(a)
        w = WeightsC(ptrs, len(names))
        h = ctypes.c_void_p()
        recs = [int(v) for r in (gemm_table or []) for v in r]
        self._gemm_table = (ctypes.c_int32 * max(len(recs), 1))(*recs)
        self._opts = ExecOptionsC(int(tune_gemms), int(pdl), int(graphs), int(l2_persist),
                                  ctypes.cast(self._gemm_table, ctypes.POINTER(ctypes.c_int32)), len(recs) // 8)
        st = self.L.sdv2_create(ctypes.byref(self._mdc), ctypes.byref(self._gc), ppp, precision, ctypes.byref(w),
                                ctypes.c_void_p(self.workspace.data_ptr()), nbytes + 1024, device,
                                ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(self._opts), ctypes.byref(h))
        if st != 0:
            if h.value:
                msg = self.L.sdv2_last_error(h).decode()
                self.L.sdv2_destroy(h)
                raise SDV2Error(f"{STATUS.get(st, st)}: {msg}")
            raise SDV2Error(STATUS.get(st, str(st)))
        self.h = h
        del keep

    # ---------------------------------------------------------------- stream
    def reset_stream(self, sd, prompt):
        """prompt: one [text_len, text_dim] array per stream (a list), or a single array
        when the handle has one stream."""
        ts = (ctypes.c_float * len(sd.timesteps))(*sd.timesteps)
        self._ts = ts
        c = StreamDescC(ts, len(sd.timesteps), sd.rope_reset_frames, sd.motion_k, sd.motion_sigma, sd.s_min,
                        sd.s_max, sd.ema_lambda, sd.sink_tau, sd.seed)
        B = getattr(self.geom, "streams", 1)
        ps = list(prompt) if isinstance(prompt, (list, tuple)) else [prompt]
        if len(ps) != B:
            raise SDV2Error(f"{len(ps)} prompts for {B} streams")
        p = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float32) for x in ps]), dtype=np.float32)
        _check(self.L.sdv2_reset_stream(self.h, ctypes.byref(c), ctypes.c_void_p(p.ctypes.data)), self.h)
        self.calls = 0

    def set_prompt(self, prompt: np.ndarray, stream: int = 0):
        p = np.ascontiguousarray(prompt, dtype=np.float32)
        _check(self.L.sdv2_set_prompt(self.h, stream, ctypes.c_void_p(p.ctypes.data)), self.h)

    def set_chunk_embedding(self, emb, stream: int = 0):
        """Visual chunk embedding h_t for the next admitted chunk of `stream` (N4)."""
        a = np.ascontiguousarray(emb, dtype=np.float64)
        self.L.sdv2_set_chunk_embedding.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32]
        _check(self.L.sdv2_set_chunk_embedding(self.h, stream, ctypes.c_void_p(a.ctypes.data), a.size), self.h)

    def denoise_chunk(self, chunk_ptr: Optional[int], out_ptr: Optional[int]) -> int:
        """chunk_ptr / out_ptr: raw host or device addresses (or None).  Returns the chunk
        index emitted into out_ptr, or -1."""
        oc = ctypes.c_int64(-1)
        cur = self.torch.cuda.current_stream(self.device)
        if cur != self.stream:      # order after the caller's producers on its stream
            self.stream.wait_stream(cur)
        _check(self.L.sdv2_denoise_chunk(self.h, ctypes.c_void_p(chunk_ptr) if chunk_ptr else None,
                                         ctypes.c_void_p(out_ptr) if out_ptr else None, ctypes.byref(oc)), self.h)
        self.calls = getattr(self, "calls", 0) + 1
        return oc.value

    def tick_info(self):
        i = TickInfoC()
        _check(self.L.sdv2_get_tick_info(self.h, ctypes.byref(i)), self.h)
        return {"call": i.call, "num_entries": i.num_entries, "chunk": list(i.chunk)[:i.steps],
                "out_chunk": i.out_chunk, "kernel_launches": i.kernel_launches}

    def set_graphs(self, on: bool):
        _check(self.L.sdv2_set_graphs(self.h, 1 if on else 0), self.h)

    def profile_enable(self, on: bool):
        _check(self.L.sdv2_profile_enable(self.h, 1 if on else 0), self.h)

    def profile_read(self):
        p = ProfileC()
        _check(self.L.sdv2_profile_read(self.h, ctypes.byref(p)), self.h)
        names = ("gemm", "self_attn", "cross_attn", "other", "blocks", "stage_extras")
        return {names[i]: {"launches": p.launches[i], "ms": p.ms[i], "flops": p.flops[i]} for i in range(6)}

    def stage_io(self, parity: int):
        io = StageIOC()
        _check(self.L.sdv2_stage_io_buffers(self.h, parity, ctypes.byref(io)), self.h)
        return io

    def cache_state(self, local_block: int, lane: int):
        st = CacheStateC()
        _check(self.L.sdv2_get_cache_state(self.h, local_block, lane, ctypes.byref(st)), self.h)
        return st

    def set_block_tap(self, tensor):
        _check(self.L.sdv2_set_block_tap(self.h, ctypes.c_void_p(tensor.data_ptr()) if tensor is not None else None),
               self.h)

    def set_block_range(self, b0, b1):
        _check(self.L.sdv2_set_block_range(self.h, b0, b1), self.h)
        self.block_range = (b0, b1)

    def block_kv(self, block, which):
        """(device pointer, bytes) of resident block `block`'s K (0) / V (1) lanes."""
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(self.L.sdv2_block_kv(self.h, block, which, ctypes.byref(p), ctypes.byref(n)), self.h)
        return p.value, n.value

    def profile_block_ms(self):
        """Mean ms per call of every resident block's span since profile_enable(True)."""
        nres = self.resident[1] - self.resident[0]
        out = (ctypes.c_double * nres)()
        _check(self.L.sdv2_profile_block_ms(self.h, out, nres), self.h)
        return list(out)

    def kv_lane(self, local_block, lane, which):
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(self.L.sdv2_kv_lane(self.h, local_block, lane, which, ctypes.byref(p), ctypes.byref(n)), self.h)
        return p.value, n.value

    def gemm_configs(self):
        """[(M, N, K, epi, MC, BN, SK, XE)] the handle's projection GEMMs run with
        (sdv2_gemm_configs; pass back as Stage(..., gemm_table=...) to pin them)."""
        cnt = ctypes.c_int32()
        _check(self.L.sdv2_gemm_configs(self.h, None, 0, ctypes.byref(cnt)), self.h)
        buf = (ctypes.c_int32 * max(8 * cnt.value, 1))()
        _check(self.L.sdv2_gemm_configs(self.h, buf, cnt.value, ctypes.byref(cnt)), self.h)
        return sorted(tuple(buf[8 * i:8 * i + 8]) for i in range(cnt.value))

    def close(self):
        if getattr(self, "h", None):
            self.L.sdv2_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ SLO batching (N2)
class LatencyPointC(ctypes.Structure):
    _fields_ = [("chunk_frames", ctypes.c_int32), ("streams", ctypes.c_int32), ("latency_s", ctypes.c_double)]


class SloC(ctypes.Structure):
    _fields_ = [("target_fps", ctypes.c_double), ("frame_deadline_s", ctypes.c_double),
                ("px_per_latent", ctypes.c_int32)]


class BatchDecisionC(ctypes.Structure):
    _fields_ = [("chunk_frames", ctypes.c_int32), ("streams", ctypes.c_int32), ("latency_s", ctypes.c_double),
                ("fps", ctypes.c_double), ("feasible", ctypes.c_int32)]


class AimdStateC(ctypes.Structure):
    _fields_ = [("streams", ctypes.c_int32), ("chunk_frames", ctypes.c_int32), ("b_max", ctypes.c_int32),
                ("streak", ctypes.c_int32), ("ok_run", ctypes.c_int32), ("infeasible", ctypes.c_int32)]


def _host_lib():
    """The host-only entry points live in both libraries; prefer the full one when built."""
    L = lib() if os.path.exists(_LIB_PATH) else ctl_lib()
    if not getattr(L, "_slo_declared", False):
        L.sdv2_slo_select.argtypes = [ctypes.POINTER(LatencyPointC), ctypes.c_int32, ctypes.POINTER(SloC),
                                      ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(BatchDecisionC)]
        L.sdv2_slo_select.restype = ctypes.c_int
        L.sdv2_slo_adapt.argtypes = [ctypes.POINTER(AimdStateC), ctypes.c_double, ctypes.POINTER(SloC)]
        L.sdv2_slo_adapt.restype = ctypes.c_int
        L.sdv2_slo_fit.argtypes = [ctypes.POINTER(LatencyPointC), ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_double)]
        L.sdv2_slo_fit.restype = ctypes.c_int
        L._slo_declared = True
    return L


def _table_c(table):
    items = sorted(table.items())
    arr = (LatencyPointC * len(items))(*[LatencyPointC(t, b, lat) for (t, b), lat in items])
    return arr, len(items)


def slo_select(table, target_fps, frame_deadline_s, buffered_frames, b_max, px_per_latent=4):
    """table {(T', B): measured call latency s} -> decision dict (library scheduler)."""
    arr, n = _table_c(table)
    out = BatchDecisionC()
    slo = SloC(target_fps, frame_deadline_s, px_per_latent)
    _check(_host_lib().sdv2_slo_select(arr, n, ctypes.byref(slo), buffered_frames, b_max, ctypes.byref(out)))
    return {"T": out.chunk_frames, "B": out.streams, "latency": out.latency_s, "fps": out.fps,
            "feasible": bool(out.feasible)}


class SloAdapter:
    """AIMD online adaptation of the batch size (library state machine)."""

    def __init__(self, B, T, b_max, streak, target_fps, frame_deadline_s, px_per_latent=4):
        self.st = AimdStateC(B, T, b_max, streak, 0, 0)
        self.slo = SloC(target_fps, frame_deadline_s, px_per_latent)

    def adapt(self, observed_latency_s):
        _check(_host_lib().sdv2_slo_adapt(ctypes.byref(self.st), observed_latency_s, ctypes.byref(self.slo)))
        return {"B": self.st.streams, "infeasible": bool(self.st.infeasible)}


def slo_fit(table):
    arr, n = _table_c(table)
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_host_lib().sdv2_slo_fit(arr, n, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


# ------------------------------------------------------- online block scheduler (N3)
def rebalance(measured_block_ms, stages, cur_bounds, ema, extra_first=0.0, extra_last=0.0, alpha=0.5,
              hysteresis=0.05):
    """Library policy sdv2_rebalance.  `ema` (list, updated in place) carries the smoothed
    per-block times between calls.  Returns (new_bounds, changed, pred_cur, pred_new)."""
    L = lib() if os.path.exists(_LIB_PATH) else ctl_lib()
    if not getattr(L, "_rb_declared", False):
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.POINTER(ctypes.c_int32)
        L.sdv2_rebalance.argtypes = [D, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, D, I, I, I, D, D]
        L.sdv2_rebalance.restype = ctypes.c_int
        L._rb_declared = True
    nb = len(measured_block_ms)
    m = (ctypes.c_double * nb)(*measured_block_ms)
    e = (ctypes.c_double * nb)(*ema)
    cb = (ctypes.c_int32 * (stages + 1))(*cur_bounds)
    nbd = (ctypes.c_int32 * (stages + 1))()
    ch = ctypes.c_int32()
    pc, pn = ctypes.c_double(), ctypes.c_double()
    _check(L.sdv2_rebalance(m, nb, stages, extra_first, extra_last, alpha, hysteresis, e, cb, nbd, ctypes.byref(ch),
                            ctypes.byref(pc), ctypes.byref(pn)))
    ema[:] = list(e)
    return list(nbd), bool(ch.value), pc.value, pn.value


def chunk_embedding(chunk: np.ndarray) -> np.ndarray:
    """Library host helper sdv2_chunk_embedding: per-channel mean of a [C, T', h, w] chunk."""
    L = lib() if os.path.exists(_LIB_PATH) else ctl_lib()
    a = np.ascontiguousarray(chunk, dtype=np.float32)
    C, T, H, W = a.shape
    out = np.zeros(C, dtype=np.float64)
    L.sdv2_chunk_embedding.argtypes = [ctypes.c_void_p] + [ctypes.c_int32] * 4 + [ctypes.c_void_p]
    L.sdv2_chunk_embedding.restype = ctypes.c_int
    _check(L.sdv2_chunk_embedding(ctypes.c_void_p(a.ctypes.data), C, T, H, W, ctypes.c_void_p(out.ctypes.data)))
    return out


# ------------------------------------------------------------ Stream-VAE stand-in (N1)
class VaeDescC(ctypes.Structure):
    _fields_ = [("video_h", ctypes.c_int32), ("video_w", ctypes.c_int32), ("dims", ctypes.c_int32 * 3),
                ("latent_channels", ctypes.c_int32), ("eps", ctypes.c_float)]


def vae_weight_order():
    """Tensor names in the order sdv2_vae_create takes them (include/sdv2.h)."""
    names = []
    enc = [("enc.conv_in", "conv"), ("enc.res1", "res"), ("enc.conv2", "conv"), ("enc.res2", "res"),
           ("enc.conv3", "conv"), ("enc.res3", "res"), ("enc.res4", "res"), ("enc.norm_out", "norm"),
           ("enc.conv_out", "conv")]
    dec = [("dec.conv_in", "conv"), ("dec.res1", "res"), ("dec.conv2", "conv"), ("dec.res2", "res"),
           ("dec.conv3", "conv"), ("dec.res3", "res"), ("dec.conv4", "conv"), ("dec.res4", "res"),
           ("dec.norm_out", "norm"), ("dec.conv_out", "conv")]
    for name, kind in enc + dec:
        p = f"vae.{name}."
        if kind == "conv":
            names += [p + "w", p + "b"]
        elif kind == "res":
            names += [p + "n1", p + "c1.w", p + "c1.b", p + "n2", p + "c2.w", p + "c2.b"]
        else:
            names += [p + "g"]
    return names


class StreamVAE:
    """Library Stream-VAE handle: encode / decode 4-frame chunks with feature caches."""

    def __init__(self, vd, H, W, weights, device=0, stream=None):
        import torch
        self.torch = torch
        L = lib()
        L.sdv2_vae_workspace_bytes.restype = ctypes.c_size_t
        L.sdv2_vae_workspace_bytes.argtypes = [ctypes.POINTER(VaeDescC)]
        L.sdv2_vae_create.argtypes = [ctypes.POINTER(VaeDescC), ctypes.POINTER(WeightsC), ctypes.c_void_p,
                                      ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        for f in ("sdv2_vae_create", "sdv2_vae_reset", "sdv2_vae_encode_chunk", "sdv2_vae_decode_chunk",
                  "sdv2_vae_destroy"):
            getattr(L, f).restype = ctypes.c_int
        L.sdv2_vae_reset.argtypes = [ctypes.c_void_p]
        L.sdv2_vae_encode_chunk.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sdv2_vae_decode_chunk.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sdv2_vae_destroy.argtypes = [ctypes.c_void_p]
        L.sdv2_vae_last_error.restype = ctypes.c_char_p
        L.sdv2_vae_last_error.argtypes = [ctypes.c_void_p]
        L.sdv2_vae_launches.restype = ctypes.c_int64
        L.sdv2_vae_launches.argtypes = [ctypes.c_void_p]
        self.L = L
        self.vd, self.H, self.W = vd, H, W
        self.desc = VaeDescC(H, W, (ctypes.c_int32 * 3)(*vd.dims), vd.latent_channels, vd.eps)
        nbytes = L.sdv2_vae_workspace_bytes(ctypes.byref(self.desc))
        if nbytes == 0:
            raise SDV2Error("invalid Stream-VAE descriptor")
        self.workspace = torch.empty(nbytes + 1024, dtype=torch.uint8, device=f"cuda:{device}")
        self.stream = stream if stream is not None else torch.cuda.Stream(device)
        names = vae_weight_order()
        keep = [np.ascontiguousarray(weights[n], dtype=np.float32) for n in names]
        ptrs = (ctypes.c_void_p * len(keep))(*[a.ctypes.data for a in keep])
        w = WeightsC(ptrs, len(keep))
        h = ctypes.c_void_p()
        st = L.sdv2_vae_create(ctypes.byref(self.desc), ctypes.byref(w), ctypes.c_void_p(self.workspace.data_ptr()),
                               nbytes + 1024, device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st != 0:
            msg = L.sdv2_vae_last_error(h).decode() if h.value else ""
            if h.value:
                L.sdv2_vae_destroy(h)
            raise SDV2Error(f"{STATUS.get(st, st)}: {msg}")
        self.h = h

    def _sync_in(self):
        cur = self.torch.cuda.current_stream()
        if cur != self.stream:
            self.stream.wait_stream(cur)

    def reset(self):
        _check(self.L.sdv2_vae_reset(self.h))

    def encode_chunk(self, video_ptr, latent_ptr):
        self._sync_in()
        st = self.L.sdv2_vae_encode_chunk(self.h, ctypes.c_void_p(video_ptr), ctypes.c_void_p(latent_ptr))
        if st != 0:
            raise SDV2Error(f"{STATUS.get(st, st)}: {self.L.sdv2_vae_last_error(self.h).decode()}")

    def decode_chunk(self, latent_ptr, video_ptr):
        self._sync_in()
        st = self.L.sdv2_vae_decode_chunk(self.h, ctypes.c_void_p(latent_ptr), ctypes.c_void_p(video_ptr))
        if st != 0:
            raise SDV2Error(f"{STATUS.get(st, st)}: {self.L.sdv2_vae_last_error(self.h).decode()}")

    def launches(self):
        return self.L.sdv2_vae_launches(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.L.sdv2_vae_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
