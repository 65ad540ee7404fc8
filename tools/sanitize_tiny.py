"""Tiny stream through the library for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): both precisions, graphs off (every launch visible), 10 chunks with
a prompt switch, a re-base and sink refresh, the same with the clean-context re-run (kv_mode 1), and the
kernel-level GEMM / attention hooks on
ragged shapes incl. the stream-K attention split.  Exit 0 iff outputs match the oracle.

  compute-sanitizer --tool memcheck python tools/sanitize_tiny.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import synthgen as sg  # noqa: E402
from gpu_harness import rel_l2, run_gpu, tiny_inputs  # noqa: E402
from oracle.stream import run_stream  # noqa: E402
from paper_2511_07399_b200.sdv2 import SDV2_BF16, SDV2_FP32, lib  # noqa: E402


def main():
    import torch
    cfg = sg.CONFIGS["tiny"]
    W, chunks, prompts = tiny_inputs(cfg, extra=cfg.geom.steps - 1)
    recs = run_stream(cfg, W, chunks, prompts, dtype=np.float64)
    worst = 0.0
    for prec, tol in ((SDV2_FP32, 1e-4), (SDV2_BF16, 2e-2)):
        outs, _, _ = run_gpu(cfg, W, chunks, prompts, prec, tap=True, graphs=False)
        for X in range(cfg.num_chunks):
            e = rel_l2(outs[X], recs[X]["out"])
            worst = max(worst, e)
            assert e <= tol, (prec, X, e)
    # clean-context re-run (kv_mode 1, n = 1): the extra pass and its descriptor
    import dataclasses
    cc = dataclasses.replace(cfg, geom=dataclasses.replace(cfg.geom, steps=1, kv_mode=1),
                             stream=dataclasses.replace(cfg.stream, timesteps=sg.SCHEDULES[1]))
    rc = run_stream(cc, W, chunks[:cc.num_chunks], prompts, dtype=np.float64)
    for prec, tol in ((SDV2_FP32, 1e-4), (SDV2_BF16, 2e-2)):
        outs, _, _ = run_gpu(cc, W, chunks[:cc.num_chunks], prompts, prec, tap=False, graphs=False)
        for X in range(cc.num_chunks):
            e = rel_l2(outs[X], rc[X]["out"])
            worst = max(worst, e)
            assert e <= tol, ("clean", prec, X, e)
    L = lib()
    P = ctypes.c_void_p
    L.sdv2_debug_attention.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P]
    s = torch.cuda.current_stream().cuda_stream
    for (Lq, Lk, H, hd) in [(300, 1000, 5, 64), (1560, 512, 12, 128)]:     # split units + in-kernel merge
        q = torch.randn(Lq, H * hd, device="cuda").bfloat16()
        k = torch.randn(Lk, H * hd, device="cuda").bfloat16()
        v = torch.randn(Lk, H * hd, device="cuda").bfloat16()
        o = torch.zeros_like(q)
        scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        assert L.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                      scratch.data_ptr(), s) == 0
    L.sdv2_debug_gemm.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P]
    for (M, N, K, epi) in [(200, 144, 192, 0), (1560, 1536, 1536, 2), (330, 8960, 1536, 1)]:
        A = torch.randn(M, K, device="cuda").bfloat16()
        Wt = torch.randn(N, K, device="cuda").bfloat16()
        b = torch.randn(N, device="cuda")
        out = torch.zeros(M, N, device="cuda") if epi >= 2 else torch.zeros(M, N, device="cuda").bfloat16()
        mod = torch.randn(6, N, device="cuda")
        e0 = torch.randn(M, 6, N, device="cuda")
        assert L.sdv2_debug_gemm(A.data_ptr(), Wt.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, epi,
                                 mod.data_ptr(), e0.data_ptr(), 2, 1560, s) == 0
    torch.cuda.synchronize()
    print(f"sanitize_tiny ok, worst rel-L2 {worst:.2e}")


if __name__ == "__main__":
    main()
