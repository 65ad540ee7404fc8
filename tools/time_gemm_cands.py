"""Time every GEMM tuner candidate (sdv2_debug_gemm_candidates / sdv2_debug_gemm_cfg) on the
DiT shapes at 1.3B 480p n = 1, cycling 30 weight buffers so W streams from HBM as in a step.
  python tools/time_gemm_cands.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_07399_b200.sdv2 import lib  # noqa: E402

P = ctypes.c_void_p
L = lib()
L.sdv2_debug_gemm_candidates.argtypes = [ctypes.c_int32] * 4 + [P, ctypes.c_int32, P]
L.sdv2_debug_gemm_cfg.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P, P]
shapes = [("QKV", 1560, 4608, 1536, 0), ("O", 1560, 1536, 1536, 2), ("crossQ", 1560, 1536, 1536, 0),
          ("crossO", 1560, 1536, 1536, 3), ("FFN1", 1560, 8960, 1536, 1), ("FFN2", 1560, 1536, 8960, 2)]
s = torch.cuda.current_stream()
for name, M, N, K, epi in shapes:
    buf = (ctypes.c_int32 * 256)()
    cnt = ctypes.c_int32()
    L.sdv2_debug_gemm_candidates(M, N, K, epi, buf, 64, ctypes.byref(cnt))
    cands = [tuple(buf[4 * i:4 * i + 4]) for i in range(cnt.value)]
    A = torch.randn(M, K, device="cuda").bfloat16()
    Ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16() for _ in range(30)]
    bias = torch.randn(N, device="cuda")
    mod = torch.randn(6, N, device="cuda")
    e0 = torch.randn(1, 6, N, device="cuda")
    out = torch.zeros(M, N, device="cuda") if epi >= 2 else torch.zeros(M, N, device="cuda").bfloat16()
    res = []
    for c in cands:
        cfg = (ctypes.c_int32 * 4)(*c)
        f = lambda w: L.sdv2_debug_gemm_cfg(A.data_ptr(), w.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                                            mod.data_ptr(), e0.data_ptr(), 2, 1560, cfg,
                                            torch.cuda.current_stream().cuda_stream)   # the capture stream
        for i in range(3):
            f(Ws[i])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(30):
                f(Ws[i])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / 90
        res.append((us, c))
    res.sort()
    flops = 2.0 * M * N * K
    print(name, " | ".join(f"MC{c[0]} BN{c[1]} XE{c[3]}: {us:.1f}us" for us, c in res[:6]),
          f"| best {flops / res[0][0] / 1e6:.0f} TFLOP/s")
