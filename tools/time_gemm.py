"""Time the tcgen05 GEMM test hook at the DiT shapes for every epilogue (CUDA events)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_07399_b200.sdv2 import lib
P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_gemm.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P]
s = torch.cuda.current_stream().cuda_stream
for (M, N, K) in [(1560, 4608, 1536), (1560, 1536, 1536), (1560, 8960, 1536), (1560, 1536, 8960), (6240, 4608, 1536),
                  (6240, 8960, 1536), (6240, 1536, 8960)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    b = torch.randn(N, device="cuda")
    mod = torch.randn(6, N, device="cuda")
    e0 = torch.randn(8, 6, N, device="cuda")
    outb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    outf = torch.zeros(M, N, device="cuda")
    for epi in range(4):
        out = outb if epi < 2 else outf
        for _ in range(3):
            L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, epi, mod.data_ptr(), e0.data_ptr(), 2, 1560, s)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(20):
            L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, epi, mod.data_ptr(), e0.data_ptr(), 2, 1560, s)
        ev[1].record(); torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) / 20 * 1e3
        print(f"M={M} N={N} K={K} epi={epi}: {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s", flush=True)
    t = torch.cuda.Event(enable_timing=True); t2 = torch.cuda.Event(enable_timing=True)
    t.record()
    for _ in range(20): torch.matmul(A, W.T)
    t2.record(); torch.cuda.synchronize()
    us = t.elapsed_time(t2) / 20 * 1e3
    print(f"   cuBLAS (torch.matmul) {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s")
