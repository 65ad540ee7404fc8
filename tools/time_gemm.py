"""Time the tcgen05 GEMM test hook at the DiT shapes (CUDA events, graph-free, back to
back) next to a warmed cuBLAS bf16 matmul of the same shape."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_07399_b200.sdv2 import lib
P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_gemm.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P]
s = torch.cuda.current_stream().cuda_stream
shapes = [(1560, 4608, 1536), (1560, 1536, 1536), (1560, 8960, 1536), (1560, 1536, 8960), (1560, 1536, 64),
          (1560, 256, 64), (6240, 4608, 1536), (6240, 1536, 1536), (6240, 8960, 1536), (6240, 1536, 8960)]
epis = [int(x) for x in os.environ.get("EPIS", "0,2").split(",")]


def t_us(fn, n=50):
    """Device time per call: n calls captured in a CUDA graph, replayed (no host launch cost)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for (M, N, K) in shapes:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    b = torch.randn(N, device="cuda")
    mod = torch.randn(6, N, device="cuda")
    e0 = torch.randn(8, 6, N, device="cuda")
    outb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    outf = torch.zeros(M, N, device="cuda")
    line = f"M={M:5d} N={N:5d} K={K:5d}"
    for epi in epis:
        out = outb if epi < 2 else outf
        us = t_us(lambda: L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, epi,
                                              mod.data_ptr(), e0.data_ptr(), 2, 1560,
                                              torch.cuda.current_stream().cuda_stream))
        line += f" | epi{epi} {us:7.1f} us {2*M*N*K/us/1e6:6.0f} TF"
    us = t_us(lambda: torch.matmul(A, W.T, out=outb))
    line += f" | cuBLAS {us:7.1f} us {2*M*N*K/us/1e6:6.0f} TF"
    print(line, flush=True)
