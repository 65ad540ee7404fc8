"""CTA-level wall-clock stamps (globaltimer) of one tcgen05 GEMM launch (test hook):
entry, set-up done, first accumulator complete, exit, relative to the earliest entry.
Usage: SDV2_GEMM_CFG=MC,BN,SK python tools/gemm_cta.py M N K epi"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_07399_b200.sdv2 import lib

M, N, K, epi = (int(x) for x in sys.argv[1:5])
P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_gemm.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P]
A = torch.randn(M, K, device="cuda").bfloat16()
W = torch.randn(N, K, device="cuda").bfloat16()
b = torch.randn(N, device="cuda")
mod = torch.randn(6, N, device="cuda")
e0 = torch.randn(8, 6, N, device="cuda")
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi < 2 else torch.zeros(M, N, device="cuda")
s = torch.cuda.current_stream().cuda_stream
f = lambda: L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, epi,
                               mod.data_ptr(), e0.data_ptr(), 2, 1560, s)
for _ in range(3):
    f()
torch.cuda.synchronize()
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "gemm_trace.csv")
os.makedirs(os.path.dirname(path), exist_ok=True)
for rep in range(2):
    os.environ["SDV2_GEMM_TRACE"] = path
    f()
    torch.cuda.synchronize()
    del os.environ["SDV2_GEMM_TRACE"]
    T = np.loadtxt(path + ".cta", delimiter=",", dtype=np.int64)
    T = T[T[:, 0] > 0]
    R = (T - T[:, 0].min()) / 1e3
    pct = lambda x: " ".join(f"{np.percentile(x, p):6.2f}" for p in (0, 50, 90, 100))
    print(f"M={M} N={N} K={K} epi={epi} cfg={os.environ.get('SDV2_GEMM_CFG')}: {len(T)} CTAs (us; min p50 p90 max)")
    print("  entry            ", pct(R[:, 0]))
    print("  set-up cost      ", pct(R[:, 1] - R[:, 0]))
    print("  to first acc done", pct(R[:, 2] - R[:, 1]))
    print("  first acc -> exit", pct(R[:, 3] - R[:, 2]))
    print("  exit             ", pct(R[:, 3]))
