"""Pipeline trace of CTA 0 of the tcgen05 GEMM (test hook).  Per k-block: 0 producer got
a free stage, 1 MMA saw the stage full; per tile: 2 MMA got the accumulator, 3 MMA issued
the tile, 4 epilogue saw it complete, 5 epilogue done.  Usage: gemm_trace.py M N K [epi]."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_07399_b200.sdv2 import lib

M, N, K = (int(x) for x in sys.argv[1:4])
epi = int(sys.argv[4]) if len(sys.argv) > 4 else 0
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
os.environ["SDV2_GEMM_TRACE"] = path
f()
torch.cuda.synchronize()
del os.environ["SDV2_GEMM_TRACE"]
T = np.loadtxt(path, delimiter=",", dtype=np.int64).reshape(2, 512, 8)
for cta in range(2):
    R = T[cta]
    if not (R > 0).any():
        continue
    base = R[R > 0].min()
    R = np.where(R > 0, R - base, -1)
    nk = int((R[:, 1] >= 0).sum())
    ntile = int((R[:, 2] >= 0).sum())
    print(f"CTA {cta}: k-blocks {nk}, tiles {ntile}")
    for t in range(ntile):
        print(f"  tile {t}: acc free {R[t,2]}, issued {R[t,3]}, epi saw {R[t,4]}, chunk0 loaded {R[t,6]}, "
              f"chunk0 done {R[t,7]}, epi done {R[t,5]}")
    if nk:
        full = R[:nk, 1]
        print("  MMA saw full (first 12):", full[:12].tolist())
        print("  producer got stage (first 12):", R[:12, 0].tolist())
        d = np.diff(full)
        print(f"  k-block period median {np.median(d):.0f} cycles, mean {d.mean():.0f}")
