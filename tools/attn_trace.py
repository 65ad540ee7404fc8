"""Per-tile pipeline trace of CTA 0 of the tcgen05 attention kernel (test hook).

Events (clock64, SM cycles): 0 MMA saw V ready, 1/2 MMA saw P half 0/1 (PV issued),
3 MMA saw K ready (S issued), 4/6 softmax half 0/1 saw S, 5/7 softmax half 0/1 arrived P,
8 K producer got a free stage, 9 V producer got a free stage, 10/12 S loaded from TMEM,
11/13 row max done.  Usage: python tools/attn_trace.py [Lq Lk H] (per-unit mode)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_07399_b200.sdv2 import lib

Lq, Lk, H = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 5120, 12)
hd = 128
P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_attention.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
s = torch.cuda.current_stream().cuda_stream
scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")
q = torch.randn(Lq, H * hd, device="cuda").bfloat16()
k = torch.randn(Lk, H * hd, device="cuda").bfloat16()
v = torch.randn(Lk, H * hd, device="cuda").bfloat16()
o = torch.zeros(Lq, H * hd, device="cuda", dtype=torch.bfloat16)
f = lambda: L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                    scratch.data_ptr(), s)
for _ in range(3):
    f()
torch.cuda.synchronize()
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "attn_trace.csv")
os.makedirs(os.path.dirname(path), exist_ok=True)
os.environ["SDV2_ATTN_TRACE"] = path
f()
torch.cuda.synchronize()
del os.environ["SDV2_ATTN_TRACE"]
T = np.loadtxt(path, delimiter=",", dtype=np.int64)
n = int((T[:, 4] > 0).sum())
base = T[T > 0].min()
R = np.where(T > 0, T - base, -1)
names = ["Vrdy", "P0", "P1", "Krdy", "S0", "A0", "S1", "A1", "Kfree", "Vfree", "ld0", "mx0", "ld1", "mx1"]
print("tile " + " ".join(f"{x:>7}" for x in names))
for t in range(n):
    print(f"{t:4d} " + " ".join(f"{R[t, e]:7d}" for e in range(len(names))))
per = np.diff(R[:n, 5])
print(f"tiles {n}; softmax-half0 period median {np.median(per[2:]):.0f} cycles; "
      f"S->arrive {np.median(R[2:n, 5] - R[2:n, 4]):.0f}; ld {np.median(R[2:n, 10] - R[2:n, 4]):.0f}; "
      f"max {np.median(R[2:n, 11] - R[2:n, 10]):.0f}; exp+st {np.median(R[2:n, 5] - R[2:n, 11]):.0f}; "
      f"A0->P0(MMA saw) {np.median(R[2:n, 1] - R[2:n, 5]):.0f}; A1->P1 {np.median(R[2:n, 2] - R[2:n, 7]):.0f}; "
      f"P1(t)->S0(t+2) {np.median(R[4:n, 4] - R[2:n - 2, 2]):.0f}")
