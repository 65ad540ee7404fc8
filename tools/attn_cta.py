"""CTA-level wall-clock stamps (globaltimer) of one tcgen05 attention launch (test hook):
entry, set-up done, first S issued, exit per CTA, relative to the earliest entry.
Usage: python tools/attn_cta.py Lq Lk H"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_07399_b200.sdv2 import lib

Lq, Lk, H = (int(x) for x in sys.argv[1:4])
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
for rep in range(2):
    os.environ["SDV2_ATTN_TRACE"] = path
    f()
    torch.cuda.synchronize()
    del os.environ["SDV2_ATTN_TRACE"]
    T = np.loadtxt(path + ".cta", delimiter=",", dtype=np.int64)
    T = T[T[:, 0] > 0]
    base = T[:, 0].min()
    R = (T - base) / 1e3   # us
    pct = lambda x: " ".join(f"{np.percentile(x, p):6.2f}" for p in (0, 50, 90, 100))
    print(f"Lq={Lq} Lk={Lk} H={H}: {len(T)} CTAs (us; min p50 p90 max)")
    print("  entry           ", pct(R[:, 0]))
    print("  set-up done     ", pct(R[:, 1]))
    print("  first S issued  ", pct(R[:, 2]))
    print("  exit            ", pct(R[:, 3]))
    print("  set-up cost     ", pct(R[:, 1] - R[:, 0]))
    print("  to first S      ", pct(R[:, 2] - R[:, 1]))
    print("  first S -> exit ", pct(R[:, 3] - R[:, 2]))
