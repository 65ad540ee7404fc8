"""CTA wall stamps (globaltimer) of one cross-attention launch (test hook): percentiles of
entry, set-up, first Q, first S, unit-0 P done, unit-0 epilogue done, last epilogue, exit
relative to the earliest entry.  Usage: python tools/xattn_cta.py [Lq Lk H]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_07399_b200.sdv2 import lib

Lq, Lk, H = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1560, 512, 12)
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
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "xattn_trace")
os.makedirs(os.path.dirname(path), exist_ok=True)
for rep in range(2):
    os.environ["SDV2_ATTN_TRACE"] = path
    f()
    torch.cuda.synchronize()
    del os.environ["SDV2_ATTN_TRACE"]
    T = np.loadtxt(path + ".xcta", delimiter=",", dtype=np.int64)
    T = T[T[:, 0] > 0]
    base = T[:, 0].min()
    R = np.where(T > 0, (T - base) / 1e3, np.nan)   # us
    pct = lambda x: " ".join(f"{np.nanpercentile(x, p):6.2f}" for p in (0, 50, 90, 100))
    names = ["entry", "set-up done", "first Q landed", "first S landed", "unit0 P done", "unit0 epi done",
             "last epi done", "exit"]
    print(f"Lq={Lq} Lk={Lk} H={H}: {len(T)} CTAs (us; min p50 p90 max)")
    for i, nme in enumerate(names):
        print(f"  {nme:16s}", pct(R[:, i]))
    print("  unit0 (Q -> epi)", pct(R[:, 5] - R[:, 2]), "| 2nd unit", pct(R[:, 6] - R[:, 5]))
