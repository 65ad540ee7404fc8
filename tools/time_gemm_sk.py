"""Time explicit GEMM configurations (MC, BN, SK, XE) incl. stream-K at the DiT shapes,
cycling 30 weight buffers as in a step (sdv2_debug_gemm_cfg).  python tools/time_gemm_sk.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_07399_b200.sdv2 import lib
P = ctypes.c_void_p
L = lib()
L.sdv2_debug_gemm_candidates.argtypes = [ctypes.c_int32] * 4 + [P, ctypes.c_int32, P]
L.sdv2_debug_gemm_cfg.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P, P]
L.sdv2_debug_gemm_cfg.restype = ctypes.c_int
shapes = [("FFN2", 1560, 1536, 8960, 2), ("FFN1", 1560, 8960, 1536, 1), ("QKV", 1560, 4608, 1536, 0),
          ("O", 1560, 1536, 1536, 2), ("crossQ", 1560, 1536, 1536, 0)]
for name, M, N, K, epi in shapes:
    buf = (ctypes.c_int32 * 256)()
    cnt = ctypes.c_int32()
    L.sdv2_debug_gemm_candidates(M, N, K, epi, buf, 64, ctypes.byref(cnt))
    cands = [tuple(buf[4 * i:4 * i + 4]) for i in range(cnt.value)]
    extra = [(mc, bn, 1, 0) for mc in (1, 2) for bn in (64, 96, 128, 160, 192, 224, 256)
             if N % (bn // mc if mc == 2 else 1) == 0 or True]
    A = torch.randn(M, K, device="cuda").bfloat16()
    Ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16() for _ in range(30)]
    bias = torch.randn(N, device="cuda")
    mod = torch.randn(6, N, device="cuda")
    e0 = torch.randn(1, 6, N, device="cuda")
    out = torch.zeros(M, N, device="cuda") if epi >= 2 else torch.zeros(M, N, device="cuda").bfloat16()
    res = []
    for c in cands + extra:
        cfg = (ctypes.c_int32 * 4)(*c)
        f = lambda w: L.sdv2_debug_gemm_cfg(A.data_ptr(), w.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                                            mod.data_ptr(), e0.data_ptr(), 2, 1560, cfg,
                                            torch.cuda.current_stream().cuda_stream)
        if f(Ws[0]) != 0:
            continue
        torch.cuda.synchronize()
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
        res.append((a.elapsed_time(b) * 1e3 / 90, c))
    res.sort()
    flops = 2.0 * M * N * K
    print(name, " | ".join(f"MC{c[0]} BN{c[1]} SK{c[2]} XE{c[3]}: {us:.1f}" for us, c in res[:8]),
          f"| best {flops / res[0][0] / 1e6:.0f} TFLOP/s", flush=True)
