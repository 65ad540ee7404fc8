"""Time the tcgen05 attention test hook (kernel + merge) at the DiT attention shapes."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_07399_b200.sdv2 import lib
P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_attention.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
s = torch.cuda.current_stream().cuda_stream
scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")
for (Lq, Lk, H, hd) in [(1560, 7800, 12, 128), (1560, 512, 12, 128), (1024, 5120, 12, 128), (1560, 1560, 12, 128)]:
    q = torch.randn(Lq, H * hd, device="cuda").bfloat16()
    k = torch.randn(Lk, H * hd, device="cuda").bfloat16()
    v = torch.randn(Lk, H * hd, device="cuda").bfloat16()
    o = torch.zeros(Lq, H * hd, device="cuda", dtype=torch.bfloat16)
    f = lambda: L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                        scratch.data_ptr(), s)
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    # replay n calls from a CUDA graph so host launch cost never shows in the device time
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        g.capture_begin()
        for _ in range(n):
            L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                    scratch.data_ptr(), cs.cuda_stream)
        g.capture_end()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    fl = 4.0 * Lq * Lk * H * hd
    qh = q.view(Lq, H, hd).transpose(0, 1).unsqueeze(0)
    kh = k.view(Lk, H, hd).transpose(0, 1).unsqueeze(0)
    vh = v.view(Lk, H, hd).transpose(0, 1).unsqueeze(0)
    for _ in range(3):
        torch.nn.functional.scaled_dot_product_attention(qh, kh, vh)
    a.record()
    for _ in range(n):
        torch.nn.functional.scaled_dot_product_attention(qh, kh, vh)
    b.record()
    torch.cuda.synchronize()
    us2 = a.elapsed_time(b) / n * 1e3
    print(f"Lq={Lq} Lk={Lk} H={H}: {us:8.1f} us {fl/us/1e6:6.0f} TF (graph, +merge) | torch SDPA {us2:8.1f} us {fl/us2/1e6:6.0f} TF", flush=True)
