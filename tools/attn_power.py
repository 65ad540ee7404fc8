"""SM clock and power while one kernel class runs back to back (graph replay for ~4 s),
sampled with nvidia-smi: is the kernel clock- (power-) or cycle-bound?
  python tools/attn_power.py"""
import ctypes, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_07399_b200.sdv2 import lib

P = ctypes.c_void_p
L_ = lib()
L_.sdv2_debug_attention.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
L_.sdv2_debug_gemm.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32, P]
scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        out.append(r)
        time.sleep(0.2)


def run(name, fn, n=20, secs=4.0):
    for _ in range(3):
        fn(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        g.capture_begin()
        for _ in range(n):
            fn(cs.cuda_stream)
        g.capture_end()
    g.replay()
    torch.cuda.synchronize()
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp))
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    reps = 0
    a.record()
    while time.time() - t0 < secs:
        g.replay()
        reps += 1
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = a.elapsed_time(b) * 1e3 / (reps * n)
    clk = sorted(float(x.split(",")[0]) for x in smp[2:] if x)
    pw = sorted(float(x.split(",")[1]) for x in smp[2:] if x)
    print(f"{name}: {us:.1f} us per launch; SM clock median {clk[len(clk) // 2]:.0f} MHz, power median "
          f"{pw[len(pw) // 2]:.0f} W; reasons {smp[len(smp) // 2].split(',')[-1].strip()}", flush=True)


hd, H = 128, 12
q = torch.randn(1560, H * hd, device="cuda").bfloat16()
k = torch.randn(7800, H * hd, device="cuda").bfloat16()
v = torch.randn(7800, H * hd, device="cuda").bfloat16()
o = torch.zeros(1560, H * hd, device="cuda", dtype=torch.bfloat16)
run("self-attention 1560x7800x12", lambda s: L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                                   o.data_ptr(), 1560, 7800, H, hd,
                                                                   scratch.data_ptr(), s))
M, N, K = 1560, 8960, 1536
A = torch.randn(M, K, device="cuda").bfloat16()
W = torch.randn(N, K, device="cuda").bfloat16()
bb = torch.randn(N, device="cuda")
mod = torch.randn(6, N, device="cuda")
e0 = torch.randn(8, 6, N, device="cuda")
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
run("FFN1 GEMM 1560x8960x1536", lambda s: L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), bb.data_ptr(), out.data_ptr(),
                                                           M, N, K, 1, mod.data_ptr(), e0.data_ptr(), 2, 1560, s))
