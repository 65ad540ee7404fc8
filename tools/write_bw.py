import torch
for mb in (8, 16, 32, 64, 2048):
    n = mb * 1024 * 1024 // 4
    x = torch.empty(n, device="cuda")
    for _ in range(3): x.fill_(1.0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): x.fill_(1.0)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    y = torch.empty_like(x)
    with torch.cuda.graph(g := torch.cuda.CUDAGraph()):
        for _ in range(20): y.copy_(x)
    g.replay(); torch.cuda.synchronize()
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    us2 = a.elapsed_time(b) / 20 * 1e3
    print(f"{mb:5d} MB: fill {us:8.1f} us = {mb*1.048576/us:6.2f} TB/s write | copy {us2:8.1f} us = {2*mb*1.048576/us2:6.2f} TB/s r+w")
