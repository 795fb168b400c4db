import torch
torch.cuda.init()
for mb in (8, 15, 30, 60, 200):
    n = mb * (1 << 20) // 4
    x = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    for name, fn in (("sum", lambda: x.sum()), ("copy", lambda: y.copy_(x)), ("mul", lambda: torch.mul(x, 2.0, out=y))):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): fn()
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        us = 1e3 * a.elapsed_time(b) / 20
        print(f"{mb:4d} MB {name:5s} {us:7.2f} us  {mb * 1.048576 / us * (2 if name != 'sum' else 1):6.2f} TB/s(moved)")
