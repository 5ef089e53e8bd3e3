"""Pinned H2D / D2H copy bandwidth and their overlap (the e2e leg's transfers)."""
import torch

for mb in (0.25, 1, 2, 4):
    n = int(mb * (1 << 20)) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, device="cuda")
    d2 = torch.empty(n, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = mb * 10 / 1024 / (e0.elapsed_time(e1) * 1e-3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    print(f"{mb:5.2f} MB  h2d {res['h2d']:6.1f} GB/s  d2h {res['d2h']:6.1f} GB/s  both {2 * mb * 10 / 1024 / (e0.elapsed_time(e1) * 1e-3):6.1f} GB/s")
