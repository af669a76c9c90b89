"""Pinned host->device copy time vs size (torch, CUDA events): is a 2 MB staged upload PCIe-rate?"""
import torch

for mb in (0.06, 0.5, 2.1, 8, 32):
    n = int(mb * 2**20 / 8)
    h = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(10):
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
    print(f"{mb:6.2f} MB  {best*1e3:8.1f} us  {n*8/best/1e6:6.1f} GB/s", flush=True)
