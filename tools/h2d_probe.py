"""Pinned host->device copy bandwidth probe (one-off measurement helper)."""
import time

import torch

dev = torch.device("cuda", 0)
for mb, parts in ((592, 1), (592, 18), (33, 1), (4, 1)):
    n = mb * (1 << 20) // 8 // parts
    hs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(parts)]
    ds = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(parts)]
    for _ in range(2):
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{mb} MB in {parts} parts: {ms:.2f} ms -> {mb * (1 << 20) / ms / 1e6:.1f} GB/s")
# two streams concurrently
n = 296 * (1 << 20) // 8
h1, h2 = torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty(n, dtype=torch.float64).pin_memory()
d1, d2 = torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"2 streams x 296 MB: {dt*1e3:.2f} ms -> {592 * (1 << 20) / dt / 1e9:.1f} GB/s")
