"""Duplex PCIe with chunked copies on two streams (does chunking keep both
directions busy?)."""
import time

import torch

n = 60_000_000
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunks, interleave):
    c = n // chunks
    if interleave:
        for k in range(chunks):
            with torch.cuda.stream(s1):
                d[k * c:(k + 1) * c].copy_(h[k * c:(k + 1) * c], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[k * c:(k + 1) * c].copy_(d2[k * c:(k + 1) * c], non_blocking=True)
    else:
        with torch.cuda.stream(s1):
            for k in range(chunks):
                d[k * c:(k + 1) * c].copy_(h[k * c:(k + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2):
            for k in range(chunks):
                h2[k * c:(k + 1) * c].copy_(d2[k * c:(k + 1) * c], non_blocking=True)


for chunks in (1, 4, 20, 60):
    for inter in (False, True):
        run(chunks, inter)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            run(chunks, inter)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        print(f"chunks {chunks:3d} interleave {inter}: {dt*1e3:.2f} ms  {2*n*8/dt/1e9:.1f} GB/s")
