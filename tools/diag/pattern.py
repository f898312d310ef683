"""Duplex PCIe in the SpAdd e2e pattern: per stage, six ~10.7 MB H2D copies
(three operands x idx/vals) on one stream while two ~32 MB D2H copies run on
another; host buffers from torch pin_memory (inputs) and cudaMallocHost-like
pinned allocations (result).  Compares with one large copy per direction."""
import time

import torch

MB = 1 << 20
stages = 8
h_in = [torch.empty(10_700_000 // 8 * stages, dtype=torch.float64).pin_memory() for _ in range(6)]
d_in = [torch.empty_like(h, device="cuda") for h in h_in]
h_out = [torch.empty(32 * MB // 8 * stages, dtype=torch.float64).pin_memory() for _ in range(2)]
d_out = [torch.empty_like(h, device="cuda") for h in h_out]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()


def run(split):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(stages):
        with torch.cuda.stream(s_up):
            for h, d in zip(h_in, d_in):
                n = h.numel() // stages
                d[k * n:(k + 1) * n].copy_(h[k * n:(k + 1) * n], non_blocking=True)
        with torch.cuda.stream(s_dn):
            for h, d in zip(h_out, d_out):
                n = h.numel() // stages
                if split:
                    for c in range(4):
                        m = n // 4
                        h[k * n + c * m:k * n + (c + 1) * m].copy_(d[k * n + c * m:k * n + (c + 1) * m], non_blocking=True)
                else:
                    h[k * n:(k + 1) * n].copy_(d[k * n:(k + 1) * n], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    byts = sum(h.numel() * 8 for h in h_in) + sum(h.numel() * 8 for h in h_out)
    return dt * 1e3, byts / dt / 1e9


for split in (False, True, False):
    print("split", split, "ms %.2f  GB/s %.1f" % run(split))
