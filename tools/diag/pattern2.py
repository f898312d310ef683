"""Duplex PCIe in the SpAdd e2e pattern with the uploads and downloads spread
over 1 or 2 streams per direction (do more copy engines help?)."""
import time

import torch

MB = 1 << 20
stages = 8
h_in = [torch.empty(10_700_000 // 8 * stages, dtype=torch.float64).pin_memory() for _ in range(6)]
d_in = [torch.empty_like(h, device="cuda") for h in h_in]
h_out = [torch.empty(32 * MB // 8 * stages, dtype=torch.float64).pin_memory() for _ in range(2)]
d_out = [torch.empty_like(h, device="cuda") for h in h_out]
ups = [torch.cuda.Stream() for _ in range(2)]
dns = [torch.cuda.Stream() for _ in range(2)]


def run(nup, ndn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(stages):
        for a, (h, d) in enumerate(zip(h_in, d_in)):
            n = h.numel() // stages
            with torch.cuda.stream(ups[a % nup]):
                d[k * n:(k + 1) * n].copy_(h[k * n:(k + 1) * n], non_blocking=True)
        for a, (h, d) in enumerate(zip(h_out, d_out)):
            n = h.numel() // stages
            with torch.cuda.stream(dns[a % ndn]):
                h[k * n:(k + 1) * n].copy_(d[k * n:(k + 1) * n], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    byts = sum(h.numel() * 8 for h in h_in) + sum(h.numel() * 8 for h in h_out)
    return dt * 1e3, byts / dt / 1e9


for _ in range(2):
    for nup, ndn in ((1, 1), (2, 1), (1, 2), (2, 2)):
        print("up streams", nup, "down streams", ndn, "ms %.2f  GB/s %.1f" % run(nup, ndn))
