"""Emulates the SpAdd host pipeline with plain copies: 6 input arrays uploaded
in blocks on one stream, 2 output arrays downloaded per block on another
stream gated by the block's upload event (optionally a host wait per block)."""
import sys
import time

import torch

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 8
HOSTWAIT = len(sys.argv) > 2 and sys.argv[2] == "hostwait"
n_in = 10_000_000  # per input array (80 MB)
ins_h = [torch.empty(n_in, dtype=torch.float64).pin_memory() for _ in range(6)]
ins_d = [torch.empty(n_in, dtype=torch.float64, device="cuda") for _ in range(6)]
n_out = 30_000_000
outs_d = [torch.empty(n_out, dtype=torch.float64, device="cuda") for _ in range(2)]
outs_h = [torch.empty(n_out, dtype=torch.float64).pin_memory() for _ in range(2)]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()


def run():
    evs = []
    ci, co = n_in // NB, n_out // NB
    for k in range(NB):
        with torch.cuda.stream(s_up):
            for a in range(6):
                ins_d[a][k * ci:(k + 1) * ci].copy_(ins_h[a][k * ci:(k + 1) * ci], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_up)
            evs.append(e)
    for k in range(NB):
        if HOSTWAIT:
            evs[k].synchronize()
        s_dn.wait_event(evs[k])
        with torch.cuda.stream(s_dn):
            for a in range(2):
                outs_h[a][k * co:(k + 1) * co].copy_(outs_d[a][k * co:(k + 1) * co], non_blocking=True)


run()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    run()
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
tot = (6 * n_in + 2 * n_out) * 8
print(f"blocks {NB} hostwait {HOSTWAIT}: {dt*1e3:.2f} ms  {tot/dt/1e9:.1f} GB/s total")
