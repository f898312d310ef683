"""Minimal driver for ncu / compute-sanitizer: runs `--steps` device-resident
calls of one BASELINE config through the C ABI (no CPU baseline, no e2e).

    python tools/profile_step.py --config 2 --steps 3
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    import torch

    from paper_1802_10574_b200 import Context
    from paper_1802_10574_b200 import generators as G

    W = bench.WORKLOADS[args.config].__new__(bench.WORKLOADS[args.config])
    W.cid = args.config
    W.name = G.CONFIG_NAMES[args.config]
    W.cfg = G.make_config(args.config, scale=args.scale)
    W.broadcast_ms, W.broadcast_bytes = 0.0, 0
    ctx = Context(0)
    W.distribute(1, 0, False)
    W.setup(ctx)
    for _ in range(args.steps):
        W.step()
    torch.cuda.synchronize()
    print("ok", W.nnz_out)


if __name__ == "__main__":
    main()
