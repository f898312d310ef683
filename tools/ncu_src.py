"""Per-CUDA-source-line instructions executed and stall samples from
`ncu -i REP --page source --csv --print-source=cuda,sass` (the rows whose
first column is a source line number).  Usage: ncu_src.py CSV [units] [top]"""
import csv
import sys
from collections import defaultdict


def main(path, units=1.0, top=40):
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    hdr = None
    with open(path, errors="replace") as fh:
        for r in csv.reader(fh):
            if len(r) > 5 and r[0] == "Line No":
                hdr = r
                ii = r.index("Instructions Executed")
                si = r.index("Warp Stall Sampling (All Samples)")
                continue
            if hdr is None or len(r) <= ii or not r[0].isdigit():
                continue
            try:
                n = float(r[ii] or 0)
                st = float(r[si] or 0)
            except ValueError:
                continue
            a = agg[int(r[0])]
            a[0] += n
            a[1] += st
            a[2] = r[1][:90]
    tot = sum(v[0] for v in agg.values()) or 1
    stot = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.4g} ({tot / units:.1f} per unit), stall samples {stot:.4g}")
    for ln, (n, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * n / tot:5.1f}% {n / units:8.2f}/unit  stall {100 * st / stot:5.1f}%  L{ln}: {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0,
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)
