"""Per-source-line executed warp instructions from an ncu source-page CSV
(`ncu -i R --page source --print-source=cuda,sass --csv`), normalised per unit."""
import csv
import sys
from collections import defaultdict


def main(path, units=1.0, top=40):
    f = hdr = None
    agg = defaultdict(lambda: [0, 0])
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6 or not r[0]:
            continue
        try:
            key = (f, int(r[0]), r[1].strip()[:90])
            agg[key][0] += int(r[hdr.index("Instructions Executed")] or 0)
            agg[key][1] += int(r[4] or 0)
        except (ValueError, IndexError):
            pass
    ti = sum(v[0] for v in agg.values()) or 1
    print(f"total warp instructions {ti} ({ti / units:.1f} per unit)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / ti:5.1f}% {v[0] / units:9.1f}/unit  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0,
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)
