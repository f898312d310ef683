"""Aggregate an ncu `--page source --print-source=cuda,sass --csv` dump per
CUDA source line: warp-stall samples and executed instructions."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    f = None
    hdr = None
    agg = defaultdict(lambda: [0, 0, ""])
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6:
            continue
        if r[0]:
            cur = (f, int(r[0]), r[1].strip()[:90])
            try:
                agg[cur][0] += int(r[4] or 0)
                agg[cur][1] += int(r[hdr.index("Instructions Executed")] or 0)
            except (ValueError, IndexError):
                pass
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*v[0]/tot_s:5.1f}% smp {100*v[1]/tot_i:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
