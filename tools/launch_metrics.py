"""Per-launch table from an ncu --csv log holding several metrics per launch.

    python tools/launch_metrics.py gpurun_out/launches.csv [last_n]
"""
import csv
import sys
from collections import OrderedDict


def main(path, last=0):
    lines = open(path).read().splitlines()
    st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    d = OrderedDict()
    for r in csv.DictReader(lines[st:]):
        e = d.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0].replace("stamgpu::<unnamed>::", "")[:44],
                                   "grid": r["Grid Size"], "block": r["Block Size"]})
        e[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    rows = list(d.values())
    if last:
        rows = rows[-last:]
    for e in rows:
        t = e.get("gpu__time_duration.sum", 0.0) / 1000
        rd = e.get("dram__bytes_read.sum", 0.0) / 1e6
        wr = e.get("dram__bytes_write.sum", 0.0) / 1e6
        print(f"{t:9.1f} us  rd {rd:9.1f} MB  wr {wr:9.1f} MB  {e['name']}  grid {e['grid']} block {e['block']}")
    print(f"total {sum(e.get('gpu__time_duration.sum', 0.0) for e in rows) / 1000:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
