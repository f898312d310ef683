"""Print per-launch kernel times from an ncu `--metrics gpu__time_duration.sum --csv` log."""
import csv
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def main(path):
    tot = 0.0
    for r in load(path):
        v = float(r["Metric Value"]) / 1000
        tot += v
        n = r["Kernel Name"].split("(")[0].replace("stamgpu::<unnamed>::", "")
        print(f"{v:9.1f} us  {n[:80]}  grid {r['Grid Size']} block {r['Block Size']}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
