"""Summarize ncu captures (gpurun_out/prof/*.ncu-rep) into profiles/:
per-kernel key metrics (duration, DRAM bytes, throughput, occupancy, IPC, L2
hit rate, top warp-stall reasons) as markdown + CSV, and traffic.json (DRAM
bytes per launch by workload/kernel, read by bench.py)."""
import csv
import json
import subprocess
import sys
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}

WORKLOAD = {  # capture name -> (bench workload, kernel label used by the library)
    "spadd_tiles": ("spadd3_200k_50perrow", "spadd_tiles<u32>"),
    "spgemm_cfg1_hashM1": ("spgemm_10k_20perrow", "spgemm_hashM1_numeric"),
    "spgemm_cfg3_long": ("spgemm_AxA_1M_powerlaw", "spgemm_long_numeric"),
    "spgemm_cfg3_hashM": ("spgemm_AxA_1M_powerlaw", "spgemm_hashM_numeric"),
    "mttkrp_dense32": ("mttkrp_dense_nell2shape_R32", "mttkrp_dense32"),
    "mttkrp_sparse": ("mttkrp_sparse_500k3_200M_R256", "mttkrp_sparse"),
}

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("launch__registers_per_thread", "regs"),
]


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def stalls(rep: Path, top=5):
    """Top warp-stall reasons from PC sampling (share of all samples)."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    pairs = []
    for i, name in enumerate(h):
        if name.startswith(pre) and not name.endswith("_not_issued"):
            try:
                pairs.append((float(v[i].replace(",", "")), name[len(pre):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in pairs) or 1.0
    pairs.sort(reverse=True)
    return ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in pairs[:top])


def main(src="gpurun_out/prof", dst="profiles", tag="r01"):
    src, dst = Path(src), Path(dst)
    dst.mkdir(exist_ok=True)
    traffic = {}
    lines = [f"# ncu captures ({tag}) — `ncu --set full --clock-control none` on B200, one launch each",
             "", "| capture | kernel | duration | DRAM read | DRAM write | DRAM % peak | SM % | "
             "occupancy % | IPC | L2 hit % | regs | top stall reasons (PC samples) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    table = []
    for rep in sorted(src.glob("*.ncu-rep")):
        h, units, v = raw(rep)
        d = {"capture": rep.stem, "kernel": v[h.index("Kernel Name")][:60]}
        for m, key in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[key] = float(v[i].replace(",", "")) * UNIT.get(units[i], 1.0)
                except ValueError:
                    d[key] = v[i]
        d["stalls"] = stalls(rep)
        table.append(d)
        if rep.stem in WORKLOAD:
            wl, kern = WORKLOAD[rep.stem]
            traffic.setdefault(wl, {})[kern] = int(d.get("dram_read", 0) + d.get("dram_write", 0))
        lines.append(
            f"| {d['capture']} | `{d['kernel']}` | {d.get('duration', 0)*1e3:.3f} ms | "
            f"{d.get('dram_read', 0)/1e6:.1f} MB | {d.get('dram_write', 0)/1e6:.1f} MB | "
            f"{d.get('dram_pct', 0):.1f} | {d.get('sm_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | "
            f"{d.get('ipc', 0):.2f} | {d.get('l2_hit_pct', 0):.1f} | {int(d.get('regs', 0))} | "
            f"{d['stalls']} |")
    (dst / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    with open(dst / f"{tag}_ncu_summary.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=sorted({k for d in table for k in d}))
        w.writeheader()
        w.writerows(table)
    old = {}
    tp = dst / "traffic.json"
    if tp.exists():
        old = json.loads(tp.read_text())
    for k, v in traffic.items():
        old.setdefault(k, {}).update(v)
    tp.write_text(json.dumps(old, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
