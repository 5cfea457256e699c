#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box, on reports from gpurun_out/).

  python tools/ncu_summary.py launches <launches.csv>          per-kernel share of a launch list
  python tools/ncu_summary.py full <report.ncu-rep> [...]      key metrics + top stall reasons
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit_scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", "")) * unit_scale.get(d.get("Metric Unit", "ns"), 1e-6)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':62s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:62]:62s} {n:8d} {ms:9.3f} {ms / tot:7.1%}")
    print(f"{'total':62s} {'':8s} {tot:9.3f}")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"== {d['Kernel Name'][:110]}")
        for k, lab in KEYS:
            if k in d:
                print(f"   {lab:18s} {d[k]} {u.get(k, '')}")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        top = sorted(st, key=lambda kv: -kv[1])[:6]
        print("   stalls           " + ", ".join(f"{k} {v / tot:.0%}" for k, v in top))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            full(p)
