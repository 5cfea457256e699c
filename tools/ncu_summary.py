#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box, on reports from gpurun_out/).

  python tools/ncu_summary.py launches <launches.csv>          per-kernel share of a launch list
  python tools/ncu_summary.py full <report.ncu-rep> [...]      key metrics + top stall reasons
  python tools/ncu_summary.py traffic <config> <report.ncu-rep> [...]
        merge per-launch DRAM bytes (read + write) by bench kernel kind into
        profiles/traffic_per_launch.json (read by bench.py for roofline.traffic)
"""
import json
import os
import re
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


# bench.py kernel kinds of the captured kernels (attention MODE enum: FWD 0, DV 1, DQ 2, DK 3;
# GEMM EPI enum: STORE 0, QKVU 1, RESID 2, F32 3)
KIND = [(r"attn_tc_kernel<0>", "attn_fwd"), (r"attn_tc_kernel<1>", "attn_bwd_dv"),
        (r"attn_tc_kernel<2>", "attn_bwd_dq"), (r"attn_tc_kernel<3>", "attn_bwd_dk_fused"),
        (r"attn_sc_kernel", "attn_bwd_scores"), (r"attn_kv_kernel", "attn_bwd_kv"),
        (r"gemm_tc_kernel<1,", "gemm_qkvu"), (r"gemm_tc_kernel<2,", "gemm_out"),
        (r"gemm_tc_kernel<0,", "gemm_dgrad"), (r"gemm_tc_kernel<3,", "gemm_wgrad"),
        (r"gln_fwd_kernel", "gln_fwd"), (r"gln_bwd", "gln_bwd"),
        # stored-score backward GEMMs (MM_DV 0, MM_DQ 1)
        (r"attn_mm_kernel<1>", "attn_bwd_dq")]  # MM_DV serves dV and dK (same kernel)


def traffic(config, paths):
    out_p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic_per_launch.json")
    db = json.load(open(out_p)) if os.path.exists(out_p) else {}
    per = collections.defaultdict(list)
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[2:]:
            d = dict(zip(h, r))
            u = dict(zip(h, units))
            name = d["Kernel Name"].replace(" ", "")
            kind = next((k for pat, k in KIND if re.search(re.escape(pat.replace(" ", "")), name)), None)
            if kind is None:
                continue
            b = sum(float(d[m].replace(",", "")) * scale.get(u[m], 1)
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            per[kind].append(b)
    cfg = db.setdefault(config, {})
    for k, v in per.items():
        cfg[k] = sum(v) / len(v)
        print(f"{k:14s} {cfg[k] / 1e9:8.3f} GB per launch ({len(v)} launches)")
    json.dump(db, open(out_p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    else:
        for p in sys.argv[2:]:
            full(p)
