#!/usr/bin/env python
"""Per-source-line warp-stall samples of one kernel from an ncu report (reads the
`--page source --print-source cuda,sass` CSV): python tools/ncu_lines.py <report> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, src = "?", {}
agg = defaultdict(lambda: [0, 0])
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 6:
        continue
    try:
        ln = int(r[0])
        s_all, s_ni = int(r[4] or 0), int(r[5] or 0)
    except ValueError:
        continue
    src[(fname, ln)] = r[1]
    agg[(fname, ln)][0] += s_all
    agg[(fname, ln)][1] += s_ni
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (a, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a:7d} {100 * a / tot:5.1f}% (not-issued {n:6d}) {f}:{ln:<5} {src[(f, ln)].strip()[:100]}")
