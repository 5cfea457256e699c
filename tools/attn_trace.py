"""Parse MTGR_ATTN_TRACE=1 output of the persistent attention kernel: per-item clock64 events of
the CTA pair of cluster 1.  usage: attn_trace.py <stderr log> [mode=N]"""
import sys

import numpy as np

EV = ["start", "tiles_done", "next_R1", "o_full", "epi_done", "S0_issued", "last_acc", "R1_load", "lastC1"]
for line in open(sys.argv[1]):
    if not line.startswith("ATTN_TRACE"):
        continue
    parts = line.split()
    mode = parts[1]
    if len(sys.argv) > 2 and mode != sys.argv[2]:
        continue
    v = np.array([int(x) for x in parts[2:]], dtype=np.int64).reshape(-1, 20, 64)
    for c in range(v.shape[0]):
        w = v[c]
        base = w[10, 0]
        n = int((w[0] > 0).sum())
        print(mode, "cta", c, "items", n, "end", int(w[4, n - 1] - base) if n else -1)
        print(" i  nt | " + " ".join("%9s" % e for e in EV) + " | epilogue chunks (from o_full)")
        for i in range(min(n, 32)):
            row = [(int(w[e, i] - base) if w[e, i] else -1) for e in range(9)]
            ch = [(int(w[11 + c, i] - w[3, i]) if w[11 + c, i] else -1) for c in range(4)]
            print("%2d %3d | " % (i, w[9, i]) + " ".join("%9d" % x for x in row) + " | " + str(ch))
        if c == 0:
            nt = int(w[9, 1])
            print(" item 1 per tile (leader MMA warp / softmax warp 4), relative to its start:")
            print("  t   S_issued  acc_issued     s_ok   t_full   period(S)")
            b1 = w[0, 1]
            for t in range(min(nt, 64)):
                per = (w[16, t] - w[16, t - 1]) if t > 0 and w[16, t - 1] else 0
                print("%3d %9d %11d %8d %8d %8d" % (t, w[16, t] - b1 if w[16, t] else -1,
                      w[17, t] - b1 if w[17, t] else -1, w[18, t] - b1 if w[18, t] else -1,
                      w[19, t] - b1 if w[19, t] else -1, per))
    if len(sys.argv) > 2:
        break
