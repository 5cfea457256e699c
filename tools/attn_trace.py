"""Parse MTGR_ATTN_TRACE=1 output: clock64 pipeline events of the CTA pair (2,0,0)/(3,0,0) of
each attention launch.  usage: attn_trace.py <stderr log> [mode=N]"""
import sys

import numpy as np

for line in open(sys.argv[1]):
    if not line.startswith("ATTN_TRACE"):
        continue
    parts = line.split()
    mode = parts[1]
    if len(sys.argv) > 2 and mode != sys.argv[2]:
        continue
    v = np.array([int(x) for x in parts[2:]], dtype=np.int64).reshape(-1, 11, 64)
    for c in range(v.shape[0]):
        w = v[c]
        base = w[10, 10] if w[10, 10] else w[10, 4]

        def rel(x):
            return (x - base) if x else -1
        print(mode, "cta", c, "start", rel(w[10, 4]), "r1_ready", rel(w[10, 3]), "mainloop_end", rel(w[10, 0]),
              "o_full", rel(w[10, 1]), "e_ok", rel(w[10, 5]), "u_ok", rel(w[10, 6]), "computed", rel(w[10, 7]),
              "barrier", rel(w[10, 8]), "stored", rel(w[10, 9]), "end", rel(w[10, 2]))
        print("   epilogue: dg", rel(w[10, 11]), "chunks", [rel(w[10, 12 + i]) for i in range(4)])
        n = int((w[6] > 0).sum())
        print(" t | mma: kvwait_s kv_ok sfree_ok | acc: twait t_ok | smx: swait s_ok tfreewait tfree_ok tfull")
        for t in range(min(n, 20)):
            print("%2d | %7d %7d %7d | %7d %7d | %7d %7d %7d %7d %7d" % (
                t, rel(w[0, t]), rel(w[1, t]), rel(w[2, t]), rel(w[3, t]), rel(w[4, t]),
                rel(w[5, t]), rel(w[6, t]), rel(w[7, t]), rel(w[8, t]), rel(w[9, t])))
    if len(sys.argv) > 2:
        break
