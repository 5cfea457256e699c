import sys, numpy as np
for line in open(sys.argv[1]):
    if not line.startswith("ATTN_TRACE"): continue
    parts = line.split(); mode = parts[1]
    if len(sys.argv) > 2 and mode != sys.argv[2]: continue
    v = np.array([int(x) for x in parts[2:]], dtype=np.int64).reshape(11, 64)
    base = v[10, 4]
    def rel(x): return (x - base) if x else -1
    print(mode, "start", 0, "r1_ready", rel(v[10, 3]), "mainloop_end(o_full wait start)", rel(v[10, 0]), "o_full", rel(v[10, 1]),
          "e_ok", rel(v[10, 5]), "u_ok", rel(v[10, 6]), "computed", rel(v[10, 7]), "barrier", rel(v[10, 8]), "stored", rel(v[10, 9]), "end", rel(v[10, 2]))
    n = int((v[6] > 0).sum())
    print(" t | mma: kvwait_s kv_ok sfree_ok | acc: twait t_ok | smx: swait s_ok tfreewait tfree_ok tfull")
    for t in range(min(n, 20)):
        print("%2d | %7d %7d %7d | %7d %7d | %7d %7d %7d %7d %7d" % (t, rel(v[0, t]), rel(v[1, t]), rel(v[2, t]), rel(v[3, t]), rel(v[4, t]), rel(v[5, t]), rel(v[6, t]), rel(v[7, t]), rel(v[8, t]), rel(v[9, t])))
    if len(sys.argv) < 3 or mode == sys.argv[2]: break
