#!/usr/bin/env python
"""Trace the coupled dK/dV kernel (MTGR_KV_TRACE) on one `small` layer, or parse a saved log.

  MTGR_KV_TRACE=1 python tools/kv_trace.py run [config] 2> log     (on the GPU box)
  python tools/kv_trace.py parse log                                 (here)
Events per item (couple 0, CTA rank 0 of the X and the Y pair; globaltimer ns): start, tiles
done, o_full, epilogue done, ntiles, first S issued, last acc issued; per tile: s_full passed and
t_full arrived (softmax warp 4), S issued (MMA warp)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg_name="small"):
    import torch
    import synth
    import paper_2505_18654_b200 as m
    cfg = synth.config(cfg_name, n_layers=1)
    dev = torch.device("cuda:0")
    seg = synth.gen_segments(cfg)
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
    X = np.concatenate([synth.gen_user_x(cfg, u, int(L[u])) for u in range(len(seg))])
    dZ = np.concatenate([synth.gen_user_dz(cfg, u, int(L[u])) for u in range(len(seg))])
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    st = m.HstuStack(lc, [m.params_to_device(synth.gen_layer_params(cfg, 0), torch.bfloat16, dev)], torch.bfloat16, dev)
    st.bind(jb)
    x = torch.from_numpy(X).to(dev, torch.bfloat16)
    dz = torch.from_numpy(dZ).to(dev, torch.bfloat16)
    for _ in range(2):
        st.forward(x)
        st.backward(dz)
    torch.cuda.synchronize()


def parse(path):
    last = None
    for line in open(path):
        if line.startswith("KV_TRACE"):
            last = line
    v = np.array([int(t) for t in last.split()[1:]], dtype=np.int64).reshape(2, 2, 26, 1024)[:, 0]
    base = min(int(x[x > 0].min()) for x in (v[0], v[1]))
    for role in (0, 1):
        w = v[role]
        n = int((w[0] > 0).sum())
        print(f"== role {'XY'[role]}: items {n}, end {int(w[3, n - 1] - base) if n else -1} ns")
        print("  i  nt    start  S0_issue tiles_done   o_full  epi_done  last_acc | per-tile ns")
        gt = 0
        for i in range(min(n, 70)):
            nt = int(w[4, i])
            r = lambda e: int(w[e, i] - base) if w[e, i] else -1
            per = (r(1) - r(5)) / nt if nt and w[1, i] and w[5, i] else 0
            print(f"{i:3d} {nt:3d} {r(0):8d} {r(5):9d} {r(1):10d} {r(2):8d} {r(3):9d} {r(6):9d} | {per:7.0f}")
            gt += nt
        s_ok = w[7][w[7] > 0]
        if len(s_ok) > 2:
            d = np.diff(s_ok)
            print(f"  s_full period: median {np.median(d):.0f} ns, p10 {np.percentile(d, 10):.0f}, p90 {np.percentile(d, 90):.0f}")
        nts = w[4][:64]
        starts = np.cumsum(np.r_[0, nts[:-1]])
        for i in (5, 6):
            g0, nt = int(starts[i]), int(nts[i])
            b = w[9][g0]
            print(f"  item {i} ({nt} tiles), ns from its first S issue: C1 load / X load / c1_full seen / S issued / s_full / t_full / x_full seen")
            for t in range(nt):
                g = g0 + t
                f = lambda e: int(w[e][g] - b) if w[e][g] else -1
                print(f"   t{t:2d} {f(10):7d} {f(11):7d} {f(12):7d} {f(9):7d} {f(7):7d} {f(8):7d} {f(13):7d}")
        a = w[8][:len(s_ok)] - w[7][:len(s_ok)]
        a = a[(w[8][:len(s_ok)] > 0)]
        if len(a):
            print(f"  softmax (s_full -> t_full) median {np.median(a):.0f} ns")


def summary(path):
    """One line per role: ns per tile over the traced couple's whole span, median tile-loop ns
    per tile, median softmax (s_full -> t_full) and epilogue (o_full -> done) ns."""
    last = None
    for line in open(path):
        if line.startswith("KV_TRACE"):
            last = line
    v = np.array([int(t) for t in last.split()[1:]], dtype=np.int64).reshape(2, 2, 26, 1024)[:, 0]
    for role in (0, 1):
        w = v[role]
        n = int((w[0] > 0).sum())
        rows = [i for i in range(n) if w[4][i] > 0]
        tiles = int(w[4][:n].sum())
        span = w[3][n - 1] - w[0][0]
        sm = w[8][:tiles] - w[7][:tiles]
        loop = np.median([(w[1][i] - w[0][i]) / w[4][i] for i in rows])
        epi = np.median([w[3][i] - w[2][i] for i in rows])
        print(f"{os.path.basename(path)} {'XY'[role]}: items {n} tiles {tiles} span/tile {span / tiles:.0f} "
              f"loop/tile {loop:.0f} softmax {np.median(sm[sm > 0]):.0f} epilogue {epi:.0f} ns")


def warps(path):
    """Per tile: each softmax warp's T-tile arrival relative to the earliest (both CTAs)."""
    last = None
    for line in open(path):
        if line.startswith("KV_TRACE"):
            last = line
    v = np.array([int(t) for t in last.split()[1:]], dtype=np.int64).reshape(2, 2, 26, 1024)
    for role in (0, 1):
        a = v[role][:, 18:26, :]            # [crank][warp][tile]
        ok = (a > 0).all(axis=(0, 1))
        rel = a[:, :, ok] - a[:, :, ok].min(axis=(0, 1), keepdims=True)
        print(f"role {'XY'[role]}: {ok.sum()} tiles; median lag (ns) behind the first warp, [crank][warp 4..11]:")
        print(np.median(rel, axis=2).astype(int))
        print("   last-warp lag median", int(np.median(rel.max(axis=(0, 1)))))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(*(sys.argv[2:3]))
    elif sys.argv[1] == "warps":
        warps(sys.argv[2])
    elif sys.argv[1] == "summary":
        for f in sys.argv[2:]:
            summary(f)
    else:
        parse(sys.argv[2])
