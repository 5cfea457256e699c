"""Run-to-run determinism check of the bf16 HSTU stack on the GPU (debug tool).

Everything except fp32 atomic accumulation order is deterministic, so two runs on identical
inputs must agree to ~1e-6 (gradients) and bit-exactly (forward activations).  Prints per-layer,
per-parameter max|a-b|/max|a| across `--runs` repetitions.
usage: python tools/determinism.py [--users 256] [--runs 4]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2505_18654_b200 as m  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--users", type=int, default=256)
ap.add_argument("--runs", type=int, default=4)
ap.add_argument("--config", default="small")
args = ap.parse_args()
dev = torch.device("cuda:0")
cfg = synth.config(args.config, users=args.users)
seg = synth.gen_segments(cfg)
L = seg.astype(np.int64).sum(1)
ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
X = np.concatenate([synth.gen_user_x(cfg, u, int(L[u])) for u in range(len(seg))])
dZ = np.concatenate([synth.gen_user_dz(cfg, u, int(L[u])) for u in range(len(seg))])
Ps = [synth.gen_layer_params(cfg, li) for li in range(cfg["n_layers"])]
jb = m.JaggedBatch.build(seg, ts, dev)
lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
stack = m.HstuStack(lc, [m.params_to_device(P, torch.bfloat16, dev) for P in Ps], torch.bfloat16, dev)
stack.bind(jb)
outs = []
for r in range(args.runs):
    z = stack.forward(torch.from_numpy(X).to(dev, torch.bfloat16)).float().clone()
    dx = stack.backward(torch.from_numpy(dZ).to(dev, torch.bfloat16)).float().clone()
    torch.cuda.synchronize()
    outs.append((z, dx, [{k: v.clone() for k, v in g.items() if k != "_flat"} for g in stack.grads]))
z0, dx0, g0 = outs[0]
for r in range(1, args.runs):
    z, dx, g = outs[r]
    print(f"run {r}: z bit-equal {bool(torch.equal(z, z0))}  max|dz| {float((z - z0).abs().max()):.3e}  "
          f"dx bit-equal {bool(torch.equal(dx, dx0))}  max|ddx| {float((dx - dx0).abs().max()):.3e}")
    for li in range(len(g)):
        errs = []
        for k in g[li]:
            a, b = g0[li][k], g[li][k]
            e = float((a - b).abs().max() / a.abs().max().clamp_min(1e-30))
            errs.append(f"{k}={e:.1e}")
        print(f"   layer {li}: " + " ".join(errs))

# ---- the attention alone, through the public API (no bias sums): outputs must be bit-equal
print("attention alone (public API), bit-equality across runs:")
T, d = jb.total_tokens, cfg["d"]
gen = torch.Generator(device="cpu").manual_seed(7)
qkvu = (torch.randn(T, 4 * d, generator=gen) * 0.5).to(dev, torch.bfloat16)
dO = torch.randn(T, d, generator=gen).to(dev, torch.bfloat16)
pre = (torch.randn(T, 4 * d, generator=gen)).to(dev, torch.bfloat16)
q, k, v = qkvu[:, :d], qkvu[:, d:2 * d], qkvu[:, 2 * d:3 * d]
ref = None
bad_all = set()
for r in range(args.runs):
    o, _ = m.attn_fwd(lc, jb, q, k, v, 4 * d)
    dq, dk, dv, _ = m.attn_bwd(lc, jb, dO, q, k, v, 4 * d, silu_pre=pre)
    torch.cuda.synchronize()
    cur = [t.clone() for t in (o, dq, dk, dv)]
    if ref is None:
        ref = cur
        continue
    msg = []
    for name, a_, b_ in zip(("o", "dq", "dk", "dv"), ref, cur):
        eq = torch.equal(a_, b_)
        n = int((a_ != b_).sum())
        rows = torch.nonzero((a_ != b_).any(1)).flatten()
        msg.append(f"{name}: {'equal' if eq else f'{n} diffs in {rows.numel()} rows (first rows {rows[:6].tolist()})'}")
        if name == "dk":
            bad_all.update(rows.cpu().tolist())
    print(f"run {r}: " + "; ".join(msg))

# where do the differing dk rows sit? (user, local row, segment)
off = jb.host["offsets"]
ns_ = seg[:, 0] + seg[:, 1]
kv_ = ns_ + seg[:, 2]
bad = np.array(sorted(bad_all), dtype=np.int64)
if bad.size:
    us_ = np.searchsorted(off, bad, side="right") - 1
    for u in np.unique(us_)[:12]:
        rows = bad[us_ == u] - off[u]
        print(f"user {u}: L={int(L[u])} ns={int(ns_[u])} kv_end={int(kv_[u])} bad local rows {rows.min()}..{rows.max()} "
              f"({rows.size}); pairs {sorted(set((rows // 256).tolist()))} cta {sorted(set(((rows // 128) % 2).tolist()))}")
