#!/usr/bin/env python
"""Benchmark of the f4 workload: sharded lookup of one step's
embedding IDs through the dynamic hash table (two-stage unique, owner all-to-all over NCCL,
find-or-insert, gather) plus its backward (segment sums, all-to-all back, SGD on the owner).

    python bench_embed.py [--ids N] [--dim D] [--steps K] [--warmup W]      (torchrun for N>1)

IDs per rank: Zipf(1.2) over a 20M vocabulary (long-tail item popularity), the count of a
`small`-config step (256 users x ~1030 tokens x 16 features ~ 4.2M).  One JSON line: IDs/s
(whole job), unique fractions, ms per step and the embed kernels' share.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ids", type=int, default=4_200_000)
    ap.add_argument("--dim", type=int, default=32)
    ap.add_argument("--vocab", type=int, default=20_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch.distributed as dist
    import paper_2505_18654_b200 as m
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    rng = np.random.default_rng(1000 + rank)
    ids = torch.from_numpy((rng.zipf(1.2, args.ids) % args.vocab).astype(np.int64)).to(dev)
    cap_v = 1 << 23
    shard = m.HashEmbedding(dim=args.dim, cap_v=cap_v, cap_k=2 * cap_v, seed=1, device=dev)
    emb = m.ShardedEmbedding(shard)
    g = torch.randn(args.ids, args.dim, device=dev, dtype=torch.bfloat16)

    def step(t):
        rows, ctx = emb.lookup(ids, now=t, dtype=torch.bfloat16)
        emb.backward_sgd(g, ctx, lr=1e-3)
        return ctx

    for w in range(args.warmup):
        ctx = step(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    m.prof_reset(); m.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(args.steps):
        ctx = step(args.warmup + s)
    e1.record()
    torch.cuda.synchronize()
    m.prof_enable(False)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    kern = m.prof_query()
    if rank == 0:
        u1 = ctx["m"]
        line = {"metric": "sharded hash-embedding lookup + backward IDs/s", "value": args.ids * world * args.steps / (ms / 1e3),
                "unit": "ids/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "dtype": "bf16 rows / fp32 table",
                "data": "synthetic Zipf(1.2) ids over a 20M vocabulary",
                "config": {"ids_per_rank": args.ids, "dim": args.dim, "unique_stage1_per_rank": u1,
                           "table_rows": shard.stats()["fresh_slots"], "cap_v": cap_v},
                "embed_kernels_ms_per_step": kern.get("embed", (0, 0.0))[1] / args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
