"""Multi-process (world_size 2, gloo, CPU) test of the data-parallel host logic:
identical LPT sharding on every rank, per-layer bucket all-reduce, 1/B_global scaling.  The
aggregated gradient must equal the pooled single-process gradient of the whole batch."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _user_grads(cfg, seg, users, P):
    """Oracle gradient SUMS of one layer over `users` (flattened in a fixed key order)."""
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    tot = None
    for u in users:
        u = int(u)
        L = int(seg[u].sum())
        X = synth.gen_user_x(cfg, u, L)
        dZ = synth.gen_user_dz(cfg, u, L)
        ts = synth.gen_user_ts(cfg, u, seg[u])
        gid = oracle.build_jagged(seg[u:u + 1])["group_id"]
        nU, nS, nR, K = (int(v) for v in seg[u])
        _, c = oracle.layer_fwd_user(X, gid, nU + nS, nR, K, ts, P, ocfg)
        _, g = oracle.layer_bwd_user(dZ, c, P, ocfg)
        flat = np.concatenate([g[k].ravel() for k in sorted(g)])
        tot = flat if tot is None else tot + flat
    return tot


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_18654_b200.dp import shard_users, GradAggregator
        cfg = synth.config("toy")
        seg = synth.gen_segments(cfg, 9)
        users, load = shard_users(seg, world, rank)  # the product LPT (libmtgr mtgr_balance_lpt)
        ro, lo = oracle.lpt(seg.astype(np.int64).sum(1), world)  # bit-exact with the oracle's
        assert np.array_equal(np.nonzero(np.asarray(ro) == rank)[0], users) and np.array_equal(lo, load)
        allu = [None] * world
        dist.all_gather_object(allu, users.tolist())
        P = synth.gen_layer_params(cfg, 0)
        g = torch.from_numpy(_user_grads(cfg, seg, users, P))
        # (mtgr_scale_f32 is a CUDA kernel: on the CPU process group the scale is torch's mul_)
        agg = GradAggregator(len(seg), scale_fn=lambda t, s: t.mul_(s))
        n = g.numel()
        agg.on_layer_done(0, g[: n // 2])   # two buckets, reduced asynchronously
        agg.on_layer_done(1, g[n // 2:])
        agg.finish(g)
        if rank == 0:
            pooled = _user_grads(cfg, seg, range(len(seg)), P) / len(seg)
            q.put((allu, load.tolist(), float(np.abs(g.numpy() - pooled).max()),
                   float(np.abs(pooled).max())))
    finally:
        dist.destroy_process_group()


def test_dp_aggregation_matches_pooled_gradient():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allu, load, err, scale = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat = sorted(u for us in allu for u in us)
    assert flat == list(range(9))                      # every user exactly once
    assert not set(allu[0]) & set(allu[1])
    assert max(load) <= (4 / 3) * max(max(load), sum(load) / world)
    assert err <= 1e-12 * max(scale, 1.0)


def _run(cmd, env=None, timeout=240):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable] + cmd, cwd=root, env=e, capture_output=True, text=True, timeout=timeout)


def test_bench_launch_two_ranks_reference_arm():
    """bench.py under torchrun with 2 ranks (the driver's launch, 127.0.0.1): rank 0 alone
    prints ONE JSON line with n_gpus 2; the other rank exits 0 without work."""
    import json
    r = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
              "--master-port", str(_free_port()), "bench.py", "--impl", "reference", "--gpus", "2",
              "--config", "toy", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"


def test_bench_rejects_gpus_world_mismatch():
    """--gpus N inside a launch of a different world size fails loudly (no silent 1-rank run)."""
    r = _run(["bench.py", "--gpus", "2", "--config", "toy"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
