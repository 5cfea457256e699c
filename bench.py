#!/usr/bin/env python
"""Benchmark of the MTGR hot path: jagged GLN + HSTU layer stack, forward + backward, on B200.

One step = every row of SURVEY §8(a) over one batch: (a1 builder + LPT run once at setup; the
batch is fixed) a2-a6 forward through all layers, a7 backward, a8 gradient aggregation
(NCCL all-reduce of per-layer buckets overlapped with the backward, then the 1/B_global scale).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config small] [--impl reference]

Multi-GPU: launched by torchrun, one process per GPU, users sharded by the token-count LPT
balancer (weak scaling: `users` per rank fixed).  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "jagged HSTU layer fwd+bwd tokens/s at 1/2/4/8 B200; % bf16 tensor peak"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="small")
    ap.add_argument("--impl", default="mtgr", choices=["mtgr", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-users", type=int, default=24, help="users in the CPU oracle sample (~10 s)")
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--post-mlp", type=int, default=1, choices=[1, 2],
                    help="post-gate MLP: one Linear (R#6) or Linear-SiLU-Linear (S:354 variant)")
    ap.add_argument("--mask", default="dynamic", choices=["dynamic", "causal", "full"],
                    help="mask mode: MTGR's dynamic mask, or the Table 4 ablation read as causal / full attention")
    ap.add_argument("--full-model", action="store_true",
                    help="step = the whole training step: sparse IDs -> sharded hash-embedding lookup -> "
                         "tokens -> stack -> head/BCE -> backward -> sparse SGD (paper_2505_18654_b200.model)")
    ap.add_argument("--tokens", action="store_true",
                    help="step also runs the Eq.4 token construction (SURVEY f2) before the stack and its backward after")
    ap.add_argument("--head", action="store_true",
                    help="step = stack fwd + candidate head/BCE (SURVEY f2) + stack bwd from the head's dZ")
    ap.add_argument("--balance", default="tokens", choices=["tokens", "flops"],
                    help="LPT cost: token count (R#19, default) or per-user FLOPs (SURVEY f3)")
    ap.add_argument("--rab", type=int, default=0, metavar="NB",
                    help="optional relative-time bias with NB buckets (R#4; 0 = Eq.5 exactly, MTGR)")
    ap.add_argument("--no-large-attn", action="store_true",
                    help="skip the MTGR-large attention sub-record (one large layer fwd+bwd, N=1 only)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


# ------------------------------------------------------------------ workload (both arms)

def visible_pairs(seg_u, ts_u, mask="dynamic"):
    """P_u = L*n_s + sum_{i >= n_s} |{j in rt : ts_j < ts_i}| + (L - n_s);
    causal mask: L (L + 1) / 2; full mask: L (n_s + n_r) + K.
    Measurement bookkeeping for the algorithmic FLOP count (not part of the hot path)."""
    nU, nS, nR, K = (int(v) for v in seg_u)
    ns, L = nU + nS, nU + nS + nR + K
    if mask == "causal":
        return L * (L + 1) // 2
    if mask == "full":
        return L * (ns + nR) + K
    rt = np.sort(ts_u[ns:ns + nR])
    rows = ts_u[ns:]
    return L * ns + int(np.searchsorted(rt, rows, side="left").sum()) + (L - ns)


def workload(cfg, rank, world, balance, cost_kind="tokens"):
    B_rank = cfg["users"]
    B_g = B_rank * world
    seg = synth.gen_segments(cfg, B_g)
    L = seg.astype(np.int64).sum(1)
    if cost_kind == "flops":
        from paper_2505_18654_b200.dp import flop_cost
        cost = flop_cost(seg, [synth.gen_user_ts(cfg, u, seg[u]) for u in range(B_g)], cfg["d"])
    else:
        cost = L
    rank_of, load = balance(cost, world)
    users = np.nonzero(rank_of == rank)[0].astype(np.int32)
    ts = [synth.gen_user_ts(cfg, int(u), seg[u]) for u in users]
    P = sum(visible_pairs(seg[u], t, cfg.get("mask_mode", "dynamic")) for u, t in zip(users, ts))
    return dict(seg=seg, users=users, ts=ts, L=L, load=load, B_g=B_g, pairs=P,
                tokens=int(L[users].sum()), tokens_global=int(L.sum()), balance=cost_kind)


def step_flops(cfg, tokens, pairs):
    """Algorithmic FLOPs of one fwd+bwd step: fwd 10Ld^2 + 4dP, bwd 20Ld^2 + 8dP
    per layer (S recompute and redundant backward products are not counted)."""
    d, nl = cfg["d"], cfg["n_layers"]
    extra = 6.0 * tokens * d * d if cfg.get("post_mlp_layers", 1) == 2 else 0.0  # second Linear
    return nl * (30.0 * tokens * d * d + 12.0 * d * pairs + extra)


def kernel_algorithmic(cfg, tokens, pairs):
    """Per-step algorithmic FLOPs (tensor) or bytes (hbm) of each kernel kind."""
    d, nl = cfg["d"], cfg["n_layers"]
    T = tokens
    p2 = 1.0 if cfg.get("post_mlp_layers", 1) == 2 else 0.0
    return {
        "attn_fwd": ("tensor", nl * 4.0 * d * pairs),
        # stored-score backward: the score kernel does the dP product (S^T is the recompute the
        # algorithmic count excludes), then one jagged GEMM each for dV, dK, dQ
        "attn_bwd_scores": ("tensor", nl * 2.0 * d * pairs),
        "attn_bwd_dv": ("tensor", nl * 2.0 * d * pairs),
        "attn_bwd_dk": ("tensor", nl * 2.0 * d * pairs),
        "attn_bwd_dq": ("tensor", nl * 2.0 * d * pairs),
        # DK kernel that also forms dP (recompute path, MTGR_ATTN_RECOMPUTE / MTGR_ATTN_BWD=fused_dk)
        "attn_bwd_dk_fused": ("tensor", nl * 4.0 * d * pairs),
        # coupled dK/dV kernel (default backward): dP, dV, dK (its S^T is the excluded recompute)
        "attn_bwd_kv": ("tensor", nl * 6.0 * d * pairs),
        # post_mlp_layers == 2: the first post-gate Linear runs on the SiLU epilogue (qkvu kind),
        # the second on the residual epilogue; each adds 2Td^2 to dgrad and wgrad
        "gemm_qkvu": ("tensor", nl * (8.0 + 2.0 * p2) * T * d * d),
        "gemm_out": ("tensor", nl * 2.0 * T * d * d),
        "gemm_dgrad": ("tensor", nl * (10.0 + 2.0 * p2) * T * d * d),
        "gemm_wgrad": ("tensor", nl * (10.0 + 2.0 * p2) * T * d * d),
        # GLN fwd: read x, write y (bf16) + 2 fp32 stats; GLN bwd: read dy, x, (o, u, p_U) ...
        # GLN1 reads x, writes x~; GLN2 reads O and U (the gate), writes y~
        "gln_fwd": ("hbm", nl * T * ((4.0 * d + 8) + (6.0 * d + 8))),
        "gln_bwd": ("hbm", nl * T * ((12.0 * d + 8) + (8.0 * d + 8))),
    }


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []  # (host time, csv line)
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi has produced a sample (it takes a while to start)."""
        t_end = time.monotonic() + timeout
        while self.proc is not None and not self.lines and time.monotonic() < t_end:
            time.sleep(0.01)

    def mark(self, t0, t1):
        """Host-time bounds of the timed region: only samples inside it are reported."""
        self.window = (t0, t1)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None:
            t0, t1 = self.window
            inside = [x for x in lines if t0 <= x[0] <= t1 + 0.03]  # + one sampling period
            lines = inside if inside else [x for x in lines if x[0] <= t1][-2:]  # the nearest under load
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def gpu_id_for(torch, dev):
    try:
        p = torch.cuda.get_device_properties(dev)
        return f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return str(dev.index or 0)


# ------------------------------------------------------------------ CPU oracle timing

def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((i.get("num_threads", 0) for i in info if i.get("user_api") == "blas"), default=0)
        return int(n) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def time_oracle(cfg, wl, n_users, start=0):
    import oracle
    ocfg = dict(d=cfg["d"], H=cfg["H"], mask_mode=cfg.get("mask_mode", "dynamic"),
                post_mlp_layers=cfg.get("post_mlp_layers", 1))
    Ps = [synth.gen_layer_params(cfg, li, cfg.get("rab_buckets", 0)) for li in range(cfg["n_layers"])]
    tok, secs = 0, 0.0
    for k in range(n_users):
        idx = (start + k) % len(wl["users"])
        u = int(wl["users"][idx])
        nU, nS, nR, K = (int(v) for v in wl["seg"][u])
        L = nU + nS + nR + K
        X = synth.gen_user_x(cfg, u, L)
        dZ = synth.gen_user_dz(cfg, u, L)
        gid = oracle.build_jagged(wl["seg"][u:u + 1])["group_id"]
        t1 = time.perf_counter()
        z, caches = oracle.stack_fwd_user(X, gid, nU + nS, nR, K, wl["ts"][idx], Ps, ocfg)
        oracle.stack_bwd_user(dZ, caches, Ps, ocfg)
        secs += time.perf_counter() - t1
        tok += L
    return tok, secs


def _seg_desc(spec):
    if spec[0] == "fixed":
        return str(spec[1])
    if spec[0] == "uniform":
        return f"U{{{spec[1]}..{spec[2]}}}"
    return f"min({spec[3]}, {spec[1]}*u^(-1/{spec[2]}))"


def workload_desc(cfg, wl, world):
    return {"workload": f"MTGR-{cfg['name']} shape: {cfg['n_layers']} layers, d={cfg['d']}, "
                        f"{cfg['H']} heads (d_h={cfg['d'] // cfg['H']}), {cfg['users']} users/rank x "
                        f"(n_U={_seg_desc(cfg['nU'])}, n_S={_seg_desc(cfg['nS'])}, "
                        f"n_r={_seg_desc(cfg['nR'])}, K={_seg_desc(cfg['K'])})",
            "users_per_rank": cfg["users"], "global_batch_users": wl["B_g"],
            "tokens_global": wl["tokens_global"], "mean_len": round(wl["tokens_global"] / wl["B_g"], 1),
            "parallelism": f"dp{world}",
            "balancer": "FLOP-cost LPT" if wl.get("balance") == "flops" else "token-count LPT",
            "mask": cfg.get("mask_mode", "dynamic"),
            "post_mlp_layers": cfg.get("post_mlp_layers", 1),
            "rab_buckets": cfg.get("rab_buckets", 0),
            "l2": "no flush: per-step activations are several GB (>> 126 MB L2)"}


# ------------------------------------------------------------------ reference arm (CPU oracle)

def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    import oracle
    wl = workload(cfg, 0, world, lambda L, w: oracle.lpt(L, w))
    for s in range(args.warmup):
        time_oracle(cfg, wl, 1, start=s)
    tok = secs = 0
    for s in range(args.steps):
        t, sec = time_oracle(cfg, wl, 1, start=args.warmup + s)
        tok += t
        secs += sec
    v = tok / secs
    cores = blas_threads()
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(cfg, wl, world), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"1 user per step ({cfg['n_layers']}-layer fwd+bwd, float64 "
                                       f"NumPy oracle), {args.steps} steps, {tok} tokens"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def run_mtgr(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2505_18654_b200 as m

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dt = torch.bfloat16
    wl = workload(cfg, rank, world, m.balance_lpt, args.balance)
    users = wl["users"]
    ts = np.concatenate(wl["ts"]) if len(users) else np.zeros(0, np.int64)
    Ls = wl["L"][users]
    X = np.concatenate([synth.gen_user_x(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
    dZ = np.concatenate([synth.gen_user_dz(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
    jb = m.JaggedBatch.build(wl["seg"], ts, dev, users=users)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"], cfg.get("rab_buckets", 0),
                     mask_mode=cfg.get("mask_mode", "dynamic"), post_mlp_layers=cfg.get("post_mlp_layers", 1))
    Ps = [m.params_to_device(synth.gen_layer_params(cfg, li, cfg.get("rab_buckets", 0)), dt, dev) for li in range(cfg["n_layers"])]
    stack = m.HstuStack(lc, Ps, dt, dev)
    stack.bind(jb)
    x_dev = torch.from_numpy(X).to(dev, dt)
    dz_dev = torch.from_numpy(dZ).to(dev, dt)
    from paper_2505_18654_b200.dp import GradAggregator
    agg = GradAggregator(wl["B_g"])  # per-layer bucket all-reduce (NCCL) + 1/B_global

    head_state = {}
    if args.head:  # candidate head + two-task BCE on the encoder output
        lab = np.concatenate([synth.gen_user_labels(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
        hp = m.head_params_to_device(synth.gen_head_params(cfg), dt, dev)
        hshapes = {"w_a": tuple(hp["w_a"].shape), "b_a": (hp["w_a"].shape[0],), "w_b": tuple(hp["w_b"].shape), "b_b": (2,)}
        al = lambda n: (n + 63) // 64 * 64  # 256-byte aligned views (16-byte TMA pointers)
        hflat = torch.zeros(sum(al(int(np.prod(v))) for v in hshapes.values()), dtype=torch.float32, device=dev)
        hviews, off = {}, 0
        for kk, shp in hshapes.items():  # the head's gradient bucket (all-reduced + scaled with the layers')
            hviews[kk] = hflat[off:off + int(np.prod(shp))].view(*shp)
            off += al(hviews[kk].numel())
        head_state = dict(params=hp, labels=torch.from_numpy(lab).to(dev), flat=hflat, views=hviews,
                          ws=None, K=int(jb.host["n_cand"].sum()))

    tok = {}
    if args.tokens:  # Eq.4 token construction from synthetic per-type feature embeddings
        k = synth.token_widths(cfg)
        per_user = [synth.gen_user_features(cfg, int(u), wl["seg"][u]) for u in users]
        feats = {t: torch.from_numpy(np.concatenate([f[t] for f in per_user] + [np.zeros((0, k[t]), np.float32)]))
                 .to(dev, dt) for t in synth.TOKEN_TYPES}
        emb = m.TokenEmbed(cfg["d"], k, m.TokenEmbed.params_to_device(synth.gen_token_params(cfg), dt, dev), dt, dev)
        emb.bind(jb, wl["seg"][users])
        tshapes = emb.grad_shapes()
        al = lambda n: (n + 63) // 64 * 64
        tflat = torch.zeros(sum(al(int(np.prod(v))) for q in tshapes.values() for v in q.values()),
                            dtype=torch.float32, device=dev)
        tviews, off = {}, 0
        for t_, q in tshapes.items():  # the token MLPs' gradient bucket
            for kk, shp in q.items():
                tviews.setdefault(t_, {})[kk] = tflat[off:off + int(np.prod(shp))].view(*shp)
                off += al(int(np.prod(shp)))
        tok = dict(emb=emb, feats=feats, flat=tflat, views=tviews)

    full = {}
    if args.full_model:
        ids = [synth.gen_user_feature_ids(cfg, int(u), wl["seg"][u]) for u in users]
        lab = np.concatenate([synth.gen_user_labels(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
        uids = np.concatenate([i["u"].reshape(-1) for i in ids])
        iids = np.concatenate([np.concatenate([i[t].reshape(-1) for i in ids]) for t in "src"])
        model = m.MTGRModel(cfg, lc, [synth.gen_layer_params(cfg, li, cfg.get("rab_buckets", 0)) for li in range(cfg["n_layers"])],
                            synth.gen_token_params(cfg), synth.gen_head_params(cfg), synth.token_widths(cfg),
                            synth.EMB_DIM, dt, dev, cap_user=1 << 20, cap_item=1 << 23,
                            n_users_global=wl["B_g"])
        model.bind(jb, wl["seg"][users])
        stack = model.stack
        full = dict(model=model, uids=torch.from_numpy(uids).to(dev), iids=torch.from_numpy(iids).to(dev),
                    labels=torch.from_numpy(lab).to(dev), n_ids=len(uids) + len(iids), t=[0])

    def step(xin=x_dev, dzin=dz_dev):
        if args.full_model:
            full["t"][0] += 1
            # layer buckets + the head/token bucket all-reduced and scaled inside the step
            full["model"].step(full["uids"], full["iids"], full["labels"], now=full["t"][0], aggregator=agg)
            return
        if args.tokens:
            xin = tok["emb"].forward(tok["feats"]).contiguous()
        z = stack.forward(xin)
        flats = [stack.grad_flat]
        if args.head:
            _, loss, dzin, hg = m.head_fwd_bwd(jb, head_state["params"], z, head_state["labels"],
                                               grads_out=head_state["views"])
            agg.on_layer_done(-1, head_state["flat"])
            flats.append(head_state["flat"])
        dx = stack.backward(dzin, on_layer_done=agg.on_layer_done)
        if args.tokens:
            tok["emb"].backward(dx, grads_out=tok["views"])
            agg.on_layer_done(-1, tok["flat"])
            flats.append(tok["flat"])
        agg.finish(*flats)

    def barrier():
        if world > 1:
            dist.barrier()

    # the clock sampler runs from the warm-up on (nvidia-smi takes a while to start); only its
    # samples inside the timed region are reported
    sampler = ClockSampler(gpu_id_for(torch, dev))
    sampler.start()
    sampler.wait_first()
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    barrier()

    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m.prof_reset()
    m.prof_enable(True)
    launches0 = m.launch_count()
    barrier()
    torch.cuda.synchronize()
    t_host0 = time.monotonic()
    ev0.record(st)
    for _ in range(args.steps):
        step()
    ev1.record(st)
    torch.cuda.synchronize()
    t_host1 = time.monotonic()
    barrier()
    launches = m.launch_count() - launches0
    m.prof_enable(False)
    sampler.mark(t_host0, t_host1)
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    kern = m.prof_query()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    tok_global = wl["tokens_global"]
    value = tok_global * args.steps / (ms_max / 1000.0)
    flops_rank = step_flops(cfg, wl["tokens"], wl["pairs"])
    pk, pk_kind = peaks()

    # per-kernel roofline from the live CUDA-event timings
    algo = kernel_algorithmic(cfg, wl["tokens"], wl["pairs"])
    kernels = {}
    for name, (n, tot) in kern.items():
        e = {"launches_per_step": n / args.steps, "ms_per_step": tot / args.steps,
             "share": tot / ms if ms > 0 else None}
        if name in algo:
            bound, work = algo[name]
            per_launch = work / max(n / args.steps, 1)
            avg_s = tot / n / 1000.0
            if bound == "tensor":
                e.update(bound="tensor", achieved_tflops=per_launch / avg_s / 1e12,
                         frac=per_launch / avg_s / 1e12 / pk["bf16_tflops_sustained"],
                         frac_burst=per_launch / avg_s / 1e12 / pk["bf16_tflops"])
            else:
                e.update(bound="hbm", achieved_gbs=per_launch / avg_s / 1e9,
                         frac=per_launch / avg_s / 1e9 / pk["hbm_gbs"])
        kernels[name] = e
    dom = max((k for k in kernels if "bound" in kernels[k]), key=lambda k: kernels[k]["ms_per_step"], default=None)
    roof = None
    if dom:
        e = kernels[dom]
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(cfg["name"], {}).get(dom)
        if e["bound"] == "tensor":
            roof = {"kernel": dom, "bound": "tensor", "achieved": e["achieved_tflops"],
                    "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s", "frac": e["frac"],
                    "traffic": traffic, "peak_source": f"{pk_kind} bf16_tflops_sustained (kernel timed inside a long step)",
                    "peak_burst": pk["bf16_tflops"], "frac_burst": e["frac_burst"]}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": e["achieved_gbs"], "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": e["frac"], "traffic": traffic, "peak_source": f"{pk_kind} hbm_gbs"}

    # ---------------------------------------------------------------- e2e through host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, torch, dist, m, stack, jb, X, dZ, ts, wl, world, dev, step)

    large = None
    if world == 1 and not args.no_large_attn and cfg["name"] != "large":
        large = run_large_attention(torch, m, dev, pk)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tok, secs = time_oracle(cfg, wl, args.cpu_users)
        cpu = {"value": tok / secs, "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
               "sample": f"{args.cpu_users} users of the rank-0 batch ({tok} tokens), "
                         f"{cfg['n_layers']}-layer fwd+bwd, float64 NumPy oracle, {secs:.1f} s"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded generator synth/, random-init weights)",
                "config": workload_desc(cfg, wl, world),
                # algorithmic FLOP/s / the burst bf16 peak (cuBLAS 8192^3 best of 10);
                # the sustained-peak fraction beside it
                "pct_bf16_peak": flops_rank * world * args.steps / (ms_max / 1000.0) / 1e12
                                 / (pk["bf16_tflops"] * world),
                "pct_bf16_peak_sustained": flops_rank * world * args.steps / (ms_max / 1000.0) / 1e12
                                           / (pk["bf16_tflops_sustained"] * world),
                "algorithmic_tflops_per_gpu": flops_rank * args.steps / (ms_max / 1000.0) / 1e12,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": int(launches), "kernels": kernels, "impl": "mtgr"}
        if large is not None:
            line["large_attention"] = large
        if args.full_model:
            line["config"]["step"] = ("full training step: sharded hash-embedding lookup (two-stage unique, "
                                      "all-to-all) -> Eq.4 tokens -> stack -> head/BCE -> backward -> sparse SGD")
            line["config"]["sparse_ids_per_rank"] = full["n_ids"]
        if args.tokens:
            line["config"]["tokens"] = "Eq.4 token construction (U embeddings + per-type MLPs) fwd/bwd in the step"
        if args.head:
            line["config"]["step"] = "stack fwd + candidate head/BCE + stack bwd (dZ from the head)"
            line["config"]["candidates_per_rank"] = head_state["K"]
        print(json.dumps(line), flush=True)


def run_large_attention(torch, m, dev, pk, layers=1, steps=3, warmup=2):
    """The north-star check in the default bench line (BASELINE.json: >= 50 % bf16 tensor-pipe
    on the attention at the MTGR-large shape): one MTGR-large layer (d=768, 3 heads, 32 users x
    4484 tokens: n_U 32, n_S 4096, n_r 100, K 256) forward + backward, CUDA-event timed per
    kernel; algorithmic TFLOP/s of each attention kernel against the burst and sustained bf16
    peaks, and the time-weighted attention fraction (all attention FLOPs / all attention time)."""
    cfg = synth.config("large", n_layers=layers)
    wl = workload(cfg, 0, 1, m.balance_lpt)
    users = wl["users"]
    ts = np.concatenate(wl["ts"])
    Ls = wl["L"][users]
    dt = torch.bfloat16
    X = np.concatenate([synth.gen_user_x(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
    dZ = np.concatenate([synth.gen_user_dz(cfg, int(u), int(l)) for u, l in zip(users, Ls)])
    jb = m.JaggedBatch.build(wl["seg"], ts, dev, users=users)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    stack = m.HstuStack(lc, [m.params_to_device(synth.gen_layer_params(cfg, li, cfg.get("rab_buckets", 0)), dt, dev)
                             for li in range(layers)], dt, dev)
    stack.bind(jb)
    x = torch.from_numpy(X).to(dev, dt)
    dz = torch.from_numpy(dZ).to(dev, dt)
    for _ in range(warmup):
        stack.forward(x)
        stack.backward(dz)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m.prof_reset()
    m.prof_enable(True)
    ev0.record(st)
    for _ in range(steps):
        stack.forward(x)
        stack.backward(dz)
    ev1.record(st)
    torch.cuda.synchronize()
    m.prof_enable(False)
    ms = ev0.elapsed_time(ev1) / steps
    kern = m.prof_query()
    algo = kernel_algorithmic(cfg, wl["tokens"], wl["pairs"])
    out, a_fl, a_ms = {}, 0.0, 0.0
    for name, (n, tot) in kern.items():
        if not name.startswith("attn_") or name not in algo:
            continue
        work = algo[name][1]
        tf = work * steps / (tot / 1000.0) / 1e12
        out[name] = {"ms_per_layer": tot / steps / layers, "achieved_tflops": tf,
                     "frac_burst": tf / pk["bf16_tflops"], "frac_sustained": tf / pk["bf16_tflops_sustained"]}
        a_fl += work * steps
        a_ms += tot
    flops = step_flops(cfg, wl["tokens"], wl["pairs"])
    del stack, x, dz
    torch.cuda.empty_cache()
    return {"workload": "MTGR-large shape: 1 layer, d=768, 3 heads (d_h=256), 32 users x 4484 tokens "
                        "(n_U 32, n_S 4096, n_r 100, K 256), T=143488, fwd+bwd, bf16",
            "ms_per_layer_step": ms / layers,
            "layer_pct_bf16_peak": flops / (ms / 1000.0) / 1e12 / pk["bf16_tflops"],
            "attention_kernels": out,
            "attention_time_weighted_frac_burst": (a_fl / (a_ms / 1000.0) / 1e12 / pk["bf16_tflops"]) if a_ms else None,
            "attention_share_of_layer": a_ms / steps / ms if ms else None,
            "note": "algorithmic FLOPs only (SURVEY §8(d): masked pairs and the backward's S recompute "
                    "excluded); tensor-pipe utilisation from ncu is in profiles/"}


def run_e2e(args, torch, dist, m, stack, jb, X, dZ, ts, wl, world, dev, step):
    """Same metric through the public API with HOST inputs: every step copies X, dZ and the
    jagged metadata from pinned host memory (copy stream, double-buffered: batch t+1 is copied
    while batch t computes) and reads the gradients back to host."""
    dt = torch.bfloat16
    h_x = torch.from_numpy(X).to(dt).pin_memory()
    h_dz = torch.from_numpy(dZ).to(dt).pin_memory()
    h_meta = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in
              (jb.host["offsets"], jb.host["n_static"], jb.host["n_rt"], jb.host["n_cand"],
               jb.host["group_id"], ts)]
    d_x = [torch.empty_like(h_x, device=dev) for _ in range(2)]
    d_dz = [torch.empty_like(h_dz, device=dev) for _ in range(2)]
    d_meta = [[torch.empty_like(t, device=dev) for t in h_meta] for _ in range(2)]
    h_grad = torch.empty(stack.grad_flat.numel(), dtype=torch.float32).pin_memory()
    h2d = h_x.numel() * 2 + h_dz.numel() * 2 + sum(t.numel() * t.element_size() for t in h_meta)
    d2h = h_grad.numel() * 4
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def enqueue_copy(i):
        b = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(free[b])
            d_x[b].copy_(h_x, non_blocking=True)
            d_dz[b].copy_(h_dz, non_blocking=True)
            for dd, hh in zip(d_meta[b], h_meta):
                dd.copy_(hh, non_blocking=True)
            ready[b].record(copy)

    def run(n):
        for b in range(2):
            free[b].record(comp)
        enqueue_copy(0)
        for i in range(n):
            b = i % 2
            if i + 1 < n:
                enqueue_copy(i + 1)
            comp.wait_event(ready[b])
            jb_i = m.JaggedBatch(d_meta[b][0], d_meta[b][1], d_meta[b][2], d_meta[b][3],
                                 d_meta[b][4], d_meta[b][5], None, jb.num_users, jb.total_tokens,
                                 jb.max_len, jb.host)
            stack.bind(jb_i)
            step(d_x[b], d_dz[b])
            free[b].record(comp)
            h_grad.copy_(stack.grad_flat, non_blocking=True)
        torch.cuda.synchronize()

    run(max(args.warmup, 1))
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(comp)
    run(args.steps)
    ev1.record(comp)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    stack.bind(jb)
    return {"value": wl["tokens_global"] * args.steps / (ms / 1000.0), "unit": "tokens/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms / args.steps,
            "note": "pinned-host inputs copied every step on a copy stream (double-buffered), grads read back"}


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1; rank 0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl != "reference":
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(env_world) if env_world is not None else args.gpus
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if env_world is not None and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        sys.exit(2)
    cfg = synth.config(args.config, mask_mode=args.mask, post_mlp_layers=args.post_mlp, rab_buckets=args.rab)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        # communicator INIT lines (nranks, transport) go to stderr; stdout carries one JSON line.
        # Set before torch is imported: NCCL reads its debug settings once, at its first call.
        # The GPU image presets NCCL_DEBUG=VERSION (version line only): raised to INFO here
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local_rank))
    try:
        run_mtgr(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
