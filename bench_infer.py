#!/usr/bin/env python
"""Inference fast-path benchmark (BASELINE configs[4]: MTGR-large forward, one
user per request with 500 candidates sharing the compressed user prefix, latency and throughput
on 1 x B200).

Requests are synthetic (`synth` config `infer`: 15 layers, d=768, 3 heads, n_U=32, n_S=4096,
n_r=100).  Each shape is captured once into a CUDA graph (`InferenceSession`) and replayed;
latency is the device time of one replay (CUDA events on the launching stream, after warm-up),
throughput batches B users into one replay.  Prints one JSON line per measurement:
  * latency vs K (candidates per request) at B=1 — sub-linear in K: the prefix dominates and
    candidates are queries only (no candidate keys are ever loaded);
  * throughput (requests/s, tokens/s) at B users per replay.
Latency lines carry the distribution over --iters requests (each request = its features copied
from pinned host memory into the session's static buffer + one replay, timed alone with CUDA
events on the stream): p50, p99, mean.
usage: python bench_infer.py [--ks 64,125,250,500] [--batches 1,8,32] [--iters 100]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_2505_18654_b200 as m  # noqa: E402
import synth  # noqa: E402
from paper_2505_18654_b200.infer import InferenceSession  # noqa: E402


def measure(cfg, seg, Ps_dev, lc, iters, dev):
    """Returns (per-request device ms list, tokens): each request copies its features from pinned
    host memory into the static buffer and replays the captured forward; requests are timed one
    by one (CUDA events around copy + replay on the launching stream)."""
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
    L = seg.astype(np.int64).sum(1)
    X = np.concatenate([synth.gen_user_x(cfg, u, int(L[u])) for u in range(len(seg))])
    sess = InferenceSession(lc, Ps_dev, torch.bfloat16, dev, seg, ts)
    hx = torch.from_numpy(X).to(torch.bfloat16).pin_memory()
    sess.set_request(hx.to(dev))
    sess.capture()
    for _ in range(3):
        sess.set_request(hx)
        sess.run()
    st = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize(dev)
    for e0, e1 in ev:
        e0.record(st)
        sess.set_request(hx)
        sess.run()
        e1.record(st)
    torch.cuda.synchronize(dev)
    return [e0.elapsed_time(e1) for e0, e1 in ev], int(L.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="64,125,250,500")
    ap.add_argument("--batches", default="1,8,32")
    ap.add_argument("--iters", type=int, default=100)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = synth.config("infer")
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    Ps_dev = [m.params_to_device(synth.gen_layer_params(cfg, li), torch.bfloat16, dev)
              for li in range(cfg["n_layers"])]
    prefix = (32, 4096, 100)
    base = dict(data="synthetic (seeded generator synth/, random-init weights)", dtype="bf16",
                n_gpus=1, timing="per request: CUDA events around the pinned-host feature copy + the "
                                  "CUDA-graph replay, after 3 warm-up requests")
    for k in [int(v) for v in args.ks.split(",")]:
        seg = np.array([[*prefix, k]], dtype=np.int32)
        lat, T = measure(cfg, seg, Ps_dev, lc, args.iters, dev)
        print(json.dumps(dict(metric="inference latency per request", value=float(np.percentile(lat, 50)), unit="ms",
                              p50_ms=float(np.percentile(lat, 50)), p99_ms=float(np.percentile(lat, 99)),
                              mean_ms=float(np.mean(lat)), requests=len(lat),
                              higher_is_better=False, config=dict(
                                  workload="MTGR-large forward (15 layers, d=768, 3 heads), 1 user per request",
                                  n_U=32, n_S=4096, n_r=100, K=k, tokens=T), **base)), flush=True)
    for b in [int(v) for v in args.batches.split(",")]:
        seg = np.array([[*prefix, 500]] * b, dtype=np.int32)
        lat, T = measure(cfg, seg, Ps_dev, lc, max(20, args.iters // 5), dev)
        ms = float(np.mean(lat))
        print(json.dumps(dict(metric="inference throughput", value=b / (ms / 1e3), unit="requests/s",
                              higher_is_better=True, ms_per_replay=ms, tokens_per_s=T / (ms / 1e3),
                              candidates_per_s=500 * b / (ms / 1e3), config=dict(
                                  workload="MTGR-large forward (15 layers, d=768, 3 heads), B users per replay",
                                  users_per_replay=b, n_U=32, n_S=4096, n_r=100, K=500, tokens=T), **base)),
              flush=True)


if __name__ == "__main__":
    main()
