"""Shared helpers for the tests: golden-fixture parsing and small seeded cases."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_fig2c():
    """Parse tests/golden/fig2c_mask.txt -> (n_s, n_r, n_c, ts int64 [L], mask uint8 [L][L])."""
    ts = None
    rows = []
    n_s = n_r = n_c = None
    with open(os.path.join(GOLDEN, "fig2c_mask.txt")) as f:
        for line in f:
            s = line.strip()
            if s.startswith("# layout:"):
                kv = dict(t.split("=") for t in s[len("# layout:"):].split())
                n_s, n_r, n_c = int(kv["n_static"]), int(kv["n_rt"]), int(kv["n_cand"])
            elif s.startswith("# ts:"):
                ts = np.array([int(t) for t in s[len("# ts:"):].split()], dtype=np.int64)
            elif s and not s.startswith("#"):
                rows.append([1 if t == "1" else 0 for t in s.split()[1:]])
    return n_s, n_r, n_c, ts, np.array(rows, dtype=np.uint8)


def tiny_user(rng, n_s, n_r, n_c, d, G=4, ts_span=50):
    """Random tiny user: x [L][d], gid [L], ts [L] (ties likely among rt/candidates)."""
    L = n_s + n_r + n_c
    x = rng.standard_normal((L, d))
    gid = np.array([0] * (n_s // 2) + [1] * (n_s - n_s // 2) + [2] * n_r + [3] * n_c)
    gid = np.minimum(gid, G - 1)
    ts = np.concatenate([np.zeros(n_s, np.int64),
                         np.sort(rng.integers(0, ts_span, n_r))[::-1],
                         np.sort(rng.integers(0, ts_span, n_c))[::-1]]).astype(np.int64)
    return x, gid, ts


def tiny_params(rng, d, H, G=4, rab_buckets=0, scale=1.0):
    p = {
        "W1": rng.standard_normal((4 * d, d)) * scale / np.sqrt(d),
        "b1": rng.standard_normal(4 * d) * 0.1,
        "W2": rng.standard_normal((d, d)) * scale / np.sqrt(d),
        "b2": rng.standard_normal(d) * 0.1,
        "gamma1": 1 + 0.2 * rng.standard_normal((G, d)),
        "beta1": 0.2 * rng.standard_normal((G, d)),
        "gamma2": 1 + 0.2 * rng.standard_normal((G, d)),
        "beta2": 0.2 * rng.standard_normal((G, d)),
    }
    if rab_buckets:
        p["rab_w"] = 0.3 * rng.standard_normal((H, rab_buckets))
    return p


def make_batch(cfg_name, n_users=None, seg=None, **over):
    """Seeded batch from synth: (cfg, seg [B][4], ts [T], X [T][d], dZ [T][d], params)."""
    import synth
    cfg = synth.config(cfg_name, **over)
    if seg is None:
        seg = synth.gen_segments(cfg, n_users)
    seg = np.asarray(seg, dtype=np.int32)
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))] + [np.zeros(0, np.int64)])
    X = np.concatenate([synth.gen_user_x(cfg, u, int(L[u])) for u in range(len(seg))] +
                       [np.zeros((0, cfg["d"]), np.float32)])
    dZ = np.concatenate([synth.gen_user_dz(cfg, u, int(L[u])) for u in range(len(seg))] +
                        [np.zeros((0, cfg["d"]), np.float32)])
    P = synth.gen_layer_params(cfg, 0, cfg.get("rab_buckets", 0))
    return cfg, seg, ts, X, dZ, P


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def p999_rel_err(got, ref, floor=1e-2):
    """99.9th percentile of the elementwise relative error |g - o| / max(|o|, floor * max|o|)
    (reported beside the max-normalised error; the floor keeps entries that are
    ~0 by cancellation from dominating)."""
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    if ref.size == 0:
        return 0.0
    den = np.maximum(np.abs(ref), floor * max(np.abs(ref).max(), 1e-30))
    return float(np.percentile(np.abs(got - ref) / den, 99.9))


def report(name, payload):
    """Append a JSON line to $MTGR_REPORT_DIR/parity_report.jsonl (GPU runs keep the numbers the
    tests print as evidence); no-op when the variable is unset."""
    import json
    d = os.environ.get("MTGR_REPORT_DIR")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "parity_report.jsonl"), "a") as f:
        f.write(json.dumps({"test": name, **payload}) + "\n")
