"""Seeded generators for MTGR-shaped jagged workloads.

Recipe (also stated in DESIGN.md §3):

* One user = segments (n_U profile, n_S lifelong behaviour, n_r real-time,
  K candidates) in that order (Eq.3-4).
* Timestamps (int64 seconds), request epoch T0 = 1_700_000_000:
  profile 0; lifelong items T0 - 86400*U[1,180]; real-time T0 - U{0..3599};
  candidates (request time) T0 - U{0..3599}; each segment sorted recent->past
  (P:274).  The toy config quantises rt/candidate times to 300 s to force ties.
* Values: X ~ N(0,1); W1, W2 ~ N(0, 1/d); biases ~ N(0, 0.02^2);
  gamma ~ 1 + N(0, 0.1^2), beta ~ N(0, 0.1^2) (distinct per group);
  rab_w ~ N(0, 0.1^2); dZ ~ N(0,1).  For bf16 workloads every value is rounded
  to the nearest bf16 (RNE) so both sides see identical inputs.
* Every stream is a PCG64 seeded by (config seed, stream id, index), so a rank
  can generate only its own users and still agree with every other rank.

No arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np

T0 = 1_700_000_000

# stream ids
_S_SEG, _S_TS, _S_X, _S_DZ, _S_PARAM, _S_LABEL, _S_HEAD, _S_FEAT, _S_TOK, _S_IDS = 11, 12, 13, 14, 15, 16, 17, 18, 19, 20

CONFIGS = {
    # name: layers, d_model, heads, users (per rank), segment recipe, dtype, seed
    "toy": dict(n_layers=1, d=64, H=2, users=4, seed=0, dtype="f32", groups=4,
                nU=("fixed", 8), nS=("uniform", 0, 32), nR=("uniform", 0, 8),
                K=("fixed", 4), ts_quantum=300),
    # small parity case spanning several 128-row tiles with ragged tails (bf16 path)
    "parity": dict(n_layers=1, d=512, H=2, users=4, seed=5, dtype="bf16", groups=4,
                   nU=("fixed", 32), nS=("uniform", 100, 420), nR=("uniform", 0, 100),
                   K=("uniform", 1, 150), ts_quantum=1),
    "parity768": dict(n_layers=1, d=768, H=3, users=3, seed=6, dtype="bf16", groups=4,
                      nU=("fixed", 32), nS=("uniform", 100, 300), nR=("uniform", 0, 100),
                      K=("uniform", 1, 100), ts_quantum=1),
    "small": dict(n_layers=3, d=512, H=2, users=256, seed=1, dtype="bf16", groups=4,
                  nU=("fixed", 32), nS=("uniform", 768, 1000), nR=("uniform", 0, 100),
                  K=("fixed", 64), ts_quantum=1),
    "middle": dict(n_layers=5, d=768, H=3, users=96, seed=2, dtype="bf16", groups=4,
                   nU=("fixed", 32), nS=("pareto", 128, 1.1, 2048), nR=("fixed", 100),
                   K=("fixed", 64), ts_quantum=1),
    "large": dict(n_layers=15, d=768, H=3, users=32, seed=3, dtype="bf16", groups=4,
                  nU=("fixed", 32), nS=("fixed", 4096), nR=("fixed", 100),
                  K=("fixed", 256), ts_quantum=1),
    "large_skew": dict(n_layers=15, d=768, H=3, users=96, seed=7, dtype="bf16", groups=4,
                       nU=("fixed", 32), nS=("pareto", 256, 1.1, 4096), nR=("fixed", 100),
                       K=("fixed", 256), ts_quantum=1),
    "infer": dict(n_layers=15, d=768, H=3, users=1, seed=4, dtype="bf16", groups=4,
                  nU=("fixed", 32), nS=("fixed", 4096), nR=("fixed", 100),
                  K=("fixed", 500), ts_quantum=1),
}


def config(name: str, **over) -> dict:
    c = dict(CONFIGS[name])
    c.update(over)
    c["name"] = name
    return c


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (round-half-to-even), returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def _draw(spec, rng, n):
    kind = spec[0]
    if kind == "fixed":
        return np.full(n, spec[1], dtype=np.int64)
    if kind == "uniform":
        return rng.integers(spec[1], spec[2], size=n, endpoint=True)
    if kind == "pareto":  # truncated Pareto: min(cap, floor(scale * u^(-1/alpha)))
        scale, alpha, cap = spec[1], spec[2], spec[3]
        u = 1.0 - rng.random(n)  # (0, 1]
        return np.minimum(cap, np.floor(scale * u ** (-1.0 / alpha))).astype(np.int64)
    raise ValueError(kind)


def gen_segments(cfg: dict, n_users: int | None = None) -> np.ndarray:
    """Segment lengths [B][4] int32 = (n_U, n_S, n_r, K) per user of the global batch."""
    B = cfg["users"] if n_users is None else n_users
    rng = _rng(cfg["seed"], _S_SEG)
    cols = [_draw(cfg[k], rng, B) for k in ("nU", "nS", "nR", "K")]
    return np.stack(cols, axis=1).astype(np.int32)


def gen_user_ts(cfg: dict, user: int, seg) -> np.ndarray:
    """Per-token timestamps (int64 s) of one user, tokens in U,S,R,C order."""
    nU, nS, nR, K = (int(v) for v in seg)
    rng = _rng(cfg["seed"], _S_TS, user)
    q = int(cfg.get("ts_quantum", 1))
    s = np.sort(T0 - 86400 * rng.integers(1, 180, size=nS, endpoint=True))[::-1]
    r = np.sort(T0 - rng.integers(0, 3599, size=nR, endpoint=True))[::-1]
    c = np.sort(T0 - rng.integers(0, 3599, size=K, endpoint=True))[::-1]
    if q > 1:
        r = (r // q) * q
        c = (c // q) * q
    return np.concatenate([np.zeros(nU, np.int64), s, r, c]).astype(np.int64)


def _vals(cfg, a):
    a = a.astype(np.float32)
    return round_bf16(a) if cfg["dtype"] == "bf16" else a


def gen_user_x(cfg: dict, user: int, n_tokens: int) -> np.ndarray:
    """Layer-0 input tokens X of one user, [n_tokens][d] float32 (bf16-exact for bf16 configs)."""
    rng = _rng(cfg["seed"], _S_X, user)
    return _vals(cfg, rng.standard_normal((n_tokens, cfg["d"]), dtype=np.float32))


def gen_user_dz(cfg: dict, user: int, n_tokens: int) -> np.ndarray:
    """Upstream gradient dZ of the last layer for one user, [n_tokens][d]."""
    rng = _rng(cfg["seed"], _S_DZ, user)
    return _vals(cfg, rng.standard_normal((n_tokens, cfg["d"]), dtype=np.float32))


def gen_layer_params(cfg: dict, layer: int, rab_buckets: int = 0) -> dict:
    """Random-init parameters of one HSTU layer (float32; W1/W2 bf16-exact for bf16 configs).

    W1 [4d][d] rows ordered Q,K,V,U; W2 [d][d]; b1 [4d]; b2 [d];
    gamma1/beta1/gamma2/beta2 [G][d]; rab_w [H][NB] when rab_buckets > 0.
    """
    d, G, H = cfg["d"], cfg["groups"], cfg["H"]
    rng = _rng(cfg["seed"], _S_PARAM, layer)
    sd = 1.0 / np.sqrt(d)
    p = {
        "W1": _vals(cfg, rng.standard_normal((4 * d, d)) * sd),
        "b1": (rng.standard_normal(4 * d) * 0.02).astype(np.float32),
        "W2": _vals(cfg, rng.standard_normal((d, d)) * sd),
        "b2": (rng.standard_normal(d) * 0.02).astype(np.float32),
        "gamma1": (1.0 + 0.1 * rng.standard_normal((G, d))).astype(np.float32),
        "beta1": (0.1 * rng.standard_normal((G, d))).astype(np.float32),
        "gamma2": (1.0 + 0.1 * rng.standard_normal((G, d))).astype(np.float32),
        "beta2": (0.1 * rng.standard_normal((G, d))).astype(np.float32),
    }
    if rab_buckets:
        p["rab_w"] = (0.1 * rng.standard_normal((H, rab_buckets))).astype(np.float32)
    if cfg.get("post_mlp_layers", 1) == 2:  # second post-gate Linear (its own stream)
        r3 = _rng(cfg["seed"], _S_PARAM, layer, 3)
        p["W3"] = _vals(cfg, r3.standard_normal((d, d)) * sd)
        p["b3"] = (r3.standard_normal(d) * 0.02).astype(np.float32)
    return p


def gen_user_labels(cfg: dict, user: int, n_tokens: int, p_click: float = 0.3,
                    p_buy: float = 0.3) -> np.ndarray:
    """Per-token uint8 labels (only candidate rows are used): bit 0 click ~ Bernoulli(p_click),
    bit 1 purchase ~ Bernoulli(p_buy) given a click (purchase implies click)."""
    rng = _rng(cfg["seed"], _S_LABEL, user)
    click = rng.random(n_tokens) < p_click
    buy = click & (rng.random(n_tokens) < p_buy)
    return (click.astype(np.uint8) | (buy.astype(np.uint8) << 1)).astype(np.uint8)


def gen_head_params(cfg: dict, d_hidden: int | None = None) -> dict:
    """Random-init candidate head (float32; w_a bf16-exact for bf16 configs):
    w_a [dh][d], b_a [dh], w_b [2][dh], b_b [2]; dh = d/2 by default."""
    d = cfg["d"]
    dh = d_hidden or d // 2
    rng = _rng(cfg["seed"], _S_HEAD)
    return {
        "w_a": _vals(cfg, rng.standard_normal((dh, d)) / np.sqrt(d)),
        "b_a": (rng.standard_normal(dh) * 0.02).astype(np.float32),
        "w_b": (rng.standard_normal((2, dh)) / np.sqrt(dh)).astype(np.float32),
        "b_b": (rng.standard_normal(2) * 0.02).astype(np.float32),
    }


TOKEN_TYPES = ("u", "s", "r", "c")


def token_widths(cfg: dict) -> dict:
    """Concatenated feature-embedding widths per item type: a token of k features uses
    embeddings of ~d/k each, so the concatenation is ~d wide; varied per type here so the
    tests exercise distinct shapes."""
    d = cfg["d"]
    return {"u": d, "s": d, "r": max(8, (d // 2) // 8 * 8), "c": max(8, (3 * d // 4) // 8 * 8)}


def gen_user_features(cfg: dict, user: int, seg) -> dict:
    """Per-type feature rows of one user (N(0,1); bf16-exact for bf16 configs):
    u [n_U][d] (the profile tokens' embeddings), s [n_S][k_s], r [n_r][k_r], c [K][k_c]."""
    rng = _rng(cfg["seed"], _S_FEAT, user)
    k = token_widths(cfg)
    n = dict(zip(TOKEN_TYPES, (int(v) for v in seg)))
    return {t: _vals(cfg, rng.standard_normal((n[t], k[t]))) for t in TOKEN_TYPES}


def gen_token_params(cfg: dict) -> dict:
    """Per item type (s, r, c): w1 [d][k_t] ~ N(0, 1/k_t), b1 [d], w2 [d][d] ~ N(0, 1/d), b2 [d]."""
    d = cfg["d"]
    k = token_widths(cfg)
    rng = _rng(cfg["seed"], _S_TOK)
    out = {}
    for t in ("s", "r", "c"):
        out[t] = {"w1": _vals(cfg, rng.standard_normal((d, k[t])) / np.sqrt(k[t])),
                  "b1": (rng.standard_normal(d) * 0.02).astype(np.float32),
                  "w2": _vals(cfg, rng.standard_normal((d, d)) / np.sqrt(d)),
                  "b2": (rng.standard_normal(d) * 0.02).astype(np.float32)}
    return out


EMB_DIM = 16  # item-feature embedding width (a token of k features has k ~ d / EMB_DIM)


def features_per_token(cfg: dict) -> dict:
    """Feature count per token type: U tokens are one d-wide feature each; item tokens
    concatenate k_t / EMB_DIM feature embeddings (token_widths)."""
    k = token_widths(cfg)
    return {"u": 1, "s": k["s"] // EMB_DIM, "r": k["r"] // EMB_DIM, "c": k["c"] // EMB_DIM}


def gen_user_feature_ids(cfg: dict, user: int, seg) -> dict:
    """Sparse feature IDs of one user's tokens, int64 [n_t][F_t] per type: feature slot f of a
    token carries (f << 40) | value, values Zipf(1.2)-distributed over a 2^24 vocabulary per slot
    (long-tail popularity), so IDs of different slots never collide; U IDs live in slots >= 4096."""
    rng = _rng(cfg["seed"], _S_IDS, user)
    F = features_per_token(cfg)
    n = dict(zip(TOKEN_TYPES, (int(v) for v in seg)))
    out = {}
    for t in TOKEN_TYPES:
        vals = (rng.zipf(1.2, (n[t], F[t])) % (1 << 24)).astype(np.int64)
        base = 4096 if t == "u" else 0
        slots = (np.arange(F[t], dtype=np.int64) + base + {"u": 0, "s": 0, "r": 64, "c": 128}[t]) << 40
        out[t] = vals + slots[None, :]
    return out
