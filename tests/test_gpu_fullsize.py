"""Parity at the benchmark's full size and launch configuration (BASELINE configs[1] 'small':
3 layers, d=512, 256 users, T~264k, bf16) on outputs the oracle can compute user by user, plus
properties that hold at any size; and the MTGR-large shape (d=768, L=4484) on one layer."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m
import synth
from tests.fixtures import p999_rel_err, rel_err, report

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _batch(cfg, users=None):
    seg = synth.gen_segments(cfg)
    users = np.arange(len(seg)) if users is None else np.asarray(users)
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, int(u), seg[u]) for u in users])
    X = np.concatenate([synth.gen_user_x(cfg, int(u), int(L[u])) for u in users])
    dZ = np.concatenate([synth.gen_user_dz(cfg, int(u), int(L[u])) for u in users])
    return seg, users, ts, X, dZ


def _run(dev, cfg, seg, users, ts, X, dZ, Ps):
    jb = m.JaggedBatch.build(seg, ts, dev, users=users.astype(np.int32))
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"], cfg.get("rab_buckets", 0))
    stack = m.HstuStack(lc, [m.params_to_device(P, torch.bfloat16, dev) for P in Ps], torch.bfloat16, dev)
    stack.bind(jb)
    z = stack.forward(torch.from_numpy(X).to(dev, torch.bfloat16))
    dx = stack.backward(torch.from_numpy(dZ).to(dev, torch.bfloat16))
    torch.cuda.synchronize()
    return jb, z.float().cpu().numpy(), dx.float().cpu().numpy(), [g["_flat"].clone() for g in stack.grads]


def _oracle_user(cfg, seg, u, ts_u, X_u, dZ_u, Ps):
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    gid = oracle.build_jagged(seg[u:u + 1])["group_id"]
    nU, nS, nR, K = (int(v) for v in seg[u])
    z, caches = oracle.stack_fwd_user(X_u, gid, nU + nS, nR, K, ts_u, Ps, ocfg)
    dx, _ = oracle.stack_bwd_user(dZ_u, caches, Ps, ocfg)
    return z, dx


def test_small_config_sampled_users_and_additivity(dev):
    cfg = synth.config("small")
    Ps = [synth.gen_layer_params(cfg, li) for li in range(cfg["n_layers"])]
    seg, users, ts, X, dZ = _batch(cfg)
    jb, z, dx, grads = _run(dev, cfg, seg, users, ts, X, dZ, Ps)
    off = jb.host["offsets"]
    L = seg.astype(np.int64).sum(1)
    for u in (0, int(np.argmax(L)), int(np.argmin(L))):
        a, b = int(off[u]), int(off[u + 1])
        zo, dxo = _oracle_user(cfg, seg, u, ts[a:b], X[a:b], dZ[a:b], Ps)
        assert rel_err(z[a:b], zo) <= 2e-2, ("Z", u)
        assert rel_err(dx[a:b], dxo) <= 2e-2, ("dX", u)
    # parameter gradients are sums over users: full batch == first half + second half (the
    # per-user arithmetic is identical; only fp32 summation order differs: split-K bounds,
    # atomics), so 1e-4 leaves room for that and nothing else
    h = len(seg) // 2
    parts = []
    for us_ in (np.arange(h), np.arange(h, len(seg))):
        s2, u2, ts2, X2, dZ2 = _batch(cfg, us_)
        parts.append(_run(dev, cfg, s2, u2, ts2, X2, dZ2, Ps)[3])
    for li in range(cfg["n_layers"]):
        full = grads[li].cpu().numpy()
        summed = (parts[0][li] + parts[1][li]).cpu().numpy()
        assert rel_err(full, summed) <= 1e-4, li


def _oracle_grads(cfg, seg, off, ts, X, dZ, Ps, users):
    """Oracle Z, dX over `users` and the parameter gradients summed over them (layer 0)."""
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    Z = np.zeros(X.shape); dX = np.zeros(X.shape)
    tot = None
    gids = oracle.build_jagged(seg)["group_id"]
    goff = oracle.build_jagged(seg)["offsets"]
    for u in users:
        a, b = int(off[u]), int(off[u + 1])
        nU, nS, nR, K = (int(v) for v in seg[u])
        gid = gids[int(goff[u]):int(goff[u + 1])]
        z, caches = oracle.stack_fwd_user(X[a:b], gid, nU + nS, nR, K, ts[a:b], Ps, ocfg)
        dx, gs = oracle.stack_bwd_user(dZ[a:b], caches, Ps, ocfg)
        Z[a:b], dX[a:b] = z, dx
        if tot is None:
            tot = {k: v.copy() for k, v in gs[0].items()}
        else:
            for k in tot:
                tot[k] += gs[0][k]
    return Z, dX, tot


def _grad_views(cfg, flat, dev):
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"], cfg.get("rab_buckets", 0))
    g = m.alloc_grads(lc, dev, flat.to(dev))
    return {k: v.cpu().numpy() for k, v in g.items() if not k.startswith("_")}


def _check_all(name, cfg, z, dx, gflat, Z, dX, G, dev, rows=None, tol=None):
    sel = slice(None) if rows is None else rows
    rep = {"Z": (rel_err(z[sel], Z[sel]), p999_rel_err(z[sel], Z[sel])),
           "dX": (rel_err(dx[sel], dX[sel]), p999_rel_err(dx[sel], dX[sel]))}
    gv = _grad_views(cfg, gflat, dev)
    for k in G:
        rep["d" + k] = (rel_err(gv[k], G[k]), p999_rel_err(gv[k], G[k]))
    report(name, rep)
    print(name, rep)
    # max-normalised <= 2e-2 (north_star); elementwise p99.9 <= 0.5 (measured <= 0.24)
    tol = tol or {}
    bad = {k: v for k, v in rep.items() if not (v[0] <= tol.get(k, 2e-2) and v[1] <= 0.5)}
    assert not bad, bad


def test_small_one_layer_all_users_gradients(dev):
    """One `small` layer over the whole bench batch (256 users, T ~ 264k, the bench's launch
    configuration: split-K weight gradients over K = T, the score kernel + stored-score GEMMs):
    Z, dX and every parameter gradient (W1, b1, W2, b2, gamma/beta 1-2) against the oracle."""
    cfg = synth.config("small")
    Ps = [synth.gen_layer_params(cfg, 0)]
    seg, users, ts, X, dZ = _batch(cfg)
    jb, z, dx, grads = _run(dev, cfg, seg, users, ts, X, dZ, Ps)
    off = jb.host["offsets"]
    Z, dX, G = _oracle_grads(cfg, seg, off, ts, X, dZ, Ps, range(len(seg)))
    _check_all("small_one_layer_all_users", cfg, z, dx, grads[0], Z, dX, G, dev)


def test_small_one_layer_all_users_rab(dev):
    """The same full bench batch with the optional relative-time bias (R#4, 16 buckets, rab_w ~
    N(0, 1)): the RAB kernel instantiations of the forward and the coupled backward, the d rab_w
    pass over the stored dS^T and the candidate diagonals, at the bench's launch configuration:
    Z, dX and every parameter gradient including d rab_w against the oracle."""
    cfg = synth.config("small", rab_buckets=16)
    P = synth.gen_layer_params(cfg, 0, 16)
    P["rab_w"] = (10.0 * P["rab_w"]).astype(np.float32)
    seg, users, ts, X, dZ = _batch(cfg)
    jb, z, dx, grads = _run(dev, cfg, seg, users, ts, X, dZ, [P])
    off = jb.host["offsets"]
    Z, dX, G = _oracle_grads(cfg, seg, off, ts, X, dZ, [P], range(len(seg)))
    assert "rab_w" in G
    # d rab_w: 5e-2 here (R#25: bf16 rounding of the attention's inputs against the
    # float64 oracle, amplified by the cancelling 1e8-term bucket sums); the kernels' own d rab_w
    # is held to 2e-2 by test_small_attention_rab_all_users with identical bf16 inputs
    _check_all("small_one_layer_all_users_rab", cfg, z, dx, grads[0], Z, dX, G, dev, tol={"drab_w": 5e-2})


def test_small_attention_rab_all_users(dev):
    """The attention alone over the full bench batch with rab (R#4, 16 buckets, rab_w ~ 8 N(0,1))
    on bf16-exact inputs the oracle sees exactly (q, k, v, u, dO drawn in bf16; scores spread
    over SiLU's curved range): o, y, dq, dk, dv and d rab_w at the bench's launch configuration.
    d rab_w sums ~10^8 visible pairs per head and bucket; with the oracle fed the same bf16
    inputs, what remains is the kernels' own arithmetic (fp32 accumulation, tanh.approx, the
    fp16 SiLU' hand-over, the bf16 dS^T the sum reads back)."""
    cfg = synth.config("small")
    seg = synth.gen_segments(cfg)
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
    jb = m.JaggedBatch.build(seg, ts, dev)
    d, H, NB = cfg["d"], cfg["H"], 16
    T = int(L.sum())
    rng = np.random.default_rng(3)
    qkvu = synth.round_bf16((rng.standard_normal((T, 4 * d)) * 0.12).astype(np.float32))
    dO = synth.round_bf16(rng.standard_normal((T, d)).astype(np.float32))
    rab = (8.0 * np.random.default_rng(5).standard_normal((H, NB))).astype(np.float32)
    lc = m.layer_cfg(d, H, rab_buckets=NB)
    a_ = torch.from_numpy(qkvu).to(dev, torch.bfloat16)
    rw = torch.from_numpy(rab).to(dev)
    o, y = m.attn_fwd(lc, jb, a_[:, 0:], a_[:, d:], a_[:, 2 * d:], 4 * d, u=a_[:, 3 * d:], rab_w=rw)
    dq, dk, dv, drab = m.attn_bwd(lc, jb, torch.from_numpy(dO).to(dev, torch.bfloat16), a_[:, 0:], a_[:, d:],
                                  a_[:, 2 * d:], 4 * d, rab_w=rw)
    got = {k: v.float().cpu().numpy() for k, v in dict(o=o, y=y, dq=dq, dk=dk, dv=dv).items()}
    ref = {k: np.zeros_like(v, dtype=np.float64) for k, v in got.items()}
    rdrab = np.zeros((H, NB))
    h = oracle.build_jagged(seg)
    for u in range(len(seg)):
        s0, e0 = h["offsets"][u], h["offsets"][u + 1]
        ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        q, k, v, uu = (qkvu[s0:e0, i * d:(i + 1) * d].astype(np.float64) for i in range(4))
        nu = 1.0 / (e0 - s0)
        oo, S, M = oracle.attn_fwd_user(q, k, v, ns, nr, nc, ts[s0:e0], H, nu, rab_w=rab.astype(np.float64))
        ref["o"][s0:e0], ref["y"][s0:e0] = oo, oo * uu
        dq_, dk_, dv_, dr = oracle.attn_bwd_user(dO[s0:e0].astype(np.float64), q, k, v, S, M, H, nu, ts[s0:e0],
                                                 rab.astype(np.float64))
        ref["dq"][s0:e0], ref["dk"][s0:e0], ref["dv"][s0:e0] = dq_, dk_, dv_
        rdrab += dr
    rep = {k: (rel_err(got[k], ref[k]), p999_rel_err(got[k], ref[k])) for k in got}
    rep["drab"] = (rel_err(drab.cpu().numpy(), rdrab), p999_rel_err(drab.cpu().numpy(), rdrab))
    report("small_attention_rab_all_users", rep)
    print(rep)
    bad = {k: v for k, v in rep.items() if not (v[0] <= 2e-2 and v[1] <= 0.5)}
    assert not bad, bad


def test_large_shape_one_layer(dev):
    """MTGR-large shape (d=768, 3 heads, L = 4484: n_static 4128, 100 real-time, 256 candidates),
    two users (mean length >= 2048: the fused DK kernel writes the scores): Z, dX and every
    parameter gradient against the oracle."""
    cfg = synth.config("large", users=2, n_layers=1)
    Ps = [synth.gen_layer_params(cfg, 0)]
    seg, users, ts, X, dZ = _batch(cfg)
    jb, z, dx, grads = _run(dev, cfg, seg, users, ts, X, dZ, Ps)
    off = jb.host["offsets"]
    Z, dX, G = _oracle_grads(cfg, seg, off, ts, X, dZ, Ps, range(len(seg)))
    _check_all("large_two_users", cfg, z, dx, grads[0], Z, dX, G, dev)


def test_attention_bitwise_deterministic(dev):
    """The attention kernels own their outputs (no atomics on the public path), so repeated runs
    on identical inputs must agree bit for bit.  The bench batch mixes long items with short and
    tile-less (candidate-only) pairs, the pattern under which a skipped barrier phase once let a
    producer refill the shared epilogue tile early (dk rows of the following item differed
    between runs)."""
    cfg = synth.config("small")
    seg = synth.gen_segments(cfg)
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    T, d = jb.total_tokens, cfg["d"]
    g = torch.Generator(device="cpu").manual_seed(11)
    qkvu = (torch.randn(T, 4 * d, generator=g) * 0.5).to(dev, torch.bfloat16)
    dO = torch.randn(T, d, generator=g).to(dev, torch.bfloat16)
    pre = torch.randn(T, 4 * d, generator=g).to(dev, torch.bfloat16)
    q, k, v = qkvu[:, :d], qkvu[:, d:2 * d], qkvu[:, 2 * d:3 * d]
    ref = None
    for _ in range(6):
        o, _ = m.attn_fwd(lc, jb, q, k, v, 4 * d)
        dq, dk, dv, _ = m.attn_bwd(lc, jb, dO, q, k, v, 4 * d, silu_pre=pre)
        torch.cuda.synchronize()
        cur = [t.clone() for t in (o, dq, dk, dv)]
        if ref is None:
            ref = cur
            continue
        for name, a_, b_ in zip(("o", "dq", "dk", "dv"), ref, cur):
            assert torch.equal(a_, b_), name
