"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on identical seeded
inputs.  Bit-exact for masks / offsets; max|g-o|/max|o| <= 1e-4 (fp32 path) and <= 2e-2 (bf16
path) for floating point (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m
from tests.fixtures import load_fig2c, make_batch, rel_err

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _dt(cfg):
    return torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16


def _t(a, dev, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)


# ------------------------------------------------------------------ masks (bit-exact)

def test_mask_dense_fig2c(dev):
    n_s, n_r, n_c, ts, golden = load_fig2c()
    jb = m.JaggedBatch.build(np.array([[2, 2, n_r, n_c]]), ts, dev)
    got = m.mask_dense(jb, 0).cpu().numpy()
    np.testing.assert_array_equal(got, golden)


def test_mask_dense_random_users(dev):
    rng = np.random.default_rng(0)
    seg = rng.integers(0, 30, (12, 4)).astype(np.int32)
    seg[3] = 0
    seg[4] = [0, 0, 5, 3]
    L = seg.sum(1)
    ts = np.concatenate([np.concatenate([np.zeros(seg[u, 0] + seg[u, 1], np.int64),
                                         rng.integers(0, 9, seg[u, 2] + seg[u, 3])]) for u in range(12)])
    jb = m.JaggedBatch.build(seg, ts, dev)
    h = oracle.build_jagged(seg)
    for u in range(12):
        if L[u] == 0:
            continue
        a, b = h["offsets"][u], h["offsets"][u + 1]
        ref = oracle.mask_dense(int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u]), ts[a:b])
        np.testing.assert_array_equal(m.mask_dense(jb, u).cpu().numpy(), ref)


def test_validate_jagged(dev):
    cfg, seg, ts, X, dZ, P = make_batch("toy")
    jb = m.JaggedBatch.build(seg, ts, dev)
    m.validate_jagged(jb, 4)
    jb.n_cand[1] += 1
    with pytest.raises(m.MtgrError) as e:
        m.validate_jagged(jb, 4)
    assert e.value.status == 9


# ------------------------------------------------------------------ GLN

@pytest.mark.parametrize("name", ["toy", "parity"])
def test_gln_fwd_bwd(dev, name):
    cfg, seg, ts, X, dZ, P = make_batch(name)
    dt = _dt(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(cfg["d"], cfg["H"])
    g = torch.from_numpy(P["gamma1"]).to(dev)
    b = torch.from_numpy(P["beta1"]).to(dev)
    x = _t(X, dev, dt)
    y, mean, rstd = m.gln_fwd(lc, jb, x, g, b)
    gid = jb.host["group_id"]
    yo, mo, ro = oracle.gln_fwd(X, gid, P["gamma1"], P["beta1"])
    assert rel_err(y.float().cpu().numpy(), yo) <= TOL[dt]
    assert rel_err(mean.cpu().numpy(), mo) <= 1e-5 + (dt == torch.bfloat16) * 1e-3
    assert rel_err(rstd.cpu().numpy(), ro) <= 1e-4
    dy = _t(dZ, dev, dt)
    dx, dg, db = m.gln_bwd(lc, jb, dy, x, mean, rstd, g)
    dxo, dgo, dbo = oracle.gln_bwd(dZ, X, gid, mo, ro, P["gamma1"])
    assert rel_err(dx.float().cpu().numpy(), dxo) <= TOL[dt]
    assert rel_err(dg.cpu().numpy(), dgo) <= TOL[dt]
    assert rel_err(db.cpu().numpy(), dbo) <= TOL[dt]


# ------------------------------------------------------------------ attention

def _attn_case(name, seed=0):
    cfg, seg, ts, X, dZ, P = make_batch(name)
    rng = np.random.default_rng(seed)
    T, d = X.shape
    import synth
    r = lambda *s: synth.round_bf16(rng.standard_normal(s).astype(np.float32)) if cfg["dtype"] == "bf16" \
        else rng.standard_normal(s).astype(np.float32)
    qkvu = r(T, 4 * d) * 0.5 + 0.3   # shift: SiLU-like positive mean
    dO = r(T, d)
    return cfg, seg, ts, qkvu, dO


@pytest.fixture(params=["kv", "stored", "stored_fused_dk", "recompute"])
def bwd_path(request, monkeypatch):
    """The tensor-core backward paths (MTGR_ATTN_BWD): kv (default) = the coupled dK/dV kernel
    stores dS^T, then the dQ GEMM; stored = the score kernel stores P^T / dS^T, then three GEMMs;
    fused_dk = the DK kernel writes the scores; MTGR_ATTN_RECOMPUTE=1 = the kernels that recompute
    the scores (the path used when the score scratch would not fit)."""
    monkeypatch.delenv("MTGR_ATTN_RECOMPUTE", raising=False)
    monkeypatch.delenv("MTGR_ATTN_FUSED_DK", raising=False)
    monkeypatch.setenv("MTGR_ATTN_BWD", {"kv": "kv", "stored": "stored", "stored_fused_dk": "fused_dk",
                                         "recompute": "kv"}[request.param])
    if request.param == "recompute":
        monkeypatch.setenv("MTGR_ATTN_RECOMPUTE", "1")
    return request.param


@pytest.mark.parametrize("mask", ["dynamic", "causal", "full"])
@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_attention_fwd_bwd(dev, name, bwd_path, mask):
    cfg, seg, ts, qkvu, dO = _attn_case(name)
    dt = _dt(cfg)
    d, H = cfg["d"], cfg["H"]
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(d, H, mask_mode=mask)
    a = _t(qkvu, dev, dt)
    o, y = m.attn_fwd(lc, jb, a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d, u=a[:, 3 * d:])
    dq, dk, dv, _ = m.attn_bwd(lc, jb, _t(dO, dev, dt), a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d)
    h = oracle.build_jagged(seg)
    got = dict(o=o, y=y, dq=dq, dk=dk, dv=dv)
    got = {k: v.float().cpu().numpy() for k, v in got.items()}
    ref = {k: np.zeros_like(got[k], dtype=np.float64) for k in got}
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        q, k, v, uu = (qkvu[s:e, i * d:(i + 1) * d].astype(np.float64) for i in range(4))
        nu = 1.0 / (e - s)
        oo, S, M = oracle.attn_fwd_user(q, k, v, ns, nr, nc, ts[s:e], H, nu, mask_mode=mask)
        ref["o"][s:e] = oo
        ref["y"][s:e] = oo * uu
        dq_, dk_, dv_, _ = oracle.attn_bwd_user(dO[s:e].astype(np.float64), q, k, v, S, M, H, nu)
        ref["dq"][s:e], ref["dk"][s:e], ref["dv"][s:e] = dq_, dk_, dv_
    for key in got:
        e = rel_err(got[key], ref[key])
        assert e <= TOL[dt], (key, e)


# ------------------------------------------------------------------ full layer

def _run_layer(dev, cfg, seg, ts, X, dZ, P, n_layers=1, Ps=None, inv_norm=None):
    dt = _dt(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev, inv_norm=inv_norm)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"], cfg.get("rab_buckets", 0),
                     mask_mode=cfg.get("mask_mode", "dynamic"), post_mlp_layers=cfg.get("post_mlp_layers", 1))
    Ps = Ps or [P]
    stack = m.HstuStack(lc, [m.params_to_device(p, dt, dev) for p in Ps], dt, dev)
    stack.bind(jb)
    z = stack.forward(_t(X, dev, dt)).float().cpu().numpy()
    dx = stack.backward(_t(dZ, dev, dt)).float().cpu().numpy()
    grads = [{k: v.cpu().numpy() for k, v in g.items()} for g in stack.grads]
    return z, dx, grads


def _oracle_stack(cfg, seg, ts, X, dZ, Ps, inv_norm=None, users=None):
    h = oracle.build_jagged(seg)
    ocfg = dict(d=cfg["d"], H=cfg["H"], mask_mode=cfg.get("mask_mode", "dynamic"),
                post_mlp_layers=cfg.get("post_mlp_layers", 1))
    Z = np.full(X.shape, np.nan)
    dX = np.full(X.shape, np.nan)
    tot = [None] * len(Ps)
    for u in range(len(seg)):
        if users is not None and u not in users:
            continue
        s, e = h["offsets"][u], h["offsets"][u + 1]
        nu = None if inv_norm is None else float(inv_norm[u])
        args = (h["group_id"][s:e], int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u]), ts[s:e])
        z, caches = oracle.stack_fwd_user(X[s:e], *args, Ps, ocfg, nu)
        dx, gs = oracle.stack_bwd_user(dZ[s:e], caches, Ps, ocfg)
        Z[s:e], dX[s:e] = z, dx
        for li, g in enumerate(gs):
            if tot[li] is None:
                tot[li] = {k: v.copy() for k, v in g.items()}
            else:
                for k in g:
                    tot[li][k] += g[k]
    return Z, dX, tot


def _compare(z, dx, grads, Z, dX, G, tol, rows=None):
    sel = slice(None) if rows is None else rows
    errs = {"Z": rel_err(z[sel], Z[sel]), "dX": rel_err(dx[sel], dX[sel])}
    if G is not None:
        for li, g in enumerate(G):
            for k in g:
                errs[f"L{li}.d{k}"] = rel_err(grads[li][k], g[k])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, bad
    return errs


@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_layer_fwd_bwd(dev, name, bwd_path):
    cfg, seg, ts, X, dZ, P = make_batch(name)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    print(_compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)]))


@pytest.mark.parametrize("mask", ["causal", "full"])
@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_layer_ablation_masks(dev, name, bwd_path, mask):
    """Table 4's "w/o dynamic mask" ablation under both readings: the plain causal mask
     and full attention with candidates isolated."""
    cfg, seg, ts, X, dZ, P = make_batch(name, mask_mode=mask)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    print(_compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)]))


@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_layer_post_mlp2(dev, name):
    """f3 variant: the 2-layer post-gate MLP (Linear-SiLU-Linear) through the C ABI."""
    cfg, seg, ts, X, dZ, P = make_batch(name, post_mlp_layers=2)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    errs = _compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)])
    assert "L0.dW3" in errs and "L0.db3" in errs
    print(errs)


@pytest.mark.parametrize("name", ["toy", "parity"])
def test_layer_edge_cases(dev, name, bwd_path):
    """Empty users, users without static / real-time / candidate segments, single tokens."""
    seg = np.array([[0, 0, 0, 0], [0, 0, 3, 2], [4, 3, 0, 0], [1, 0, 0, 1], [0, 0, 0, 1],
                    [2, 130, 0, 5], [0, 0, 0, 0], [3, 1, 140, 0], [1, 1, 1, 1]], np.int32)
    cfg, seg, ts, X, dZ, P = make_batch(name, seg=seg)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    _compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)])


def test_layer_rab_fp32(dev):
    """Optional relative-time bias (R#4) on the fp32 path."""
    cfg, seg, ts, X, dZ, P = make_batch("toy", rab_buckets=16)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    _compare(z, dx, grads, Z, dX, G, 1e-4)


@pytest.mark.parametrize("mask", ["dynamic", "causal", "full"])
@pytest.mark.parametrize("name", ["parity", "parity768"])
def test_attention_rab_bf16(dev, name, bwd_path, mask):
    """The rab term (R#4) on the tcgen05 kernels: o, y, dq, dk, dv and drab against the oracle
    (drab: the kv / stored paths sum the stored dS^T, the recompute path inside the DQ kernel).
    rab_w ~ 8 N(0, 1) over 16 buckets (the synthetic time gaps, seconds within the real-time hour
    up to months to the static items, fill buckets 0..11 and the capped 15), large enough that a
    wrong bucket, sign or missing term moves the outputs far beyond the tolerance (checked: the
    outputs without rab differ from the oracle's by > 10x the tolerance; 0.42 on "parity")."""
    cfg, seg, ts, qkvu, dO = _attn_case(name)
    dt = _dt(cfg)
    d, H, NB = cfg["d"], cfg["H"], 16
    rab = (8.0 * np.random.default_rng(5).standard_normal((H, NB))).astype(np.float32)
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(d, H, rab_buckets=NB, mask_mode=mask)
    a = _t(qkvu, dev, dt)
    rw = torch.from_numpy(rab).to(dev)
    o, y = m.attn_fwd(lc, jb, a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d, u=a[:, 3 * d:], rab_w=rw)
    dq, dk, dv, drab = m.attn_bwd(lc, jb, _t(dO, dev, dt), a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d, rab_w=rw)
    h = oracle.build_jagged(seg)
    got = dict(o=o, y=y, dq=dq, dk=dk, dv=dv)
    got = {k: v.float().cpu().numpy() for k, v in got.items()}
    ref = {k: np.zeros_like(got[k], dtype=np.float64) for k in got}
    ref_norab = np.zeros_like(got["o"], dtype=np.float64)
    rdrab = np.zeros((H, NB))
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        if e == s:
            continue
        ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        q, k, v, uu = (qkvu[s:e, i * d:(i + 1) * d].astype(np.float64) for i in range(4))
        nu = 1.0 / (e - s)
        oo, S, M = oracle.attn_fwd_user(q, k, v, ns, nr, nc, ts[s:e], H, nu, rab_w=rab.astype(np.float64),
                                        mask_mode=mask)
        ref["o"][s:e] = oo
        ref["y"][s:e] = oo * uu
        ref_norab[s:e] = oracle.attn_fwd_user(q, k, v, ns, nr, nc, ts[s:e], H, nu, mask_mode=mask)[0]
        dq_, dk_, dv_, dr = oracle.attn_bwd_user(dO[s:e].astype(np.float64), q, k, v, S, M, H, nu, ts[s:e],
                                                 rab.astype(np.float64))
        ref["dq"][s:e], ref["dk"][s:e], ref["dv"][s:e] = dq_, dk_, dv_
        rdrab += dr
    assert rel_err(ref_norab, ref["o"]) > 10 * TOL[dt]  # the rab term is not negligible here
    errs = {k: rel_err(got[k], ref[k]) for k in got}
    errs["drab"] = rel_err(drab.cpu().numpy(), rdrab)
    bad = {k: e for k, e in errs.items() if not e <= TOL[dt]}
    assert not bad, (bad, errs)


@pytest.mark.parametrize("name", ["parity", "parity768"])
def test_layer_rab_bf16(dev, name, bwd_path):
    """A whole bf16 layer with rab on (R#4): z, dX and every parameter gradient incl. d rab_w."""
    cfg, seg, ts, X, dZ, P = make_batch(name, rab_buckets=16)
    P = dict(P, rab_w=(10.0 * P["rab_w"]).astype(np.float32))  # ~N(0, 1): a visible term
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    errs = _compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)])
    assert "L0.drab_w" in errs
    print(errs)


def test_stack_three_layers_bf16(dev):
    import synth
    cfg, seg, ts, X, dZ, P = make_batch("parity")
    Ps = [synth.gen_layer_params(cfg, li) for li in range(3)]
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P, Ps=Ps)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, Ps)
    _compare(z, dx, grads, Z, dX, G, 2e-2)


@pytest.mark.parametrize("name", ["toy", "parity"])
def test_candidate_leakage_bitwise(dev, name):
    """Perturbing other candidates (values only: layout unchanged) leaves a candidate's output
    bitwise identical on the GPU."""
    cfg, seg, ts, X, dZ, P = make_batch(name)
    z1, _, _ = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    h = oracle.build_jagged(seg)
    u = 0
    s = int(h["offsets"][u]); ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
    j = s + ns + nr  # first candidate of user 0
    X2 = X.copy()
    X2[j + 1:s + ns + nr + nc] += 3.0
    z2, _, _ = _run_layer(dev, cfg, seg, ts, X2, dZ, P)
    np.testing.assert_array_equal(z1[j], z2[j])


def test_removal_invariance_fixed_norm(dev):
    """With a caller-fixed 1/N (inv_norm), dropping other candidates leaves a candidate's output
    unchanged up to summation order."""
    cfg, seg, ts, X, dZ, P = make_batch("toy")
    inv = np.full(len(seg), 1 / 64.0, np.float32)
    z1, _, _ = _run_layer(dev, cfg, seg, ts, X, dZ, P, inv_norm=inv)
    h = oracle.build_jagged(seg)
    s, ns, nr, nc = int(h["offsets"][0]), int(h["n_static"][0]), int(h["n_rt"][0]), int(h["n_cand"][0])
    seg2 = seg.copy(); seg2[0, 3] = 1
    keep = np.r_[0:s + ns + nr + 1, s + ns + nr + nc:len(X)]
    z2, _, _ = _run_layer(dev, cfg, seg2, ts[keep], X[keep], dZ[keep], P, inv_norm=inv)
    np.testing.assert_allclose(z2[s + ns + nr], z1[s + ns + nr], rtol=0, atol=1e-5)


# ------------------------------------------------------------------ GEMM utility

@pytest.mark.parametrize("akm,bkm", [(1, 1), (1, 0), (0, 0), (0, 1)])
@pytest.mark.parametrize("c_f32", [0, 1])
def test_gemm_bf16(dev, akm, bkm, c_f32):
    import synth
    rng = np.random.default_rng(akm * 2 + bkm)
    M, N, K = 304, 520, 200 if c_f32 == 0 else 1000  # ragged tails, 16-byte rows
    A = synth.round_bf16(rng.standard_normal((M, K)).astype(np.float32))
    B = synth.round_bf16(rng.standard_normal((N, K)).astype(np.float32))
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    At = A if akm else np.ascontiguousarray(A.T)
    Bt = B if bkm else np.ascontiguousarray(B.T)
    C = m.gemm(_t(At, dev, torch.bfloat16), _t(Bt, dev, torch.bfloat16), M, N, K,
               At.shape[1], akm, Bt.shape[1], bkm, c_f32=bool(c_f32))
    assert rel_err(C.float().cpu().numpy(), ref) <= (1e-5 if c_f32 else 8e-3)


def test_scale(dev):
    g = torch.arange(1000, dtype=torch.float32, device=dev)
    m.scale_(g, 0.25)
    np.testing.assert_array_equal(g.cpu().numpy(), np.arange(1000, dtype=np.float32) * 0.25)


@pytest.mark.parametrize("name", ["toy", "parity"])
def test_layer_single_shared_ln(dev, name):
    """Table 4 "w/o GLN": one LayerNorm for every token is the layer with
    num_groups = 1 and every group id 0 (the group-affine parameters collapse to one row)."""
    cfg, seg, ts, X, dZ, P = make_batch(name)
    P1 = dict(P)
    for k in ("gamma1", "beta1", "gamma2", "beta2"):
        P1[k] = np.ascontiguousarray(P[k][:1])
    dt = _dt(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    jb.group_id.zero_()
    lc = m.layer_cfg(cfg["d"], cfg["H"], 1)
    stack = m.HstuStack(lc, [m.params_to_device(P1, dt, dev)], dt, dev)
    stack.bind(jb)
    z = stack.forward(_t(X, dev, dt)).float().cpu().numpy()
    dx = stack.backward(_t(dZ, dev, dt)).float().cpu().numpy()
    grads = [{k: v.cpu().numpy() for k, v in g.items()} for g in stack.grads]
    h = oracle.build_jagged(seg)
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    Z, dX = np.zeros(X.shape), np.zeros(X.shape)
    G = None
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        gid0 = np.zeros(e - s, dtype=np.uint8)
        args = (gid0, int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u]), ts[s:e])
        zz, caches = oracle.stack_fwd_user(X[s:e], *args, [P1], ocfg)
        dd, gs = oracle.stack_bwd_user(dZ[s:e], caches, [P1], ocfg)
        Z[s:e], dX[s:e] = zz, dd
        G = [{k: v.copy() for k, v in gs[0].items()}] if G is None else [{k: G[0][k] + gs[0][k] for k in G[0]}]
    _compare(z, dx, grads, Z, dX, G, TOL[dt])


@pytest.mark.parametrize("name", ["parity", "parity768"])
def test_layer_register_row_copy(dev, name, monkeypatch):
    """The row operands moved into TMEM through the softmax warps' registers (MTGR_ROW_CP=0,
    MTGR_SC_CP=0) instead of tcgen05.cp: same results."""
    monkeypatch.setenv("MTGR_ROW_CP", "0")
    monkeypatch.setenv("MTGR_SC_CP", "0")
    monkeypatch.setenv("MTGR_ATTN_BWD", "stored")
    cfg, seg, ts, X, dZ, P = make_batch(name)
    z, dx, grads = _run_layer(dev, cfg, seg, ts, X, dZ, P)
    Z, dX, G = _oracle_stack(cfg, seg, ts, X, dZ, [P])
    _compare(z, dx, grads, Z, dX, G, TOL[_dt(cfg)])
