"""Bit-exact mask probes and leakage tests through the tensor-core attention kernels.

The float parity tests compare values under a 2e-2 max-normalised tolerance, which a single
wrong mask entry can hide.  Here the inputs are built so that every output element equals one
mask entry times a known constant:

  probe "o / dV":  q = k = 1/16 (s_ij = 1 for every pair), v = dO = one-hot rows
                   -> o_i[c]  = nu silu(1) m_{i, j(c)}      (the forward's key predicate)
                   -> dV_j[c] = nu silu(1) m_{i(c), j}      (P^T of the backward)
  probe "dK":      q = one-hot rows, k = 1 (s = 1 where q is set), v = dO = 1/16 (dP = 1)
                   -> dK_j[c] = nu silu'(1) m_{i(c), j}    (dS^T of the backward)
  probe "dQ":      q = 1, k = one-hot rows, v = dO = 1/16
                   -> dQ_i[c] = nu silu'(1) m_{i, j(c)}    (dS of the backward)

where the one-hot row of user-local token t is e_{t mod 256} in head t // 256 (zero in the other
heads), so one call covers every (reader, read) pair of users up to 256 H tokens.  The nonzero
pattern of each output must equal the oracle's mask (P:335-338 with DESIGN.md R#8-R#12; the
causal mask of P:324-326 for mask_mode causal) element for element, and each value must match
the oracle.  The users put n_static and n_static + n_rt at every tile edge the kernels use
(64-column tiles, 32-column warp halves, 128-row CTAs, 256-row pairs), with tied and unsorted
real-time / candidate timestamps.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m
from tests.fixtures import make_batch, p999_rel_err, rel_err, report

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


# (n_U, n_S, n_r, K): n_static = n_U + n_S and kv_end = n_static + n_r on tile edges
PROBE_SEGS = [
    (0, 0, 5, 3), (1, 0, 0, 1), (32, 32, 63, 10), (32, 95, 1, 5), (32, 96, 128, 64),
    (1, 254, 2, 3), (32, 224, 200, 40), (2, 0, 300, 20), (16, 300, 129, 60), (10, 500, 0, 0),
    (0, 0, 400, 0), (5, 5, 5, 300), (0, 0, 0, 0), (32, 31, 1, 1), (64, 64, 64, 64),
    (1, 0, 255, 256), (0, 1, 31, 33), (0, 63, 1, 0), (0, 0, 129, 127),
]
PROBE_SEGS_768 = PROBE_SEGS + [(32, 480, 256, 0), (1, 511, 130, 100), (0, 0, 700, 68), (200, 300, 200, 68)]


def _probe_batch(H, seed=0):
    """Segments (L <= 256 H) and timestamps: real-time and candidate times drawn from 12 values
    (ties everywhere) in random order (neither sorted nor monotone)."""
    segs = PROBE_SEGS if H == 2 else PROBE_SEGS_768
    seg = np.array([s for s in segs if sum(s) <= 256 * H], np.int32)
    rng = np.random.default_rng(seed)
    ts = []
    for nU, nS, nR, K in seg:
        ts.append(np.concatenate([np.zeros(nU, np.int64), 1000 + rng.integers(0, 50, nS),
                                  5000 + rng.integers(0, 12, nR), 5000 + rng.integers(0, 12, K)]))
    return seg, np.concatenate(ts).astype(np.int64)


def _onehot(seg, H, d):
    """[T][d]: user-local token t -> 1 at column (t // 256) * 256 + t % 256 (= t for d_h 256)."""
    T = int(seg.sum())
    a = np.zeros((T, d), np.float32)
    off = 0
    for L in seg.sum(1):
        a[off + np.arange(L), np.arange(L)] = 1.0
        off += L
    return a


def _probe_inputs(kind, seg, H):
    d = 256 * H
    T = int(seg.sum())
    one_hot = _onehot(seg, H, d)
    c16 = np.full((T, d), 1 / 16, np.float32)
    ones = np.ones((T, d), np.float32)
    if kind == "o_dv":
        q, k, v, dO = c16, c16, one_hot, one_hot
    elif kind == "dk":
        q, k, v, dO = one_hot, ones, c16, c16
    else:  # "dq"
        q, k, v, dO = ones, one_hot, c16, c16
    return q, k, v, dO


PROBED = {"o_dv": ("o", "dv"), "dk": ("dk",), "dq": ("dq",)}


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


def _attn_oracle(seg, ts, q, k, v, dO, H, mask):
    h = oracle.build_jagged(seg)
    T, d = q.shape
    ref = {n: np.zeros((T, d)) for n in ("o", "dq", "dk", "dv")}
    for u in range(len(seg)):
        s, e = int(h["offsets"][u]), int(h["offsets"][u + 1])
        if e == s:
            continue
        ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        f = lambda a: a[s:e].astype(np.float64)
        o, S, M = oracle.attn_fwd_user(f(q), f(k), f(v), ns, nr, nc, ts[s:e], H, 1.0 / (e - s), mask_mode=mask)
        dq, dk, dv, _ = oracle.attn_bwd_user(f(dO), f(q), f(k), f(v), S, M, H, 1.0 / (e - s))
        ref["o"][s:e], ref["dq"][s:e], ref["dk"][s:e], ref["dv"][s:e] = o, dq, dk, dv
    return ref


def _attn_gpu(dev, seg, ts, q, k, v, dO, H, mask):
    d = q.shape[1]
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(d, H, mask_mode=mask)
    T = q.shape[0]
    qkvu = np.concatenate([q, k, v, np.ones((T, d), np.float32)], axis=1)
    a = torch.from_numpy(qkvu).to(dev, torch.bfloat16)
    o, _ = m.attn_fwd(lc, jb, a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d)
    dq, dk, dv, _ = m.attn_bwd(lc, jb, torch.from_numpy(dO).to(dev, torch.bfloat16),
                               a[:, 0:], a[:, d:], a[:, 2 * d:], 4 * d)
    torch.cuda.synchronize()
    return {n: t.float().cpu().numpy() for n, t in dict(o=o, dq=dq, dk=dk, dv=dv).items()}


@pytest.mark.parametrize("mask", list(m.MASK_MODES))
@pytest.mark.parametrize("kind", ["o_dv", "dk", "dq"])
@pytest.mark.parametrize("H", [2, 3])
def test_mask_probe_bit_exact(dev, bwd_path, mask, kind, H):
    seg, ts = _probe_batch(H)
    q, k, v, dO = _probe_inputs(kind, seg, H)
    got = _attn_gpu(dev, seg, ts, q, k, v, dO, H, mask)
    ref = _attn_oracle(seg, ts, q, k, v, dO, H, mask)
    for name in PROBED[kind]:
        g, r = got[name], ref[name]
        gz, rz = g != 0, r != 0
        bad = np.argwhere(gz != rz)
        assert bad.size == 0, (name, "mask pattern differs at (token, column)", bad[:10].tolist(),
                               int(bad.shape[0]))
        nz = rz
        relv = np.abs(g[nz] - r[nz]) / np.abs(r[nz])
        assert relv.max() <= 1e-2, (name, float(relv.max()))
    # the other outputs of the call: ordinary parity
    for name in ("o", "dq", "dk", "dv"):
        assert rel_err(got[name], ref[name]) <= 2e-2, name


def _mask_of_layout(seg, ts, mask):
    h = oracle.build_jagged(seg)
    out = []
    for u in range(len(seg)):
        s, e = int(h["offsets"][u]), int(h["offsets"][u + 1])
        out.append(oracle.mask_for(mask, int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u]), ts[s:e]))
    return out


def test_probe_covers_every_pair(dev):
    """The probe's one-hot windows cover every (reader, read) pair of the probe users, and the
    users' masks contain every kind of entry (static, real-time earlier / tied / later,
    candidate diagonal)."""
    for H in (2, 3):
        seg, ts = _probe_batch(H)
        assert int(seg.sum(1).max()) <= 256 * H
        ms = _mask_of_layout(seg, ts, "dynamic")
        h = oracle.build_jagged(seg)
        tied = later = 0
        for u, M in enumerate(ms):
            s = int(h["offsets"][u]); ns, nr = int(h["n_static"][u]), int(h["n_rt"][u])
            t = ts[s:s + M.shape[0]]
            for i in range(ns, M.shape[0]):
                rt = t[ns:ns + nr]
                tied += int(((rt == t[i]) & (np.arange(ns, ns + nr) != i)).sum())
                later += int((rt > t[i]).sum())
        assert tied > 100 and later > 100


# ------------------------------------------------------------------ leakage through real-time tokens

def test_realtime_leakage_bitwise_bf16(dev):
    """Rule 2: a candidate sees real-time tokens that occurred strictly before it (R#10:
    equal timestamps are invisible).  Perturbing every real-time token with ts >= the
    candidate's, including exact ties, and every other candidate leaves the candidate's output of
    a 3-layer bf16 stack bitwise identical (the layout is unchanged and masked entries are exact
    zeros)."""
    import synth
    seg = np.array([[32, 300, 150, 40], [8, 100, 220, 90], [32, 220, 4, 12]], np.int32)
    cfg, seg, ts, X, dZ, P = make_batch("parity", seg=seg)
    rng = np.random.default_rng(3)
    h = oracle.build_jagged(seg)
    ts = ts.copy()
    for u in range(len(seg)):  # coarse times: ties between real-time tokens and candidates
        s = int(h["offsets"][u]); ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        ts[s + ns:s + ns + nr + nc] = 7000 + rng.integers(0, 15, nr + nc)
    Ps = [synth.gen_layer_params(cfg, li) for li in range(3)]
    dt = torch.bfloat16
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    stack = m.HstuStack(lc, [m.params_to_device(p, dt, dev) for p in Ps], dt, dev)
    stack.bind(jb)
    z1 = stack.forward(torch.from_numpy(X).to(dev, dt)).float().cpu().numpy()
    checked = 0
    for u in range(len(seg)):
        s = int(h["offsets"][u]); ns, nr, nc = int(h["n_static"][u]), int(h["n_rt"][u]), int(h["n_cand"][u])
        for c in (s + ns + nr, s + ns + nr + nc // 2):
            rt = np.arange(s + ns, s + ns + nr)
            hidden = rt[ts[rt] >= ts[c]]
            assert (ts[hidden] == ts[c]).any() or nr < 10
            others = np.setdiff1d(np.arange(s + ns + nr, s + ns + nr + nc), [c])
            X2 = X.copy()
            X2[hidden] += synth.round_bf16(rng.standard_normal((len(hidden), X.shape[1])).astype(np.float32) * 4)
            X2[others] -= 2.0
            z2 = stack.forward(torch.from_numpy(X2).to(dev, dt)).float().cpu().numpy()
            np.testing.assert_array_equal(z1[c], z2[c])
            # and the perturbation does reach the tokens that may see it
            if len(hidden):
                assert not np.array_equal(z1[hidden], z2[hidden])
            checked += 1
    assert checked == 2 * len(seg)


# ------------------------------------------------------------------ zero-mean scores

def test_zero_mean_scores_attention(dev, bwd_path):
    """Scores ~ N(0, 3^2) (q, k zero-mean): SiLU and SiLU' on their curved and negative branches
    (the tanh.approx forms of the kernels).  Max-normalised error <= 2e-2 per tensor; the
    99.9th-percentile elementwise error is reported."""
    cfg, seg, ts, X, dZ, P = make_batch("parity")
    rng = np.random.default_rng(21)
    import synth
    T, d = X.shape
    H = cfg["H"]
    sd = np.sqrt(3.0 / 16.0)  # q.k over 256 dims: std 16 sd^2 = 3
    qkvu = synth.round_bf16((rng.standard_normal((T, 4 * d)) * sd).astype(np.float32))
    dO = synth.round_bf16(rng.standard_normal((T, d)).astype(np.float32))
    q, k, v = qkvu[:, :d], qkvu[:, d:2 * d], qkvu[:, 2 * d:3 * d]
    # the scores really are spread over both branches
    s01 = (q[:200, :256].astype(np.float64) @ k[:200, :256].T.astype(np.float64)).ravel()
    assert abs(s01.mean()) < 0.5 and 2.0 < s01.std() < 4.0 and (s01 < -2).mean() > 0.2
    got = _attn_gpu(dev, seg, ts, q, k, v, dO, H, "dynamic")
    ref = _attn_oracle(seg, ts, q, k, v, dO, H, "dynamic")
    rep = {}
    for name in ("o", "dq", "dk", "dv"):
        e = rel_err(got[name], ref[name])
        rep[name] = (e, p999_rel_err(got[name], ref[name]))
        assert e <= 2e-2, (name, e)
        # elementwise: bf16 P / dS and output rounding (2^-9 each) on sums with cancellation;
        # measured 0.07 (floor 1e-2 max|o|, tests/fixtures.p999_rel_err)
        assert rep[name][1] <= 0.15, (name, rep[name])
    report("zero_mean_attention[%s]" % bwd_path, rep)
    print("zero-mean attention (max-normalised, p99.9 elementwise):", rep)


def test_zero_mean_scores_layer(dev, bwd_path):
    """The layer with linear Q/K/V/U (qkvu_silu = 0, R#5's flag) and Q, K weights scaled so the
    scores are zero-mean with std ~3: the whole forward and backward against the oracle."""
    import synth
    cfg, seg, ts, X, dZ, P = make_batch("parity")
    d = cfg["d"]
    P = dict(P)
    W1 = P["W1"].copy()
    W1[:2 * d] = synth.round_bf16(W1[:2 * d] * np.float32(np.sqrt(3.0 / 16.0)))
    P["W1"] = W1
    dt = torch.bfloat16
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(d, cfg["H"], cfg["groups"], qkvu_silu=False)
    stack = m.HstuStack(lc, [m.params_to_device(P, dt, dev)], dt, dev)
    stack.bind(jb)
    z = stack.forward(torch.from_numpy(X).to(dev, dt)).float().cpu().numpy()
    dx = stack.backward(torch.from_numpy(dZ).to(dev, dt)).float().cpu().numpy()
    grads = {k: v.cpu().numpy() for k, v in stack.grads[0].items() if not k.startswith("_")}
    h = oracle.build_jagged(seg)
    ocfg = dict(d=d, H=cfg["H"], qkvu_silu=False)
    Zo, caches = oracle.layer_fwd_jagged(X, h["offsets"], h["n_static"], h["n_rt"], h["n_cand"],
                                         h["group_id"], ts, P, ocfg)
    dXo, go = oracle.layer_bwd_jagged(dZ, h["offsets"], caches, P, ocfg)
    S = np.concatenate([c.S[0].ravel()[:20000] for c in caches.values()])
    assert abs(S.mean()) < 1.0 and S.std() > 1.5 and (S < -2).mean() > 0.1
    rep = {"Z": (rel_err(z, Zo), p999_rel_err(z, Zo)), "dX": (rel_err(dx, dXo), p999_rel_err(dx, dXo))}
    for k in go:
        rep["d" + k] = (rel_err(grads[k], go[k]), p999_rel_err(grads[k], go[k]))
    report("zero_mean_layer[%s]" % bwd_path, rep)
    print("zero-mean layer (max-normalised, p99.9 elementwise):", rep)
    # max-normalised <= 2e-2 (north_star); elementwise p99.9 <= 0.5 (bf16 storage of every
    # intermediate - X~, p, a, O, Y~ - each rounded at 2^-9 of its own scale; measured <= 0.25)
    bad = {k: v for k, v in rep.items() if not (v[0] <= 2e-2 and v[1] <= 0.5)}
    assert not bad, bad
