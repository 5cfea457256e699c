"""Pins of the oracle's HSTU layer (Eq.5-6) and its backward."""
import math

import numpy as np
import pytest
import torch

from oracle import (layer_fwd_user, layer_bwd_user, stack_fwd_user, stack_bwd_user,
                    attn_fwd_user, mask_dense)
from tests.fixtures import tiny_user, tiny_params

CFG = dict(d=8, H=2, eps=1e-6, qkvu_silu=True)


# ---------------------------------------------------------------- closed forms

def test_all_static_user_is_dense_silu_attention():
    """n_r = K = 0: every mask entry is 1, Eq.5 reduces to (silu(Q K^T)/L) V per head."""
    rng = np.random.default_rng(0)
    L, d, H = 11, 12, 3
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    o, _, M = attn_fwd_user(q, k, v, L, 0, 0, np.zeros(L, np.int64), H, 1.0 / L)
    assert M.all()
    tq, tk, tv = (torch.from_numpy(a) for a in (q, k, v))
    dh = d // H
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        ref = torch.nn.functional.silu(tq[:, sl] @ tk[:, sl].T) / L @ tv[:, sl]
        np.testing.assert_allclose(o[:, sl], ref.numpy(), atol=1e-12)


def test_candidate_row_closed_form_without_rt():
    """n_r = 0: candidate i reads the static block and itself: o_i = nu (sum_{j<n_s} silu(q_i.k_j) v_j
    + silu(q_i.k_i) v_i) (rules 1 and 3)."""
    rng = np.random.default_rng(1)
    n_s, n_c, d = 5, 4, 6
    L = n_s + n_c
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    nu = 1.0 / L
    o, _, _ = attn_fwd_user(q, k, v, n_s, 0, n_c, np.arange(L), 1, nu)
    for i in range(n_s, L):
        acc = sum(torch.nn.functional.silu(torch.tensor(q[i] @ k[j])).item() * v[j] for j in range(n_s))
        acc = acc + torch.nn.functional.silu(torch.tensor(q[i] @ k[i])).item() * v[i]
        np.testing.assert_allclose(o[i], nu * acc, atol=1e-12)


@pytest.mark.parametrize("seed", range(5))
def test_attention_triple_loop_bruteforce(seed):
    """Scalar triple loop of Eq.5 with the three mask rules evaluated per pair."""
    rng = np.random.default_rng(seed)
    n_s, n_r, n_c = (int(v) for v in rng.integers(0, 4, 3))
    L = n_s + n_r + n_c
    if L == 0:
        return
    H, dh = 2, 3
    d = H * dh
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    ts = np.concatenate([np.zeros(n_s, np.int64), rng.integers(0, 4, n_r + n_c)])
    nu = 1.0 / L
    o, _, _ = attn_fwd_user(q, k, v, n_s, n_r, n_c, ts, H, nu)
    for h in range(H):
        for i in range(L):
            for c in range(dh):
                acc = 0.0
                for j in range(L):
                    if i < n_s:
                        vis = j < n_s
                    else:
                        vis = j < n_s or i == j or (n_s <= j < n_s + n_r and ts[j] < ts[i])
                    if not vis:
                        continue
                    s = sum(q[i, h * dh + e] * k[j, h * dh + e] for e in range(dh))
                    acc += s / (1.0 + math.exp(-s)) * nu * v[j, h * dh + c]
                assert abs(o[i, h * dh + c] - acc) < 1e-12


def test_scalar_transcription_L2_d2():
    """L=2 (one profile token, one candidate), d=2, 1 head, written as scalar arithmetic."""
    rng = np.random.default_rng(3)
    d, G, eps = 2, 4, 1e-6
    P = tiny_params(rng, d, 1, G)
    x = rng.standard_normal((2, d))
    gid = np.array([0, 3])
    ts = np.array([0, 5])
    z, _ = layer_fwd_user(x, gid, 1, 0, 1, ts, P, dict(d=2, H=1, eps=eps))

    def ln(row, g, b):
        m = (row[0] + row[1]) / 2
        var = ((row[0] - m) ** 2 + (row[1] - m) ** 2) / 2
        r = 1 / math.sqrt(var + eps)
        return [g[c] * (row[c] - m) * r + b[c] for c in range(2)]

    def silu(s):
        return s / (1 + math.exp(-s))

    a = []
    xt = []
    for i in range(2):
        xt.append(ln(x[i], P["gamma1"][gid[i]], P["beta1"][gid[i]]))
        a.append([silu(sum(P["W1"][o][c] * xt[i][c] for c in range(2)) + P["b1"][o]) for o in range(8)])
    q = [r[0:2] for r in a]; k = [r[2:4] for r in a]; v = [r[4:6] for r in a]; u = [r[6:8] for r in a]
    dot = lambda p_, q_: p_[0] * q_[0] + p_[1] * q_[1]
    o0 = [0.5 * silu(dot(q[0], k[0])) * v[0][c] for c in range(2)]                  # static reads static
    o1 = [0.5 * (silu(dot(q[1], k[0])) * v[0][c] + silu(dot(q[1], k[1])) * v[1][c]) for c in range(2)]
    for i, oi in enumerate((o0, o1)):
        y = [oi[c] * u[i][c] for c in range(2)]
        yt = ln(y, P["gamma2"][gid[i]], P["beta2"][gid[i]])
        zi = [sum(P["W2"][o][c] * yt[c] for c in range(2)) + P["b2"][o] + x[i][o] for o in range(2)]
        np.testing.assert_allclose(z[i], zi, rtol=1e-12, atol=1e-12)


def test_zero_fixed_point():
    """x = 0, biases 0, beta 0 -> z = 0."""
    rng = np.random.default_rng(4)
    P = tiny_params(rng, 8, 2)
    for key in ("b1", "b2", "beta1", "beta2"):
        P[key] = np.zeros_like(P[key])
    x, gid, ts = tiny_user(rng, 3, 3, 3, 8)
    z, _ = layer_fwd_user(np.zeros_like(x), gid, 3, 3, 3, ts, P, CFG)
    assert np.all(z == 0)


def test_residual_identity():
    """W2 = 0, b2 = 0 makes the layer the identity on token values."""
    rng = np.random.default_rng(5)
    P = tiny_params(rng, 8, 2)
    P["W2"] = np.zeros_like(P["W2"]); P["b2"] = np.zeros_like(P["b2"])
    x, gid, ts = tiny_user(rng, 4, 3, 2, 8)
    z, _ = layer_fwd_user(x, gid, 4, 3, 2, ts, P, CFG)
    np.testing.assert_array_equal(z, x)


# ---------------------------------------------------------------- backward

def _fd_check(seed, n_s, n_r, n_c, rab, n_layers=1):
    rng = np.random.default_rng(seed)
    d, H = 8, 2
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d, ts_span=6)
    if rab:
        ts = ts + np.concatenate([np.zeros(n_s, np.int64), rng.integers(0, 300, n_r + n_c)])
    Ps = [tiny_params(rng, d, H, rab_buckets=6 if rab else 0) for _ in range(n_layers)]
    w = rng.standard_normal(x.shape)

    def loss(xx, PP):
        z, _ = stack_fwd_user(xx, gid, n_s, n_r, n_c, ts, PP, CFG)
        return (z * w).sum()

    z, caches = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    dx, grads = stack_bwd_user(w, caches, Ps, CFG)
    h = 1e-6
    num = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        xp = x.copy(); xp[idx] += h
        xm = x.copy(); xm[idx] -= h
        num[idx] = (loss(xp, Ps) - loss(xm, Ps)) / (2 * h)
    np.testing.assert_allclose(dx, num, rtol=1e-5, atol=1e-6)
    for li in range(n_layers):
        for key, g in grads[li].items():
            num = np.zeros_like(g)
            for idx in np.ndindex(g.shape):
                Pp = [dict(P) for P in Ps]; Pm = [dict(P) for P in Ps]
                Pp[li][key] = Ps[li][key].copy(); Pp[li][key][idx] += h
                Pm[li][key] = Ps[li][key].copy(); Pm[li][key][idx] -= h
                num[idx] = (loss(x, Pp) - loss(x, Pm)) / (2 * h)
            np.testing.assert_allclose(g, num, rtol=1e-5, atol=1e-6, err_msg=f"layer {li} {key}")


@pytest.mark.parametrize("seed,n_s,n_r,n_c", [(0, 3, 4, 3), (1, 2, 0, 3), (2, 4, 3, 0), (3, 0, 3, 2)])
def test_layer_backward_finite_differences(seed, n_s, n_r, n_c):
    _fd_check(seed, n_s, n_r, n_c, rab=False)


def test_layer_backward_finite_differences_rab():
    _fd_check(7, 3, 4, 3, rab=True)


def test_stack_backward_finite_differences():
    _fd_check(9, 2, 3, 2, rab=False, n_layers=2)


# ---------------------------------------------------------------- invariants

def _user(seed, n_s=4, n_r=5, n_c=5, d=8):
    rng = np.random.default_rng(seed)
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d, ts_span=10)
    Ps = [tiny_params(rng, d, 2) for _ in range(2)]
    return x, gid, ts, Ps


def test_leakage_exactly_zero_through_stack():
    """a candidate's outputs do not depend on other candidates, nor on rt tokens at or
    after its request time — bitwise, through two stacked layers."""
    n_s, n_r, n_c = 4, 5, 5
    x, gid, ts, Ps = _user(11, n_s, n_r, n_c)
    z, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    rng = np.random.default_rng(99)
    for j in range(n_s + n_r, n_s + n_r + n_c):
        x2 = x.copy()
        for t in range(n_s + n_r + n_c):
            other_cand = t >= n_s + n_r and t != j
            late_rt = n_s <= t < n_s + n_r and ts[t] >= ts[j]
            if other_cand or late_rt:
                x2[t] = rng.standard_normal(x.shape[1]) * 10
        z2, _ = stack_fwd_user(x2, gid, n_s, n_r, n_c, ts, Ps, CFG)
        np.testing.assert_array_equal(z2[j], z[j])


def test_removal_invariance_with_fixed_normaliser():
    """with a fixed 1/N, dropping the other candidates leaves candidate j's output
    unchanged (associativity tolerance 1e-12)."""
    n_s, n_r, n_c = 4, 5, 5
    x, gid, ts, Ps = _user(12, n_s, n_r, n_c)
    nu = 1 / 17.0
    z, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG, nu=nu)
    for j in range(n_s + n_r, n_s + n_r + n_c):
        keep = list(range(n_s + n_r)) + [j]
        zj, _ = stack_fwd_user(x[keep], gid[keep], n_s, n_r, 1, ts[keep], Ps, CFG, nu=nu)
        np.testing.assert_allclose(zj[-1], z[j], rtol=0, atol=1e-12)


def test_removal_changes_output_with_length_normaliser():
    """Eq.5's literal 1/L_u couples candidates through L_u (S:344 scope statement)."""
    n_s, n_r, n_c = 4, 5, 5
    x, gid, ts, Ps = _user(13, n_s, n_r, n_c)
    z, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    j = n_s + n_r
    keep = list(range(n_s + n_r)) + [j]
    zj, _ = stack_fwd_user(x[keep], gid[keep], n_s, n_r, 1, ts[keep], Ps, CFG)
    assert np.abs(zj[-1] - z[j]).max() > 1e-6


def test_candidate_permutation_equivariance():
    """permuting candidates permutes outputs and leaves parameter gradients unchanged."""
    n_s, n_r, n_c = 4, 5, 5
    x, gid, ts, Ps = _user(14, n_s, n_r, n_c)
    perm = np.arange(n_s + n_r + n_c)
    perm[n_s + n_r:] = n_s + n_r + np.random.default_rng(1).permutation(n_c)
    z, c1 = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    zp, c2 = stack_fwd_user(x[perm], gid[perm], n_s, n_r, n_c, ts[perm], Ps, CFG)
    np.testing.assert_allclose(zp, z[perm], atol=1e-12)
    w = np.random.default_rng(2).standard_normal(x.shape)
    dx, g = stack_bwd_user(w, c1, Ps, CFG)
    dxp, gp = stack_bwd_user(w[perm], c2, Ps, CFG)
    np.testing.assert_allclose(dxp, dx[perm], atol=1e-11)
    for li in range(2):
        for key in g[li]:
            np.testing.assert_allclose(gp[li][key], g[li][key], atol=1e-10)


def test_mask_is_shared_by_layers():
    """the same mask is applied in every layer of the stack."""
    x, gid, ts, Ps = _user(15)
    _, caches = stack_fwd_user(x, gid, 4, 5, 5, ts, Ps, CFG)
    np.testing.assert_array_equal(caches[0].M, caches[1].M)
    np.testing.assert_array_equal(caches[0].M, mask_dense(4, 5, 5, ts))


# ---------------------------------------------------------------- 2-layer post-gate MLP (R#6 variant)

def _params2(rng, d, H):
    P = tiny_params(rng, d, H)
    P["W3"] = rng.standard_normal((d, d)) / np.sqrt(d)
    P["b3"] = rng.standard_normal(d) * 0.1
    return P


def test_post_mlp2_matches_torch_and_residual():
    """post_mlp_layers=2: z - x = Linear(W3,b3)(SiLU(Linear(W2,b2)(GLN2(y)))) (torch.nn on the
    layer's own yt); W3 = b3 = 0 gives the residual identity z = x."""
    rng = np.random.default_rng(21)
    d, H = 8, 2
    x, gid, ts = tiny_user(rng, 3, 3, 2, d)
    P = _params2(rng, d, H)
    cfg2 = dict(CFG, post_mlp_layers=2)
    z, c = layer_fwd_user(x, gid, 3, 3, 2, ts, P, cfg2)
    net = torch.nn.Sequential(torch.nn.Linear(d, d), torch.nn.SiLU(), torch.nn.Linear(d, d)).double()
    with torch.no_grad():
        net[0].weight.copy_(torch.from_numpy(P["W2"])); net[0].bias.copy_(torch.from_numpy(P["b2"]))
        net[2].weight.copy_(torch.from_numpy(P["W3"])); net[2].bias.copy_(torch.from_numpy(P["b3"]))
        ref = net(torch.from_numpy(c.yt)).numpy()
    np.testing.assert_allclose(z - x, ref, rtol=1e-12, atol=1e-12)
    P0 = dict(P, W3=np.zeros((d, d)), b3=np.zeros(d))
    np.testing.assert_array_equal(layer_fwd_user(x, gid, 3, 3, 2, ts, P0, cfg2)[0], x)


def test_post_mlp2_backward_finite_differences():
    rng = np.random.default_rng(22)
    d, H = 8, 2
    x, gid, ts = tiny_user(rng, 3, 3, 2, d)
    P = _params2(rng, d, H)
    cfg2 = dict(CFG, post_mlp_layers=2)
    w = rng.standard_normal(x.shape)
    z, c = layer_fwd_user(x, gid, 3, 3, 2, ts, P, cfg2)
    dx, g = layer_bwd_user(w, c, P, cfg2)
    f = lambda xx, PP: (layer_fwd_user(xx, gid, 3, 3, 2, ts, PP, cfg2)[0] * w).sum()
    h = 1e-6
    num = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        xp = x.copy(); xp[idx] += h
        xm = x.copy(); xm[idx] -= h
        num[idx] = (f(xp, P) - f(xm, P)) / (2 * h)
    np.testing.assert_allclose(dx, num, rtol=1e-5, atol=1e-6)
    for key in ("W2", "b2", "W3", "b3", "W1"):
        num = np.zeros_like(P[key])
        for idx in np.ndindex(P[key].shape):
            Pp = dict(P); Pp[key] = P[key].copy(); Pp[key][idx] += h
            Pm = dict(P); Pm[key] = P[key].copy(); Pm[key][idx] -= h
            num[idx] = (f(x, Pp) - f(x, Pm)) / (2 * h)
        np.testing.assert_allclose(g[key], num, rtol=1e-5, atol=1e-6, err_msg=key)
