"""Pins of the oracle's full-mask mode: Table 4's "w/o dynamic mask" ablation read as
full attention: the dynamic mask removed except that candidates stay visible
to themselves only (rule 3).  m_ij = [j < n_s + n_r] or [i == j]."""
import numpy as np
import pytest
import torch

from oracle import attn_fwd_user, mask_dense, mask_full, stack_fwd_user, stack_bwd_user
from tests.fixtures import tiny_user, tiny_params

CFG = dict(d=8, H=2, eps=1e-6, qkvu_silu=True, mask_mode="full")
DYN = dict(CFG, mask_mode="dynamic")


def test_full_without_candidates_is_plain_attention():
    """No candidates: nothing is masked, Eq.5 is silu(Q K^T)/L V per head (torch, no mask)."""
    rng = np.random.default_rng(3)
    L, d, H = 11, 6, 2
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    ts = rng.integers(0, 5, L)
    o, _, M = attn_fwd_user(q, k, v, 4, 7, 0, ts, H, 1.0 / L, mask_mode="full")
    assert M.all()
    tq, tk, tv = (torch.from_numpy(a) for a in (q, k, v))
    dh = d // H
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        ref = torch.nn.functional.silu(tq[:, sl] @ tk[:, sl].T) / L @ tv[:, sl]
        np.testing.assert_allclose(o[:, sl], ref.numpy(), atol=1e-12)


def test_full_candidate_row_closed_form():
    """A candidate row reads every static and real-time token plus itself: o_c = nu (sum_{j <
    n_s + n_r} silu(q_c.k_j) v_j + silu(q_c.k_c) v_c), computed with torch on the kept keys."""
    rng = np.random.default_rng(4)
    n_s, n_r, n_c, d, H = 3, 4, 3, 6, 1
    L = n_s + n_r + n_c
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    o, _, _ = attn_fwd_user(q, k, v, n_s, n_r, n_c, rng.integers(0, 9, L), H, 1.0 / L, mask_mode="full")
    tq, tk, tv = (torch.from_numpy(a) for a in (q, k, v))
    for c in range(n_s + n_r, L):
        keep = list(range(n_s + n_r)) + [c]
        ref = torch.nn.functional.silu(tk[keep] @ tq[c]) @ tv[keep] / L
        np.testing.assert_allclose(o[c], ref.numpy(), atol=1e-12)
    for i in range(n_s + n_r):  # static and real-time rows: every non-candidate key
        ref = torch.nn.functional.silu(tk[:n_s + n_r] @ tq[i]) @ tv[:n_s + n_r] / L
        np.testing.assert_allclose(o[i], ref.numpy(), atol=1e-12)


def test_full_contains_dynamic_and_equals_it_without_realtime():
    """Every pair the dynamic mask shows is shown by the full mask; with no real-time tokens the
    two coincide (static rows read static columns, the rest add their diagonal)."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        n_s, n_r, n_c = (int(x) for x in rng.integers(0, 7, 3))
        L = n_s + n_r + n_c
        ts = rng.integers(0, 4, L)
        F, D = mask_full(n_s, n_r, n_c), mask_dense(n_s, n_r, n_c, ts)
        assert (F >= D).all()
        np.testing.assert_array_equal(mask_full(n_s, 0, n_c), mask_dense(n_s, 0, n_c, ts[:n_s + n_c]))


def test_full_mask_candidates_isolated_static_rows_see_realtime():
    """Candidates stay isolated from each other (bitwise, through a 2-layer stack), while static
    rows now depend on real-time tokens (they do not under the dynamic mask)."""
    rng = np.random.default_rng(6)
    n_s, n_r, n_c, d = 4, 3, 4, 8
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d)
    Ps = [tiny_params(rng, d, 2) for _ in range(2)]
    z, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    x2 = x.copy()
    x2[n_s + n_r] = rng.standard_normal(d) * 3.0  # first candidate
    z2, _ = stack_fwd_user(x2, gid, n_s, n_r, n_c, ts, Ps, CFG)
    np.testing.assert_array_equal(z2[n_s + n_r + 1:], z[n_s + n_r + 1:])
    np.testing.assert_array_equal(z2[:n_s + n_r], z[:n_s + n_r])
    x3 = x.copy()
    x3[n_s] = rng.standard_normal(d) * 3.0  # first real-time token
    zf, _ = stack_fwd_user(x3, gid, n_s, n_r, n_c, ts, Ps, CFG)
    zd, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, DYN)
    zd3, _ = stack_fwd_user(x3, gid, n_s, n_r, n_c, ts, Ps, DYN)
    assert np.abs(zf[:n_s] - z[:n_s]).max() > 1e-6
    np.testing.assert_array_equal(zd3[:n_s], zd[:n_s])


@pytest.mark.parametrize("seed", [0, 1])
def test_full_backward_finite_differences(seed):
    rng = np.random.default_rng(seed)
    n_s, n_r, n_c, d = 3, 3, 2, 8
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d)
    Ps = [tiny_params(rng, d, 2)]
    w = rng.standard_normal(x.shape)
    _, caches = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    dx, grads = stack_bwd_user(w, caches, Ps, CFG)
    h = 1e-6

    def loss(xx, PP):
        return (stack_fwd_user(xx, gid, n_s, n_r, n_c, ts, PP, CFG)[0] * w).sum()
    num = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        xp = x.copy(); xp[idx] += h
        xm = x.copy(); xm[idx] -= h
        num[idx] = (loss(xp, Ps) - loss(xm, Ps)) / (2 * h)
    np.testing.assert_allclose(dx, num, rtol=1e-5, atol=1e-6)
    for key in ("W1", "b1"):
        g = grads[0][key]
        idxs = list(np.ndindex(g.shape))[:40]
        num = []
        for idx in idxs:
            Pp = [dict(Ps[0])]; Pm = [dict(Ps[0])]
            Pp[0][key] = Ps[0][key].copy(); Pp[0][key][idx] += h
            Pm[0][key] = Ps[0][key].copy(); Pm[0][key][idx] -= h
            num.append((loss(x, Pp) - loss(x, Pm)) / (2 * h))
        np.testing.assert_allclose([g[i] for i in idxs], num, rtol=1e-5, atol=1e-6)
