"""Pins of the oracle's causal-mask mode: Table 4's "w/o dynamic mask" ablation, i.e.
HSTU's causal mask that MTGR replaces.  m_ij = [j <= i] over the packed order."""
import numpy as np
import pytest
import torch

from oracle import (attn_fwd_user, mask_causal, mask_dense, stack_fwd_user, stack_bwd_user)
from tests.fixtures import tiny_user, tiny_params

CFG = dict(d=8, H=2, eps=1e-6, qkvu_silu=True, mask_mode="causal")
DYN = dict(CFG, mask_mode="dynamic")


def test_causal_equals_dynamic_on_chronological_realtime_sequence():
    """With no static tokens, no candidates and strictly increasing timestamps, the dynamic rule
    for real-time tokens ("visible to tokens that occur afterward") is exactly causality
    over the packed order."""
    L = 9
    ts = np.arange(100, 100 + L, dtype=np.int64)
    np.testing.assert_array_equal(mask_causal(L), mask_dense(0, L, 0, ts))


def test_causal_attention_is_torch_tril_attention():
    """Causal Eq.5 = (silu(Q K^T) masked by torch.tril) / L @ V per head (library mask)."""
    rng = np.random.default_rng(3)
    L, d, H = 10, 6, 2
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    o, _, _ = attn_fwd_user(q, k, v, 3, 4, 3, np.arange(L), H, 1.0 / L, mask_mode="causal")
    tq, tk, tv = (torch.from_numpy(a) for a in (q, k, v))
    tri = torch.tril(torch.ones(L, L, dtype=torch.float64))
    dh = d // H
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        ref = (torch.nn.functional.silu(tq[:, sl] @ tk[:, sl].T) * tri) / L @ tv[:, sl]
        np.testing.assert_allclose(o[:, sl], ref.numpy(), atol=1e-12)


def test_causal_prefix_property():
    """The defining property of a causal mask: with a fixed 1/N, the outputs of the first i
    tokens of a stack equal those of the stack run on that prefix alone."""
    rng = np.random.default_rng(4)
    n_s, n_r, n_c, d = 4, 3, 4, 8
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d)
    Ps = [tiny_params(rng, d, 2) for _ in range(2)]
    nu = 1 / 13.0
    z, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG, nu=nu)
    L = n_s + n_r + n_c
    for i in range(1, L + 1):
        ns_i = min(n_s, i); nr_i = min(n_r, max(0, i - n_s)); nc_i = i - ns_i - nr_i
        zi, _ = stack_fwd_user(x[:i], gid[:i], ns_i, nr_i, nc_i, ts[:i], Ps, CFG, nu=nu)
        np.testing.assert_allclose(zi, z[:i], rtol=0, atol=1e-12)


def test_causal_mask_leaks_between_candidates():
    """P:326 "Using a simple causal mask in MTGR could result in information leakage": under
    the causal mask the last candidate depends on earlier candidates; under the dynamic mask it
    does not (bitwise)."""
    rng = np.random.default_rng(5)
    n_s, n_r, n_c, d = 4, 3, 4, 8
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d)
    Ps = [tiny_params(rng, d, 2)]
    x2 = x.copy()
    x2[n_s + n_r] = rng.standard_normal(d) * 3.0  # the first candidate (not a shift: GLN removes those)
    last = n_s + n_r + n_c - 1
    zc, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
    zc2, _ = stack_fwd_user(x2, gid, n_s, n_r, n_c, ts, Ps, CFG)
    zd, _ = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, DYN)
    zd2, _ = stack_fwd_user(x2, gid, n_s, n_r, n_c, ts, Ps, DYN)
    assert np.abs(zc2[last] - zc[last]).max() > 1e-6
    np.testing.assert_array_equal(zd2[last], zd[last])


@pytest.mark.parametrize("seed", [0, 1])
def test_causal_backward_finite_differences(seed):
    rng = np.random.default_rng(seed)
    n_s, n_r, n_c, d = 3, 3, 2, 8
    x, gid, ts = tiny_user(rng, n_s, n_r, n_c, d)
    Ps = [tiny_params(rng, d, 2)]
    w = rng.standard_normal(x.shape)
    z, caches = stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, CFG)
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
    for key in ("W1", "b1", "gamma1"):
        g = grads[0][key]
        num = np.zeros_like(g)
        for idx in list(np.ndindex(g.shape))[:40]:
            Pp = [dict(Ps[0])]; Pm = [dict(Ps[0])]
            Pp[0][key] = Ps[0][key].copy(); Pp[0][key][idx] += h
            Pm[0][key] = Ps[0][key].copy(); Pm[0][key][idx] -= h
            num[idx] = (loss(x, Pp) - loss(x, Pm)) / (2 * h)
        idxs = list(np.ndindex(g.shape))[:40]
        np.testing.assert_allclose([g[i] for i in idxs], [num[i] for i in idxs], rtol=1e-5, atol=1e-6)
