"""Pins of the oracle's Group-Layer Norm."""
import numpy as np
import pytest
import torch

from oracle import gln_fwd, gln_bwd


def test_group_equal_params_is_textbook_layernorm():
    """with one (gamma, beta) shared by all groups GLN is torch's layer_norm."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((37, 48)) * 3 + 1
    gid = rng.integers(0, 4, 37)
    g1 = rng.standard_normal(48)
    b1 = rng.standard_normal(48)
    y, mean, rstd = gln_fwd(x, gid, np.tile(g1, (4, 1)), np.tile(b1, (4, 1)), eps=1e-6)
    ref = torch.nn.functional.layer_norm(torch.from_numpy(x), (48,), torch.from_numpy(g1),
                                         torch.from_numpy(b1), eps=1e-6).numpy()
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


def test_per_group_affine_selected_by_group_id():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((20, 16))
    gid = np.array([0, 1, 2, 3] * 5)
    gam = rng.standard_normal((4, 16))
    bet = rng.standard_normal((4, 16))
    y, _, _ = gln_fwd(x, gid, gam, bet)
    plain = torch.nn.functional.layer_norm(torch.from_numpy(x), (16,), eps=1e-6).numpy()
    for i in range(20):
        np.testing.assert_allclose(y[i], gam[gid[i]] * plain[i] + bet[gid[i]], atol=1e-12)


def test_constant_row_maps_to_beta():
    """a constant token normalises to 0, so the output is its group's beta."""
    x = np.full((3, 64), 0.5)
    gid = np.array([0, 2, 3])
    bet = np.arange(4 * 64, dtype=np.float64).reshape(4, 64)
    y, mean, rstd = gln_fwd(x, gid, np.ones((4, 64)) * 7, bet)
    np.testing.assert_array_equal(y, bet[gid])
    np.testing.assert_array_equal(mean, 0.5)


def test_normalised_moments():
    """per-row mean 0 and (biased) variance var/(var+eps) of the normalised token."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((10, 128)) * 5
    y, mean, rstd = gln_fwd(x, np.zeros(10, int), np.ones((1, 128)), np.zeros((1, 128)))
    np.testing.assert_allclose(y.mean(1), 0, atol=1e-12)
    var = x.var(1)
    np.testing.assert_allclose(y.var(1), var / (var + 1e-6), rtol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_backward_matches_finite_differences(seed):
    rng = np.random.default_rng(seed)
    L, d, G = 7, 6, 3
    x = rng.standard_normal((L, d))
    gid = rng.integers(0, G, L)
    gam = rng.standard_normal((G, d))
    bet = rng.standard_normal((G, d))
    w = rng.standard_normal((L, d))

    def f(x_, g_, b_):
        return (gln_fwd(x_, gid, g_, b_)[0] * w).sum()

    _, mean, rstd = gln_fwd(x, gid, gam, bet)
    dx, dg, db = gln_bwd(w, x, gid, mean, rstd, gam)
    h = 1e-6
    for arr, grad, which in ((x, dx, 0), (gam, dg, 1), (bet, db, 2)):
        num = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            args_p = [x.copy(), gam.copy(), bet.copy()]
            args_m = [x.copy(), gam.copy(), bet.copy()]
            args_p[which][idx] += h
            args_m[which][idx] -= h
            num[idx] = (f(*args_p) - f(*args_m)) / (2 * h)
        np.testing.assert_allclose(grad, num, rtol=1e-6, atol=1e-7)
