"""Pins of the oracle's builder, LPT balancer and gradient aggregation."""
import itertools

import numpy as np
import pytest

from oracle import (build_jagged, lpt, BudgetError, aggregate_sum, aggregate_weighted,
                    layer_fwd_jagged, layer_bwd_jagged)
from tests.fixtures import tiny_params


def test_build_jagged_hand_example():
    seg = np.array([[2, 1, 1, 1], [0, 0, 0, 0], [1, 0, 2, 3]])
    j = build_jagged(seg)
    np.testing.assert_array_equal(j["offsets"], [0, 5, 5, 11])
    np.testing.assert_array_equal(j["n_static"], [3, 0, 1])
    np.testing.assert_array_equal(j["n_rt"], [1, 0, 2])
    np.testing.assert_array_equal(j["n_cand"], [1, 0, 3])
    np.testing.assert_array_equal(j["group_id"], [0, 0, 1, 2, 3, 0, 2, 2, 3, 3, 3])


def test_lpt_spec_fixtures():
    """S:389-391."""
    r, load = lpt([10] * 8, 4)
    assert list(np.bincount(r, minlength=4)) == [2, 2, 2, 2]
    r, load = lpt([3, 1, 4, 1, 5], 1)
    assert set(r) == {0} and load[0] == 14
    # long tail: {900, 100 x 12} on 4 ranks -> 900 | 400 | 400 | 400 (OPT = 900)
    r, load = lpt([900] + [100] * 12, 4)
    assert sorted(load.tolist()) == [400, 400, 400, 900]


def test_lpt_tie_breaks():
    r, load = lpt([5, 5, 5, 5], 2)
    np.testing.assert_array_equal(r, [0, 1, 0, 1])
    r, load = lpt([1, 7, 7, 3], 3)
    # order: u1 (7) -> r0, u2 (7) -> r1, u3 (3) -> r2, u0 (1) -> r2 (load 3 < 7)
    np.testing.assert_array_equal(r, [2, 0, 1, 2])
    np.testing.assert_array_equal(load, [7, 7, 4])


def test_lpt_budget_error():
    with pytest.raises(BudgetError):
        lpt([5, 12, 3], 2, cap=10)


@pytest.mark.parametrize("seed", range(25))
def test_lpt_against_bruteforce_optimum(seed):
    """Graham: LPT makespan <= (4/3 - 1/(3W)) * OPT; OPT by exhaustive search (n <= 8, W <= 3)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 9))
    W = int(rng.integers(1, 4))
    cost = rng.integers(1, 50, n)
    r, load = lpt(cost, W)
    assert np.all(np.bincount(r, weights=cost, minlength=W) == load)
    opt = min(max(np.bincount(np.array(a), weights=cost, minlength=W))
              for a in itertools.product(range(W), repeat=n))
    assert opt <= load.max() <= (4 / 3 - 1 / (3 * W)) * opt + 1e-9


def test_pooled_gradient_identity():
    """P:360 / S:399: per-rank gradient sums aggregated over an LPT partition equal the pooled
    single-worker gradient; the BS-weighted mean of per-rank means is the same quantity."""
    rng = np.random.default_rng(0)
    d, H = 8, 2
    cfg = dict(d=d, H=H)
    seg = np.array([[2, int(rng.integers(0, 6)), int(rng.integers(0, 4)), int(rng.integers(1, 4))]
                    for _ in range(7)])
    P = tiny_params(rng, d, H)
    j = build_jagged(seg)
    T = int(j["offsets"][-1])
    X = rng.standard_normal((T, d))
    ts = rng.integers(0, 9, T)
    dZ = rng.standard_normal((T, d))
    args = (j["offsets"], j["n_static"], j["n_rt"], j["n_cand"], j["group_id"], ts)
    _, caches = layer_fwd_jagged(X, *args, P, cfg)
    _, pooled = layer_bwd_jagged(dZ, j["offsets"], caches, P, cfg)
    B = len(seg)
    pooled = {k: v / B for k, v in pooled.items()}
    rank_of, _ = lpt(seg.sum(1), 3)
    sums, means, bs = [], [], []
    for w in range(3):
        users = set(np.nonzero(rank_of == w)[0].tolist())
        _, cw = layer_fwd_jagged(X, *args, P, cfg, users=users)
        _, gw = layer_bwd_jagged(dZ, j["offsets"], cw, P, cfg)
        sums.append(gw)
        means.append({k: v / len(users) for k, v in gw.items()})
        bs.append(len(users))
    agg = aggregate_sum(sums, B)
    wag = aggregate_weighted(means, bs)
    for k in pooled:
        np.testing.assert_allclose(agg[k], pooled[k], rtol=0, atol=1e-12)
        np.testing.assert_allclose(wag[k], pooled[k], rtol=0, atol=1e-12)
