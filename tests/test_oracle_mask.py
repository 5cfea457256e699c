"""Pins of the oracle's dynamic mask (Fig.2(c))."""
import numpy as np
import pytest

from oracle import mask_dense, mask_rules_pairwise, rab_bucket
from oracle.mask import STATIC, REALTIME, CANDIDATE
from tests.fixtures import load_fig2c


def test_fig2c_worked_example_dense():
    n_s, n_r, n_c, ts, golden = load_fig2c()
    assert golden.shape == (9, 9)
    np.testing.assert_array_equal(mask_dense(n_s, n_r, n_c, ts), golden)


def test_fig2c_worked_example_rules():
    n_s, n_r, n_c, ts, golden = load_fig2c()
    kinds = [STATIC] * n_s + [REALTIME] * n_r + [CANDIDATE] * n_c
    np.testing.assert_array_equal(mask_rules_pairwise(kinds, ts), golden)


@pytest.mark.parametrize("seed", range(20))
def test_dense_equals_rule_interpreter(seed):
    rng = np.random.default_rng(seed)
    n_s, n_r, n_c = (int(v) for v in rng.integers(0, 7, 3))
    ts = np.concatenate([np.zeros(n_s, np.int64), rng.integers(0, 6, n_r + n_c)])
    kinds = [STATIC] * n_s + [REALTIME] * n_r + [CANDIDATE] * n_c
    np.testing.assert_array_equal(mask_dense(n_s, n_r, n_c, ts), mask_rules_pairwise(kinds, ts))


@pytest.mark.parametrize("seed", range(10))
def test_structural_invariants(seed):
    """diagonal all 1; candidate columns 0 off the diagonal; static columns all 1
    for non-static rows and static rows; static rows never read rt/candidates (R#8)."""
    rng = np.random.default_rng(100 + seed)
    n_s, n_r, n_c = (int(v) for v in rng.integers(1, 8, 3))
    ts = np.concatenate([np.zeros(n_s, np.int64), rng.integers(0, 5, n_r + n_c)])
    m = mask_dense(n_s, n_r, n_c, ts)
    L = n_s + n_r + n_c
    assert np.all(np.diag(m) == 1)
    cand = m[:, n_s + n_r:] - np.eye(L, dtype=np.uint8)[:, n_s + n_r:]
    assert np.all(cand == 0)
    assert np.all(m[:, :n_s] == 1)
    assert np.all(m[:n_s, n_s:] == 0)


def test_equal_timestamps_invisible():
    """R#10 ("occur afterward"): an rt token at the same second as a candidate is masked."""
    m = mask_dense(1, 1, 1, np.array([0, 7, 7]))
    assert m[2, 1] == 0 and m[1, 2] == 0
    m = mask_dense(1, 1, 1, np.array([0, 6, 7]))
    assert m[2, 1] == 1


def test_order_independence_of_rt():
    """R#12: permuting the rt tokens (with their times) permutes the mask, nothing else."""
    rng = np.random.default_rng(7)
    n_s, n_r, n_c = 3, 6, 4
    ts = np.concatenate([np.zeros(n_s, np.int64), rng.integers(0, 20, n_r + n_c)])
    m = mask_dense(n_s, n_r, n_c, ts)
    perm = np.arange(n_s + n_r + n_c)
    perm[n_s:n_s + n_r] = n_s + rng.permutation(n_r)
    m2 = mask_dense(n_s, n_r, n_c, ts[perm])
    np.testing.assert_array_equal(m2, m[np.ix_(perm, perm)])


def test_rab_bucket_exact():
    dt = np.array([0, 1, -1, 2, 3, 4, 7, 8, 1023, 1024, -1025, 2**40], dtype=np.int64)
    want = [0, 0, 0, 1, 1, 2, 2, 3, 9, 10, 10, 40]
    np.testing.assert_array_equal(rab_bucket(dt, 64), want)
    np.testing.assert_array_equal(rab_bucket(dt, 8), np.minimum(want, 7))
