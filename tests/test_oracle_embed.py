"""Pins of the oracle's hash-embedding semantics."""
import numpy as np
import pytest

from oracle import TableModel, init_row, mix64, unique_with_inverse


def test_splitmix64_reference_vectors():
    """The published splitmix64 sequence from state 0: outputs are mix64(k * golden)."""
    g = 0x9E3779B97F4A7C15
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert [mix64((k * g) & ((1 << 64) - 1)) for k in range(4)] == ref


def test_init_rows_are_uniform_and_key_dependent():
    rows = np.stack([init_row(7, k, 64, 0.5) for k in range(400)])
    assert rows.dtype == np.float32 and np.abs(rows).max() <= 0.5
    assert abs(rows.mean()) < 0.01 and abs(rows.var() - 0.25 / 3) < 0.005  # U(-0.5, 0.5)
    assert not np.array_equal(init_row(7, 1, 8, 0.5), init_row(7, 2, 8, 0.5))
    assert not np.array_equal(init_row(7, 1, 8, 0.5), init_row(8, 1, 8, 0.5))
    np.testing.assert_array_equal(init_row(7, -5, 8, 0.5), init_row(7, -5, 8, 0.5))


def test_table_model_lifecycle():
    t = TableModel(4, seed=3, scale=0.1)
    r = t.lookup([5, 9, 5], now=10)
    np.testing.assert_array_equal(r[0], r[2])
    np.testing.assert_array_equal(r[0], init_row(3, 5, 4, 0.1))
    t.sgd([5, 5], np.ones((2, 4)), lr=0.5)            # duplicates accumulate
    np.testing.assert_allclose(t.lookup([5], now=20)[0], init_row(3, 5, 4, 0.1) - 1.0)
    t.evict(ts_before=15)                             # 9 (last 10) goes, 5 (last 20) stays
    assert 9 not in t.rows and 5 in t.rows
    np.testing.assert_array_equal(t.lookup([9], now=30)[0], init_row(3, 9, 4, 0.1))  # fresh row
    assert np.all(t.lookup([77], insert=False) == 0) and 77 not in t.rows


@pytest.mark.parametrize("seed", range(3))
def test_unique_inverse(seed):
    ids = np.random.default_rng(seed).integers(-50, 50, 300)
    u, inv = unique_with_inverse(ids)
    np.testing.assert_array_equal(u[inv], ids)
    assert len(set(u.tolist())) == len(u)
