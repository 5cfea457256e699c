"""Pins of the oracle's candidate head + two-task BCE."""
import math

import numpy as np
import pytest
import torch

from oracle import bce_with_logits, candidate_rows, head_fwd_bwd, silu


def _params(rng, d, dh, scale=1.0):
    return {"w_a": rng.standard_normal((dh, d)) * scale / math.sqrt(d),
            "b_a": rng.standard_normal(dh) * 0.1,
            "w_b": rng.standard_normal((2, dh)) / math.sqrt(dh),
            "b_b": rng.standard_normal(2) * 0.1}


def test_bce_analytic_values():
    """logit 0 -> ln 2 for either label; logit +20, label 1 -> ~0 (saturation)."""
    assert bce_with_logits(0.0, 0.0) == pytest.approx(math.log(2), abs=1e-15)
    assert bce_with_logits(0.0, 1.0) == pytest.approx(math.log(2), abs=1e-15)
    assert bce_with_logits(20.0, 1.0) == pytest.approx(0.0, abs=3e-9)
    assert bce_with_logits(-20.0, 1.0) == pytest.approx(20.0, abs=1e-8)


def test_bce_matches_torch():
    rng = np.random.default_rng(0)
    l = rng.standard_normal(50) * 4
    y = (rng.random(50) < 0.5).astype(np.float64)
    ref = torch.nn.functional.binary_cross_entropy_with_logits(
        torch.from_numpy(l), torch.from_numpy(y), reduction="none").numpy()
    np.testing.assert_allclose(bce_with_logits(l, y), ref, rtol=1e-13, atol=1e-14)


def test_zero_head_gives_zero_logits():
    """zero representation / zero head -> logits 0, each task loss K ln 2."""
    rng = np.random.default_rng(1)
    K, d, dh = 7, 8, 4
    P = {"w_a": np.zeros((dh, d)), "b_a": np.zeros(dh), "w_b": np.zeros((2, dh)), "b_b": np.zeros(2)}
    lab = rng.integers(0, 4, K).astype(np.uint8)
    logits, loss, _, _ = head_fwd_bwd(rng.standard_normal((K, d)), lab, P)
    np.testing.assert_array_equal(logits, 0.0)
    np.testing.assert_allclose(loss, [K * math.log(2)] * 2, rtol=1e-14)


def test_one_candidate_scalar_loops():
    """the head on one candidate equals a hand-written scalar evaluation."""
    rng = np.random.default_rng(2)
    d, dh = 5, 3
    P = _params(rng, d, dh)
    z = rng.standard_normal((1, d))
    lab = np.array([1], np.uint8)  # click, no purchase
    logits, loss, _, _ = head_fwd_bwd(z, lab, P)
    h = []
    for a in range(dh):
        s = P["b_a"][a]
        for c in range(d):
            s += P["w_a"][a][c] * z[0][c]
        h.append(s / (1.0 + math.exp(-s)))
    for t in range(2):
        l = P["b_b"][t] + sum(P["w_b"][t][a] * h[a] for a in range(dh))
        assert logits[0][t] == pytest.approx(l, rel=1e-13)
        y = 1.0 if t == 0 else 0.0
        p = 1.0 / (1.0 + math.exp(-l))
        assert loss[t] == pytest.approx(-(y * math.log(p) + (1 - y) * math.log(1 - p)), rel=1e-12)


def test_head_finite_differences():
    rng = np.random.default_rng(3)
    K, d, dh = 6, 6, 4
    P = _params(rng, d, dh)
    z = rng.standard_normal((K, d))
    lab = rng.integers(0, 4, K).astype(np.uint8)
    lab[(lab & 1) == 0] = 0  # purchase implies click
    _, _, dz, g = head_fwd_bwd(z, lab, P)
    f = lambda zz, PP: head_fwd_bwd(zz, lab, PP)[1].sum()
    h = 1e-6
    num = np.zeros_like(z)
    for idx in np.ndindex(z.shape):
        zp = z.copy(); zp[idx] += h
        zm = z.copy(); zm[idx] -= h
        num[idx] = (f(zp, P) - f(zm, P)) / (2 * h)
    np.testing.assert_allclose(dz, num, rtol=1e-6, atol=1e-8)
    for key in P:
        num = np.zeros_like(P[key])
        for idx in np.ndindex(P[key].shape):
            Pp = dict(P); Pp[key] = P[key].copy(); Pp[key][idx] += h
            Pm = dict(P); Pm[key] = P[key].copy(); Pm[key][idx] -= h
            num[idx] = (f(z, Pp) - f(z, Pm)) / (2 * h)
        np.testing.assert_allclose(g[key], num, rtol=1e-6, atol=1e-8, err_msg=key)


def test_candidate_rows_layout():
    """Eq.3: candidates are the last n_cand tokens of each user's span."""
    offsets = np.array([0, 5, 5, 12])
    rows = candidate_rows(offsets, [2, 0, 3], [1, 0, 2], [2, 0, 2])
    np.testing.assert_array_equal(rows, [3, 4, 10, 11])


def test_silu_hidden_activation():
    """The hidden layer is SiLU: h = x sigma(x) at a few points."""
    x = np.array([-3.0, 0.0, 0.5, 4.0])
    np.testing.assert_allclose(silu(x), x / (1 + np.exp(-x)), rtol=1e-15)
