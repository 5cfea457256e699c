"""Pins of the oracle's token construction (Eq.4)."""
import math

import numpy as np
import torch

from oracle import mlp_fwd, tokens_user, tokens_user_bwd


def _P(rng, d, k):
    return {"w1": rng.standard_normal((d, k)) / math.sqrt(k), "b1": rng.standard_normal(d) * 0.1,
            "w2": rng.standard_normal((d, d)) / math.sqrt(d), "b2": rng.standard_normal(d) * 0.1}


def _case(seed, n=(3, 4, 2, 3), d=8, k=(8, 6, 5)):
    rng = np.random.default_rng(seed)
    feats = {"u": rng.standard_normal((n[0], d)), "s": rng.standard_normal((n[1], k[0])),
             "r": rng.standard_normal((n[2], k[1])), "c": rng.standard_normal((n[3], k[2]))}
    P = {"s": _P(rng, d, k[0]), "r": _P(rng, d, k[1]), "c": _P(rng, d, k[2])}
    return feats, P, n


def test_mlp_matches_torch_sequential():
    """MLP = Linear -> SiLU -> Linear (R#23) equals torch.nn on the same weights."""
    rng = np.random.default_rng(0)
    P = _P(rng, 6, 5)
    F = rng.standard_normal((7, 5))
    net = torch.nn.Sequential(torch.nn.Linear(5, 6), torch.nn.SiLU(), torch.nn.Linear(6, 6)).double()
    with torch.no_grad():
        net[0].weight.copy_(torch.from_numpy(P["w1"])); net[0].bias.copy_(torch.from_numpy(P["b1"]))
        net[2].weight.copy_(torch.from_numpy(P["w2"])); net[2].bias.copy_(torch.from_numpy(P["b2"]))
        ref = net(torch.from_numpy(F)).numpy()
    np.testing.assert_allclose(mlp_fwd(F, P)[0], ref, rtol=1e-13, atol=1e-14)


def test_layout_is_eq4_concatenation():
    """Eq.4: rows are [Feat_U | Feat_S | Feat_R | Feat_I] in order; U rows are the embeddings."""
    feats, P, n = _case(1)
    X, _ = tokens_user(feats, P)
    assert X.shape == (sum(n), 8)
    np.testing.assert_array_equal(X[:n[0]], feats["u"])
    b = np.cumsum((0,) + n)
    for i, t in enumerate(("s", "r", "c")):
        np.testing.assert_allclose(X[b[i + 1]:b[i + 2]], mlp_fwd(feats[t], P[t])[0], rtol=0, atol=0)


def test_zero_weights_give_bias_rows():
    """W2 = 0: every item token equals b2 of its type (dimension unification of a constant)."""
    feats, P, n = _case(2)
    for t in P:
        P[t]["w2"] = np.zeros_like(P[t]["w2"])
    X, _ = tokens_user(feats, P)
    b = np.cumsum((0,) + n)
    for i, t in enumerate(("s", "r", "c")):
        np.testing.assert_array_equal(X[b[i + 1]:b[i + 2]], np.broadcast_to(P[t]["b2"], (n[i + 1], 8)))


def test_backward_finite_differences():
    feats, P, n = _case(3)
    X, caches = tokens_user(feats, P)
    w = np.random.default_rng(4).standard_normal(X.shape)
    dfe, g = tokens_user_bwd(w, n, caches, P)
    f = lambda fe, PP: (tokens_user(fe, PP)[0] * w).sum()
    h = 1e-6
    for t in feats:
        num = np.zeros_like(feats[t])
        for idx in np.ndindex(feats[t].shape):
            fp = dict(feats); fp[t] = feats[t].copy(); fp[t][idx] += h
            fm = dict(feats); fm[t] = feats[t].copy(); fm[t][idx] -= h
            num[idx] = (f(fp, P) - f(fm, P)) / (2 * h)
        np.testing.assert_allclose(dfe[t], num, rtol=1e-6, atol=1e-8, err_msg=t)
    for t in ("s", "r", "c"):
        for key in P[t]:
            num = np.zeros_like(P[t][key])
            for idx in np.ndindex(P[t][key].shape):
                Pp = {s: dict(P[s]) for s in P}; Pm = {s: dict(P[s]) for s in P}
                Pp[t][key] = P[t][key].copy(); Pp[t][key][idx] += h
                Pm[t][key] = P[t][key].copy(); Pm[t][key][idx] -= h
                num[idx] = (f(feats, Pp) - f(feats, Pm)) / (2 * h)
            np.testing.assert_allclose(g[t][key], num, rtol=1e-6, atol=1e-8, err_msg=f"{t}.{key}")
