"""Token construction of Eq.4 — TEST INFRASTRUCTURE ONLY.

Per user, X = Concat([Feat_U, Feat_S, Feat_R, Feat_I]) (Eq.4) where the U tokens are the
given d-wide feature embeddings ("each feature is naturally converted to individual token",
P:296) and every S / R / candidate item token is MLP(Concat(Emb)) of its concatenated feature
embeddings.  Reading R#23: one MLP per item type, Linear(k -> d), SiLU,
Linear(d -> d).  Pins: tests/test_oracle_token.py.
"""
from __future__ import annotations

import numpy as np

from .layer import silu, dsilu


def mlp_fwd(F, P):
    """Feat = W2 silu(W1 f + b1) + b2 for each row f of F.  Returns (Y, cache)."""
    F = np.asarray(F, dtype=np.float64)
    W1, b1 = np.asarray(P["w1"], np.float64), np.asarray(P["b1"], np.float64)
    W2, b2 = np.asarray(P["w2"], np.float64), np.asarray(P["b2"], np.float64)
    pre = F @ W1.T + b1
    h = silu(pre)
    return h @ W2.T + b2, (F, pre, h)


def mlp_bwd(dY, cache, P):
    F, pre, h = cache
    W1, W2 = np.asarray(P["w1"], np.float64), np.asarray(P["w2"], np.float64)
    g = {"w2": dY.T @ h, "b2": dY.sum(axis=0)}
    dpre = (dY @ W2) * dsilu(pre)
    g["w1"] = dpre.T @ F
    g["b1"] = dpre.sum(axis=0)
    return dpre @ W1, g


def tokens_user(feats: dict, P: dict):
    """One user's token rows [U | S | R | candidates] (Eq.4).  feats: u [n_U][d], s, r, c item
    features; P: {"s","r","c"} MLP parameters.  Returns (X [L][d], caches)."""
    parts, caches = [np.asarray(feats["u"], np.float64)], {}
    for t in ("s", "r", "c"):
        y, caches[t] = mlp_fwd(feats[t], P[t])
        parts.append(y)
    return np.concatenate(parts, axis=0), caches


def tokens_user_bwd(dX, n_seg, caches, P):
    """Backward of tokens_user given dX [L][d]; n_seg = (n_U, n_S, n_r, K).
    Returns (dfeats, grads per type)."""
    dX = np.asarray(dX, np.float64)
    b = np.cumsum([0] + [int(v) for v in n_seg])
    dfe = {"u": dX[b[0]:b[1]]}
    grads = {}
    for i, t in enumerate(("s", "r", "c")):
        dfe[t], grads[t] = mlp_bwd(dX[b[i + 1]:b[i + 2]], caches[t], P[t])
    return dfe, grads
