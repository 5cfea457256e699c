"""Jagged-batch drivers for the oracle: loop the per-user layer over a packed batch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Users never interact (the mask never crosses users: user-level aggregation,
P:281-282), so a jagged batch is exactly the list of its users.
"""
from __future__ import annotations

import numpy as np

from .layer import layer_fwd_user, layer_bwd_user


def _spans(offsets, n_static, n_rt, n_cand):
    for u in range(len(offsets) - 1):
        yield u, int(offsets[u]), int(offsets[u + 1]), int(n_static[u]), int(n_rt[u]), int(n_cand[u])


def layer_fwd_jagged(X, offsets, n_static, n_rt, n_cand, group_id, ts, P, cfg,
                     inv_norm=None, users=None):
    """Returns (Z [T][d] float64, {user: LayerCache}).  `users` restricts to a subset (rows
    of other users are left as NaN)."""
    X = np.asarray(X, dtype=np.float64)
    Z = np.full_like(X, np.nan)
    caches = {}
    for u, a, b, ns, nr, nc in _spans(offsets, n_static, n_rt, n_cand):
        if users is not None and u not in users:
            continue
        assert ns + nr + nc == b - a
        nu = None if inv_norm is None else float(inv_norm[u])
        Z[a:b], caches[u] = layer_fwd_user(X[a:b], group_id[a:b], ns, nr, nc, ts[a:b], P, cfg, nu)
    return Z, caches


def layer_bwd_jagged(dZ, offsets, caches, P, cfg):
    """Returns (dX [T][d] float64, grads summed over the users in `caches`)."""
    dZ = np.asarray(dZ, dtype=np.float64)
    dX = np.full_like(dZ, np.nan)
    tot = None
    for u, c in sorted(caches.items()):
        a, b = int(offsets[u]), int(offsets[u + 1])
        dX[a:b], g = layer_bwd_user(dZ[a:b], c, P, cfg)
        if tot is None:
            tot = {k: v.copy() for k, v in g.items()}
        else:
            for k in tot:
                tot[k] += g[k]
    return dX, tot
