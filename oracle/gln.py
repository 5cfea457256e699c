"""Group-Layer Normalization (§4.2: "Features of the same domain
form a group ... the group layer norm ensures that tokens from different domains
share a similar distribution"; Eq.6; Fig.2(b) caption P:273).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading R#13: per-token LayerNorm statistics over d_model, affine (gamma, beta)
selected by the token's group id.  R#14: biased variance, eps = 1e-6.
"""
from __future__ import annotations

import numpy as np


def gln_fwd(x, gid, gamma, beta, eps=1e-6):
    """x [L][d], gid [L] int, gamma/beta [G][d] -> (y [L][d], mean [L], rstd [L]); float64."""
    x = np.asarray(x, dtype=np.float64)
    gamma = np.asarray(gamma, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    mean = x.mean(axis=1)
    var = ((x - mean[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean[:, None]) * rstd[:, None]
    y = gamma[gid] * xhat + beta[gid]
    return y, mean, rstd


def gln_bwd(dy, x, gid, mean, rstd, gamma, n_groups=None):
    """Backward of gln_fwd.  Returns (dx [L][d], dgamma [G][d], dbeta [G][d]).

    dgamma[g] = sum_{i: g_i = g} dy_i * xhat_i,  dbeta[g] = sum_{i: g_i = g} dy_i,
    dxhat = dy * gamma[g_i],
    dx = rstd * (dxhat - mean_c(dxhat) - xhat * mean_c(dxhat * xhat)).
    """
    dy = np.asarray(dy, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    gamma = np.asarray(gamma, dtype=np.float64)
    G = gamma.shape[0] if n_groups is None else n_groups
    xhat = (x - mean[:, None]) * rstd[:, None]
    dgamma = np.zeros((G, x.shape[1]))
    dbeta = np.zeros((G, x.shape[1]))
    for g in range(G):
        sel = gid == g
        dgamma[g] = (dy[sel] * xhat[sel]).sum(axis=0)
        dbeta[g] = dy[sel].sum(axis=0)
    dxhat = dy * gamma[gid]
    dx = rstd[:, None] * (dxhat - dxhat.mean(axis=1, keepdims=True)
                          - xhat * (dxhat * xhat).mean(axis=1, keepdims=True))
    return dx, dgamma, dbeta
