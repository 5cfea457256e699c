"""HSTU encoder layer of MTGR, forward and backward, one user at a time, float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Forward (§4.2):
  X~ = GroupLN(X)
  K, Q, V, U = MLP_{K/Q/V/U}(X~)                         P:313  (R#5: SiLU(X~ W1^T + b1))
  V~ = silu(Q K^T) / (n_U + n_S + n_r + K) * M  V        Eq.5, P:314-317  (R#1 row = reader,
                                                         R#2 mask after silu and 1/N, R#3 N = L_u)
  X  = MLP(GroupLN(V~ * U)) + X                          Eq.6, P:320  (R#6 MLP = one Linear,
                                                         R#7 gate then GLN2)
Optional relative-time bias rab (R#4; not in the paper): s_ij += rab_w[h, bucket(ts_i - ts_j)].

Backward: reverse-mode of the same expressions, written out term by term (no
autograd), verified against central finite differences in tests/test_oracle_layer.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .gln import gln_fwd, gln_bwd
from .mask import mask_dense, mask_for, rab_bucket


def silu(s):
    """silu(s) = s * sigmoid(s)."""
    with np.errstate(over="ignore"):
        return s / (1.0 + np.exp(-s))


def dsilu(s):
    """d/ds silu(s) = sigmoid(s) * (1 + s * (1 - sigmoid(s)))."""
    with np.errstate(over="ignore"):
        sg = 1.0 / (1.0 + np.exp(-s))
    return sg * (1.0 + s * (1.0 - sg))


def _heads(d, H):
    dh = d // H
    return [slice(h * dh, (h + 1) * dh) for h in range(H)]


def attn_fwd_user(q, k, v, n_s, n_r, n_c, ts, H, nu, rab_w=None, mask_mode="dynamic"):
    """Eq.5 per head h:  s_ij = q_i . k_j (+ rab),  A_ij = silu(s_ij) * m_ij * nu,  o_i = sum_j A_ij v_j.

    Masked entries are exact zeros (select, not multiply: R#2).  Returns (o, S list, M).
    mask_mode: "dynamic" (MTGR) or "causal" (the Table 4 ablation).
    """
    L, d = q.shape
    M = mask_for(mask_mode, n_s, n_r, n_c, ts)
    vis = M.astype(bool)
    o = np.zeros((L, d))
    S = []
    for h, sl in enumerate(_heads(d, H)):
        s = q[:, sl] @ k[:, sl].T
        if rab_w is not None:
            s = s + rab_w[h][rab_bucket(ts[:, None] - ts[None, :], rab_w.shape[1])]
        A = np.where(vis, silu(s) * nu, 0.0)
        o[:, sl] = A @ v[:, sl]
        S.append(s)
    return o, S, M


def attn_bwd_user(do, q, k, v, S, M, H, nu, ts=None, rab_w=None):
    """Backward of attn_fwd_user given dO (pre-gate).  Returns (dq, dk, dv, drab or None).

    dv = A^T do;  dA = do v^T;  ds = dA * silu'(s) * m * nu;  dq = ds k;  dk = ds^T q;
    drab[h, b] = sum_{bucket(i,j) = b} ds_ij.
    """
    L, d = q.shape
    vis = M.astype(bool)
    dq = np.zeros((L, d)); dk = np.zeros((L, d)); dv = np.zeros((L, d))
    drab = None if rab_w is None else np.zeros_like(rab_w, dtype=np.float64)
    for h, sl in enumerate(_heads(d, H)):
        s = S[h]
        A = np.where(vis, silu(s) * nu, 0.0)
        dv[:, sl] = A.T @ do[:, sl]
        dA = do[:, sl] @ v[:, sl].T
        ds = np.where(vis, dA * dsilu(s) * nu, 0.0)
        dq[:, sl] = ds @ k[:, sl]
        dk[:, sl] = ds.T @ q[:, sl]
        if rab_w is not None:
            b = rab_bucket(ts[:, None] - ts[None, :], rab_w.shape[1])
            np.add.at(drab[h], b.ravel(), ds.ravel())
    return dq, dk, dv, drab


@dataclass
class LayerCache:
    x: np.ndarray
    gid: np.ndarray
    n_s: int
    n_r: int
    n_c: int
    ts: np.ndarray
    nu: float
    xt: np.ndarray
    mu1: np.ndarray
    r1: np.ndarray
    p: np.ndarray
    a: np.ndarray
    o: np.ndarray
    S: list
    M: np.ndarray
    y: np.ndarray
    yt: np.ndarray
    mu2: np.ndarray
    r2: np.ndarray


def _f64(P):
    return {k: np.asarray(v, dtype=np.float64) for k, v in P.items()}


def layer_fwd_user(x, gid, n_s, n_r, n_c, ts, P, cfg, nu=None):
    """One HSTU layer for one user.  x [L][d]; P params (synth.gen_layer_params layout).

    cfg: dict(d, H, eps=1e-6, qkvu_silu=True, mask_mode="dynamic").  nu: 1/N override (default
    1/L_u, R#3).
    Returns (z [L][d], LayerCache).
    """
    P = _f64(P)
    x = np.asarray(x, dtype=np.float64)
    gid = np.asarray(gid, dtype=np.int64)
    ts = np.asarray(ts, dtype=np.int64)
    L, d = x.shape
    H = cfg["H"]
    eps = cfg.get("eps", 1e-6)
    if nu is None:
        nu = 1.0 / L if L > 0 else 0.0
    xt, mu1, r1 = gln_fwd(x, gid, P["gamma1"], P["beta1"], eps)
    p = xt @ P["W1"].T + P["b1"]
    a = silu(p) if cfg.get("qkvu_silu", True) else p.copy()
    q, k, v, u = a[:, :d], a[:, d:2 * d], a[:, 2 * d:3 * d], a[:, 3 * d:]
    o, S, M = attn_fwd_user(q, k, v, n_s, n_r, n_c, ts, H, nu, P.get("rab_w"),    # Eq.5
                            cfg.get("mask_mode", "dynamic"))
    y = o * u                                                            # Eq.6 gate
    yt, mu2, r2 = gln_fwd(y, gid, P["gamma2"], P["beta2"], eps)          # Eq.6 GroupLN
    if cfg.get("post_mlp_layers", 1) == 2:
        # "another MLP" read as Linear -> SiLU -> Linear (R#6 variant)
        hpre = yt @ P["W2"].T + P["b2"]
        z = silu(hpre) @ P["W3"].T + P["b3"] + x
    else:
        hpre = None
        z = yt @ P["W2"].T + P["b2"] + x                                 # Eq.6 MLP + X (R#6)
    c = LayerCache(x, gid, n_s, n_r, n_c, ts, nu, xt, mu1, r1, p, a, o, S, M, y, yt, mu2, r2)
    c.hpre = hpre
    return z, c


def layer_bwd_user(dz, c: LayerCache, P, cfg):
    """Backward of layer_fwd_user.  Returns (dx, grads) with grads summed over the user's tokens."""
    P = _f64(P)
    dz = np.asarray(dz, dtype=np.float64)
    d = c.x.shape[1]
    H = cfg["H"]
    g = {}
    if getattr(c, "hpre", None) is not None:
        # z = silu(hpre) W3^T + b3 + x,  hpre = yt W2^T + b2
        h = silu(c.hpre)
        g["W3"] = dz.T @ h
        g["b3"] = dz.sum(axis=0)
        dpre = (dz @ P["W3"]) * dsilu(c.hpre)
        g["W2"] = dpre.T @ c.yt
        g["b2"] = dpre.sum(axis=0)
        dyt = dpre @ P["W2"]
    else:
        # z = yt W2^T + b2 + x
        g["W2"] = dz.T @ c.yt
        g["b2"] = dz.sum(axis=0)
        dyt = dz @ P["W2"]
    # yt = GLN2(y)
    dy, g["gamma2"], g["beta2"] = gln_bwd(dyt, c.y, c.gid, c.mu2, c.r2, P["gamma2"])
    # y = o * u
    u = c.a[:, 3 * d:]
    do = dy * u
    du = dy * c.o
    q, k, v = c.a[:, :d], c.a[:, d:2 * d], c.a[:, 2 * d:3 * d]
    dq, dk, dv, drab = attn_bwd_user(do, q, k, v, c.S, c.M, H, c.nu, c.ts, P.get("rab_w"))
    if drab is not None:
        g["rab_w"] = drab
    da = np.concatenate([dq, dk, dv, du], axis=1)
    dp = da * dsilu(c.p) if cfg.get("qkvu_silu", True) else da
    # p = xt W1^T + b1
    g["W1"] = dp.T @ c.xt
    g["b1"] = dp.sum(axis=0)
    dxt = dp @ P["W1"]
    # xt = GLN1(x)
    dx, g["gamma1"], g["beta1"] = gln_bwd(dxt, c.x, c.gid, c.mu1, c.r1, P["gamma1"])
    dx = dx + dz
    return dx, g


def stack_fwd_user(x, gid, n_s, n_r, n_c, ts, Ps, cfg, nu=None):
    """Encoder stack: layers applied in sequence with the same mask."""
    caches = []
    for P in Ps:
        x, c = layer_fwd_user(x, gid, n_s, n_r, n_c, ts, P, cfg, nu)
        caches.append(c)
    return x, caches


def stack_bwd_user(dz, caches, Ps, cfg):
    grads = [None] * len(Ps)
    for li in range(len(Ps) - 1, -1, -1):
        dz, grads[li] = layer_bwd_user(dz, caches[li], Ps[li], cfg)
    return dz, grads
