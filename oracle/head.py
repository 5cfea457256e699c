"""Candidate logit head and the two-task loss — TEST INFRASTRUCTURE ONLY.

"The representation of the tokens of candidates are used for logit via another MLP module"
(Fig.2(a) caption); the tasks are CTR and CTCVR.  Reading R#21 (
sizes from S:358): per candidate token c of the encoder output,
    h_c = SiLU(W_a z_c + b_a),   l_c = W_b h_c + b_b   (l_c = [ctr logit, ctcvr logit])
    loss_ctr   = sum_c BCE(l_c[0], click_c)
    loss_ctcvr = sum_c BCE(l_c[1], click_c AND purchase_c)
    BCE(l, y)  = -y log sigma(l) - (1 - y) log(1 - sigma(l))
Sums over candidates (the 1/B scaling is the aggregation step, R#20).  Parity pins:
tests/test_oracle_head.py (ln 2 at logit 0, saturation, hand scalar loop, FD, zero head).
"""
from __future__ import annotations

import numpy as np

from .layer import silu, dsilu


def candidate_rows(offsets, n_static, n_rt, n_cand):
    """Global row indices of the candidate tokens, user-major (layout [U|S|R|cand], Eq.3)."""
    rows = []
    for u in range(len(n_cand)):
        start = int(offsets[u]) + int(n_static[u]) + int(n_rt[u])
        rows.extend(range(start, start + int(n_cand[u])))
    return np.asarray(rows, dtype=np.int64)


def bce_with_logits(l, y):
    """-y log sigma(l) - (1-y) log(1 - sigma(l)), written as softplus(l) - y l (exact identity)."""
    l = np.asarray(l, dtype=np.float64)
    return np.logaddexp(0.0, l) - y * l


def sigmoid(l):
    return 0.5 * (1.0 + np.tanh(0.5 * np.asarray(l, dtype=np.float64)))


def head_fwd_bwd(zc, labels, P):
    """zc [K][d] candidate representations; labels uint8 [K] (bit 0 click, bit 1 purchase).
    Returns (logits [K][2], loss [2], dzc [K][d], grads) for d(loss[0] + loss[1])."""
    zc = np.asarray(zc, dtype=np.float64)
    Wa, ba = np.asarray(P["w_a"], np.float64), np.asarray(P["b_a"], np.float64)
    Wb, bb = np.asarray(P["w_b"], np.float64), np.asarray(P["b_b"], np.float64)
    lab = np.asarray(labels, dtype=np.uint8)
    y = np.stack([(lab & 1) != 0, (lab & 3) == 3], axis=1).astype(np.float64)
    pre = zc @ Wa.T + ba
    h = silu(pre)
    logits = h @ Wb.T + bb
    loss = bce_with_logits(logits, y).sum(axis=0)
    dl = sigmoid(logits) - y                   # d BCE / d l
    g = {"w_b": dl.T @ h, "b_b": dl.sum(axis=0)}
    dpre = (dl @ Wb) * dsilu(pre)
    g["w_a"] = dpre.T @ zc
    g["b_a"] = dpre.sum(axis=0)
    dzc = dpre @ Wa
    return logits, loss, dzc, g
