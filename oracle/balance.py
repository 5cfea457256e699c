"""Jagged batch builder, dynamic-BS load balancer and gradient aggregation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §5 "Load balance": "Each GPU's local BS is adjusted based
on the actual sequence length of the input data, ensuring a similar
computational load.  Additionally, we've tweaked the gradient aggregation
strategy to weight each GPU's gradients according to its BS".
Reading R#19: a fixed global batch is partitioned by LPT (longest processing
time first) over a per-user cost (default the token count L_u); ties broken
by (cost desc, user index asc) and (load asc, rank asc); rank-local users
kept in ascending global index.  R#20: aggregation = all-reduce-sum of
per-rank gradient sums / B_global.
"""
from __future__ import annotations

import numpy as np


class BudgetError(ValueError):
    """A single user's cost exceeds the per-rank budget."""


def build_jagged(seg4):
    """User-level aggregation layout (Eq.3; Eq.4).

    seg4 [B][4] = (n_U, n_S, n_r, K) per user, in batch order.
    Returns dict(offsets [B+1] int32 (exclusive prefix sum of L_u), n_static, n_rt, n_cand [B]
    int32, group_id [T] uint8 = 0 (U) | 1 (S) | 2 (R) | 3 (candidates) per token).
    """
    seg4 = np.asarray(seg4, dtype=np.int64).reshape(-1, 4)
    B = seg4.shape[0]
    offsets = [0]
    gid = []
    for u in range(B):
        nU, nS, nR, K = (int(v) for v in seg4[u])
        offsets.append(offsets[-1] + nU + nS + nR + K)
        gid += [0] * nU + [1] * nS + [2] * nR + [3] * K
    return dict(
        offsets=np.array(offsets, dtype=np.int32),
        n_static=(seg4[:, 0] + seg4[:, 1]).astype(np.int32),
        n_rt=seg4[:, 2].astype(np.int32),
        n_cand=seg4[:, 3].astype(np.int32),
        group_id=np.array(gid, dtype=np.uint8),
    )


def lpt(cost, world, cap=None):
    """Greedy LPT partition of users over `world` ranks (R#19).

    Users in order (cost desc, index asc); each goes to the rank with (load asc, rank asc).
    Returns (rank_of [B] int32, load [world] int64).  Raises BudgetError if a cost > cap.
    """
    cost = [int(c) for c in np.asarray(cost).ravel()]
    if world < 1:
        raise ValueError("world must be >= 1")
    if cap is not None and any(c > cap for c in cost):
        raise BudgetError("user cost exceeds cap")
    order = sorted(range(len(cost)), key=lambda u: (-cost[u], u))
    load = [0] * world
    rank_of = [-1] * len(cost)
    for u in order:
        r = min(range(world), key=lambda w: (load[w], w))
        rank_of[u] = r
        load[r] += cost[u]
    return np.array(rank_of, dtype=np.int32), np.array(load, dtype=np.int64)


def aggregate_sum(rank_grad_sums, n_users_global):
    """P:360 with R#20: g = (sum over ranks of per-rank gradient SUMS) / B_global."""
    out = {}
    for k in rank_grad_sums[0]:
        out[k] = sum(np.asarray(gs[k], dtype=np.float64) for gs in rank_grad_sums) / n_users_global
    return out


def aggregate_weighted(rank_grad_means, bs):
    """P:360 literally: g = sum_w bs_w * gbar_w / sum_w bs_w."""
    tot = float(sum(bs))
    out = {}
    for k in rank_grad_means[0]:
        out[k] = sum(b * np.asarray(gm[k], dtype=np.float64) for gm, b in zip(rank_grad_means, bs)) / tot
    return out
