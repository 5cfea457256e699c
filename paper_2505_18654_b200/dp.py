"""Data-parallel plumbing of the MTGR training step (§5 "Load balance").

* Sharding: the global batch of users is partitioned over ranks by the token-count LPT balancer
  of libmtgr (`mtgr_balance_lpt`, reading R#19).  Every rank recomputes the same partition from
  the same seeded batch, so no communication is needed to agree on it.
* Aggregation (R#20): each rank's backward produces gradient SUMS over its users; per-layer
  buckets are all-reduced (sum) as soon as that layer's backward is enqueued (overlapping the
  backward of the layers below), then scaled once by 1/B_global (`mtgr_scale_f32`) — identical to
  weighting each rank's mean gradient by its batch size.

torch.distributed supplies the process group (NCCL over NVLink on the GPU box, gloo in the CPU
tests); the arithmetic of the step stays in libmtgr.
"""
from __future__ import annotations

import numpy as np


def visible_pairs(seg_u, ts_u) -> int:
    """Attention work of one user: P_u = L*n_s + sum_{i>=n_s} |{j in rt: ts_j < ts_i}| + (L-n_s)
    (static rows read the n_s static keys; real-time and candidate rows additionally read the
    earlier real-time tokens and themselves)."""
    nU, nS, nR, K = (int(v) for v in seg_u)
    ns, L = nU + nS, nU + nS + nR + K
    rt = np.sort(np.asarray(ts_u[ns:ns + nR]))
    return L * ns + int(np.searchsorted(rt, np.asarray(ts_u[ns:]), side="left").sum()) + (L - ns)


def flop_cost(seg4, ts_list, d: int) -> np.ndarray:
    """FLOP-aware balancer cost: per-user fwd+bwd FLOPs of one layer divided
    by d, `30 L_u d + 12 P_u` (projections 30 L d^2, attention 12 d P_u), as int64.  The
    token count L_u (the default cost) ignores that attention work grows like L_u n_s."""
    seg4 = np.asarray(seg4)
    L = seg4.astype(np.int64).sum(1)
    P = np.array([visible_pairs(seg4[u], ts_list[u]) for u in range(len(seg4))], dtype=np.int64)
    return 30 * L * int(d) + 12 * P


def shard_users(seg4: np.ndarray, world: int, rank: int, cost=None, balance=None):
    """Users (ascending global index) assigned to `rank` by LPT over `cost` (default L_u)."""
    seg4 = np.asarray(seg4)
    if cost is None:
        cost = seg4.astype(np.int64).sum(1)
    if balance is None:
        from .api import balance_lpt as balance
    rank_of, load = balance(np.asarray(cost, dtype=np.int64), world)
    return np.nonzero(np.asarray(rank_of) == rank)[0].astype(np.int32), np.asarray(load)


class GradAggregator:
    """Per-layer bucket all-reduce (sum) overlapped with the backward, then 1/B_global scaling.

    Use `on_layer_done` as the HstuStack.backward hook and call `finish(flat)` after the
    backward.  `scale_fn(tensor, s)` defaults to libmtgr's mtgr_scale_f32.
    """

    def __init__(self, n_users_global: int, group=None, scale_fn=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.inv_b = 1.0 / float(n_users_global)
        if scale_fn is None:
            from .api import scale_ as scale_fn
        self.scale_fn = scale_fn
        self._works = []

    def on_layer_done(self, li, bucket):
        if self.world > 1:
            self._works.append(self.dist.all_reduce(bucket, group=self.group, async_op=True))

    def finish(self, *flats):
        """Wait for every bucket's all-reduce, then scale each flat gradient buffer by 1/B_global."""
        while self._works:
            self._works.pop(0).wait()
        for flat in flats:
            self.scale_fn(flat, self.inv_b)
        return flats[0] if len(flats) == 1 else flats
