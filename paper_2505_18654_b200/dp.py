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

    def finish(self, flat):
        while self._works:
            self._works.pop(0).wait()
        self.scale_fn(flat, self.inv_b)
        return flat
