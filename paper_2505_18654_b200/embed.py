"""Dynamic hash embedding and the sharded embedding lookup (§5
P:352-355).  Thin marshalling over libmtgr (include/mtgr.h, csrc/embed.cu): every step of the
table and of the lookup runs in libmtgr kernels; torch.distributed (NCCL) moves the ID and row
buffers between ranks (the all-to-all of P:355).

Lookup of one batch of IDs on rank r of W ("two-stage ID unique ... before and after ID
communication"):
  1. unique the local IDs                            (stage 1: mtgr_unique)
  2. group them by owner rank, hash(id) % W          (mtgr_partition_ids)
  3. all-to-all of counts, then of the IDs
  4. unique the received IDs                         (stage 2)
  5. find-or-insert in the local shard, gather rows  (mtgr_hash_find_or_insert / _gather)
  6. rows back to the received order, all-to-all back, then to the original positions
Backward: segment-sum of the row gradients by the stage-1 inverse, all-to-all to the owners,
segment-sum by the stage-2 inverse, SGD update of the owned rows (mtgr_hash_sgd).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import HashTable, check, lib, MTGR_F32, MTGR_BF16
from .api import _p, _stream, _ws, _dt


class HashEmbedding:
    """One shard of the dynamic hash table: decoupled key structure (cap_k buckets) and value
    structure (cap_v rows of dim fp32 + counter / timestamp / owner key).  All device memory is
    allocated here with torch (the library never allocates)."""

    def __init__(self, dim: int, cap_v: int, cap_k: int | None = None, seed: int = 0,
                 init_scale: float = 0.05, device="cuda"):
        cap_k = cap_k or 1 << max(4, int(np.ceil(np.log2(max(2 * cap_v, 16)))))
        assert cap_k & (cap_k - 1) == 0
        dev = torch.device(device)
        self.dim, self.cap_v, self.device = dim, cap_v, dev
        self.keys = torch.empty(cap_k, dtype=torch.int64, device=dev)
        self.slots = torch.empty(cap_k, dtype=torch.int32, device=dev)
        self.values = torch.empty((cap_v, dim), dtype=torch.float32, device=dev)
        self.counter = torch.zeros(cap_v, dtype=torch.int32, device=dev)
        self.ts = torch.zeros(cap_v, dtype=torch.int64, device=dev)
        self.slot_key = torch.zeros(cap_v, dtype=torch.int64, device=dev)
        self.alloc = torch.zeros(3, dtype=torch.int32, device=dev)
        self.free_stack = torch.zeros(cap_v, dtype=torch.int32, device=dev)
        self.seed, self.init_scale = seed, init_scale
        self._mk()
        check(lib().mtgr_hash_init(ctypes.byref(self.t), _stream()))

    def _mk(self):
        self.t = HashTable(self.keys.data_ptr(), self.slots.data_ptr(), self.keys.numel(),
                           self.values.data_ptr(), self.counter.data_ptr(), self.ts.data_ptr(),
                           self.slot_key.data_ptr(), self.cap_v, self.dim, self.alloc.data_ptr(),
                           self.free_stack.data_ptr(), self.seed, self.init_scale)

    @property
    def cap_k(self) -> int:
        return self.keys.numel()

    def find_or_insert(self, ids: torch.Tensor, now: int = 0, insert: bool = True) -> torch.Tensor:
        ids = ids.contiguous()
        slots = torch.empty(ids.numel(), dtype=torch.int32, device=self.device)
        check(lib().mtgr_hash_find_or_insert(ctypes.byref(self.t), _p(ids), ids.numel(), int(now),
                                             1 if insert else 0, _p(slots), _stream()))
        return slots

    def gather(self, slots: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
        out = torch.empty((slots.numel(), self.dim), dtype=dtype, device=self.device)
        check(lib().mtgr_hash_gather(ctypes.byref(self.t), _p(slots), slots.numel(), _dt(dtype), _p(out),
                                     _stream()))
        return out

    def sgd(self, slots: torch.Tensor, grads: torch.Tensor, lr: float):
        grads = grads.contiguous()
        check(lib().mtgr_hash_sgd(ctypes.byref(self.t), _p(slots), slots.numel(), _dt(grads.dtype), _p(grads),
                                  float(lr), _stream()))

    def evict(self, ts_before: int):
        check(lib().mtgr_hash_evict(ctypes.byref(self.t), int(ts_before), _stream()))

    def expand(self, new_cap_k: int):
        """Grow the key structure only; the value structure is shared."""
        nk = torch.empty(new_cap_k, dtype=torch.int64, device=self.device)
        ns = torch.empty(new_cap_k, dtype=torch.int32, device=self.device)
        check(lib().mtgr_hash_expand(ctypes.byref(self.t), _p(nk), _p(ns), new_cap_k, _stream()))
        self.keys, self.slots = nk, ns
        self._mk()

    def stats(self) -> dict:
        a = self.alloc.cpu().tolist()
        return {"fresh_slots": a[0], "free_stack": a[1], "failed": a[2]}


def unique(ids: torch.Tensor):
    """(uniq, inverse): uniq = distinct ids (order unspecified), uniq[inverse] == ids."""
    ids = ids.contiguous()
    n = ids.numel()
    uniq = torch.empty(max(n, 1), dtype=torch.int64, device=ids.device)
    inv = torch.empty(max(n, 1), dtype=torch.int32, device=ids.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=ids.device)
    ws = _ws(lib().mtgr_unique_workspace_bytes(n), ids.device)
    check(lib().mtgr_unique(_p(ids), n, _p(uniq), _p(inv), _p(cnt), _p(ws), ws.numel(), _stream()))
    m = int(cnt.item())
    return uniq[:m], inv[:n]


def segment_sum(g: torch.Tensor, inverse: torch.Tensor, n_out: int) -> torch.Tensor:
    out = torch.empty((max(n_out, 1), g.shape[1]), dtype=torch.float32, device=g.device)
    check(lib().mtgr_segment_sum(_dt(g.dtype), _p(g.contiguous()), _p(inverse), inverse.numel(), g.shape[1],
                                 _p(out), n_out, _stream()))
    return out[:n_out]


def take_rows(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    out = torch.empty((idx.numel(), src.shape[1]), dtype=src.dtype, device=src.device)
    check(lib().mtgr_take_rows(_dt(src.dtype), _p(src.contiguous()), _p(idx), idx.numel(), src.shape[1], _p(out),
                               _stream()))
    return out


def put_rows(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(src)
    check(lib().mtgr_put_rows(_dt(src.dtype), _p(src.contiguous()), _p(idx), idx.numel(), src.shape[1], _p(out),
                              _stream()))
    return out


class ShardedEmbedding:
    """The embedding lookup of P:355 over W ranks: each rank owns the IDs with
    hash(id ^ salt) % W == rank in its own HashEmbedding shard."""

    SALT = 0x5bd1e995

    def __init__(self, shard: HashEmbedding, group=None):
        import torch.distributed as dist
        self.shard, self.group = shard, group
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1

    def _a2a(self, send: torch.Tensor, send_counts: list, recv_counts: list, row: int):
        if self.world == 1:
            return send
        out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=send_counts, group=self.group)
        return out

    def lookup(self, ids: torch.Tensor, now: int = 0, dtype=torch.float32):
        """Rows [n][dim] for ids [n] (int64).  Returns (rows, ctx for backward)."""
        dev = ids.device
        W = self.world
        u1, inv1 = unique(ids)                                         # stage 1
        m = u1.numel()
        counts = torch.zeros(W, dtype=torch.int32, device=dev)
        dest = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        starts = torch.empty(2 * W, dtype=torch.int32, device=dev)
        send = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        pos = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        check(lib().mtgr_partition_ids(_p(u1), m, W, self.SALT, _p(counts), _p(dest), _p(starts), _p(send), _p(pos),
                                       _stream()))
        if W > 1:
            rc = torch.empty_like(counts)
            self.dist.all_to_all_single(rc, counts, group=self.group)
            send_counts, recv_counts = counts.cpu().tolist(), rc.cpu().tolist()
        else:
            send_counts = recv_counts = [m]
        recv = self._a2a(send[:m], send_counts, recv_counts, 1)        # IDs to their owners
        u2, inv2 = unique(recv)                                        # stage 2
        slots = self.shard.find_or_insert(u2, now)
        rows2 = self.shard.gather(slots, dtype)
        rows_r = take_rows(rows2, inv2)                                # received order
        back = self._a2a(rows_r, recv_counts, send_counts, self.shard.dim)
        rows1 = take_rows(back, pos[:m])                               # stage-1 unique order
        out = take_rows(rows1, inv1)                                   # original positions
        ctx = dict(inv1=inv1, m=m, pos=pos[:m], send_counts=send_counts, recv_counts=recv_counts,
                   inv2=inv2, slots=slots)
        return out, ctx

    def backward_sgd(self, grads: torch.Tensor, ctx: dict, lr: float):
        """Apply -lr * (sum of the gradients of every occurrence) to the owned rows."""
        g1 = segment_sum(grads, ctx["inv1"], ctx["m"])                 # per stage-1 unique id
        g_send = put_rows(g1, ctx["pos"])                              # send-buffer order
        g_recv = self._a2a(g_send, ctx["send_counts"], ctx["recv_counts"], self.shard.dim)
        g2 = segment_sum(g_recv, ctx["inv2"], ctx["slots"].numel())    # per stage-2 unique id
        self.shard.sgd(ctx["slots"], g2, lr)
