"""The whole MTGR training step on one rank (Fig.2(a), Eq.4, §5
P:352-362): sparse feature IDs -> sharded dynamic-hash embedding lookup (two-stage unique +
all-to-all) -> Eq.4 token construction -> HSTU encoder stack -> candidate head and the
CTR/CTCVR loss, and back: dense gradients aggregated over the ranks, embedding rows
updated by SGD on their owner shard.  Orchestration only: every step runs in libmtgr kernels;
torch.distributed moves buffers between ranks.

Two tables: U features (one d-wide embedding per profile token) and item features
(EMB_DIM-wide embeddings, k_t / EMB_DIM of them concatenated per S / R / candidate token,
P:297-301).  A token's feature IDs are laid out token-major, so the looked-up rows of a type are
already its [n_t][k_t] feature matrix (a view, no copy).
"""
from __future__ import annotations

import numpy as np
import torch

from .api import HstuStack, JaggedBatch, TokenEmbed, head_fwd_bwd, params_to_device, head_params_to_device
from .embed import HashEmbedding, ShardedEmbedding


class MTGRModel:
    def __init__(self, cfg: dict, layer_cfg, layer_params: list, token_params: dict, head_params: dict,
                 widths: dict, emb_dim: int, dtype: torch.dtype, device, cap_user: int, cap_item: int,
                 lr_sparse: float = 1e-3, seed: int = 0, group=None, n_users_global: int | None = None):
        self.cfg, self.dtype, self.device = cfg, dtype, torch.device(device)
        self.d, self.emb_dim, self.lr_sparse = cfg["d"], emb_dim, lr_sparse
        self.widths = widths
        self.stack = HstuStack(layer_cfg, [params_to_device(p, dtype, device) for p in layer_params], dtype, device)
        self.tokens = TokenEmbed(self.d, widths, TokenEmbed.params_to_device(token_params, dtype, device), dtype, device)
        self.head = head_params_to_device(head_params, dtype, device)
        self.user_table = ShardedEmbedding(HashEmbedding(self.d, cap_user, seed=seed, init_scale=0.5, device=device),
                                           group)
        self.item_table = ShardedEmbedding(HashEmbedding(emb_dim, cap_item, seed=seed + 1, init_scale=0.5,
                                                         device=device), group)
        # R#20: gradients are per-rank SUMS; with n_users_global the dense buckets are
        # all-reduced and scaled by 1/B_global (GradAggregator) and the sparse SGD applies
        # lr / B_global to the summed row gradients (= lr x the batch-weighted mean)
        self.grad_scale = 1.0 if n_users_global is None else 1.0 / float(n_users_global)
        # head + token-MLP gradients live in one flat fp32 bucket (their all-reduce unit)
        shapes = [("head", k, v) for k, v in {"w_a": tuple(self.head["w_a"].shape), "b_a": (self.head["w_a"].shape[0],),
                                             "w_b": tuple(self.head["w_b"].shape), "b_b": (2,)}.items()]
        shapes += [(t, k, v) for t, q in self.tokens.grad_shapes().items() for k, v in q.items()]
        # each view starts on a 256-byte boundary (the GEMMs' TMA descriptors need 16-byte
        # aligned pointers)
        al = lambda n: (n + 63) // 64 * 64
        n = sum(al(int(np.prod(shp))) for _, _, shp in shapes)
        self.dense_flat = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.head_grads, self.token_grads, off = {}, {}, 0
        for owner, k, shp in shapes:
            v = self.dense_flat[off:off + int(np.prod(shp))].view(*shp)
            off += al(v.numel())
            if owner == "head":
                self.head_grads[k] = v
            else:
                self.token_grads.setdefault(owner, {})[k] = v

    def bind(self, jb: JaggedBatch, seg4: np.ndarray):
        self.jb = jb
        self.n = {t: int(np.asarray(seg4)[:, i].sum()) for i, t in enumerate("usrc")}
        self.stack.bind(jb)
        self.tokens.bind(jb, seg4)

    def _item_views(self, buf: torch.Tensor) -> dict:
        """Per-type [n_t][k_t] views of one [n_item_ids][emb_dim] buffer (S | R | candidates)."""
        views, off = {}, 0
        for t in "src":
            n_ids = self.n[t] * (self.widths[t] // self.emb_dim)
            views[t] = buf[off:off + n_ids].view(self.n[t], self.widths[t])
            off += n_ids
        return views

    def step(self, user_ids: torch.Tensor, item_ids: torch.Tensor, labels: torch.Tensor, now: int = 0,
             on_layer_done=None, aggregator=None):
        """user_ids: int64 [n_U] (one per profile token); item_ids: int64 [n_S F_s + n_r F_r +
        n_C F_c] = the S, R and candidate tokens' feature IDs (user-major, token-major, feature
        fastest), as the data loader packs them; labels: uint8 [T].
        aggregator: a dp.GradAggregator: the layer buckets are all-reduced as each layer's
        backward is enqueued, the head + token bucket after the token backward, and both are
        scaled by 1/B_global at the end (R#20).
        Returns (loss [2] sums, dense gradients: per-rank sums, or the aggregated mean)."""
        if aggregator is not None and on_layer_done is None:
            on_layer_done = aggregator.on_layer_done
        # sparse lookups (one two-stage-unique all-to-all per table)
        urows, uctx = self.user_table.lookup(user_ids, now, self.dtype)
        irows, ictx = self.item_table.lookup(item_ids, now, self.dtype)
        feats = dict(self._item_views(irows), u=urows)
        # dense forward / loss / backward
        x = self.tokens.forward(feats)
        z = self.stack.forward(x.contiguous())
        _, loss, dz, head_grads = head_fwd_bwd(self.jb, self.head, z, labels, grads_out=self.head_grads)
        dx = self.stack.backward(dz, on_layer_done=on_layer_done)
        ditem = torch.empty_like(irows)
        dfeats, token_grads = self.tokens.backward(dx, out=self._item_views(ditem), grads_out=self.token_grads)
        if aggregator is not None:
            aggregator.on_layer_done(-1, self.dense_flat)
        # sparse updates on the owners (row gradients summed over every rank by the all-to-all)
        lr = self.lr_sparse * self.grad_scale
        self.user_table.backward_sgd(dfeats["u"], uctx, lr)
        self.item_table.backward_sgd(ditem, ictx, lr)
        if aggregator is not None:
            aggregator.finish(self.stack.grad_flat, self.dense_flat)
        return loss, {"head": head_grads, "tokens": token_grads, "layers": self.stack.grads}
