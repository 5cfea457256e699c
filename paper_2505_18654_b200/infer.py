"""Inference fast path.

MTGR serves one *request* per user: the user's compressed sequence
`[U profile | S lifelong | R real-time | K candidates]` (Eq.3/Eq.4) runs once through the
encoder and the K candidate rows are the outputs scored downstream ("the user's
behaviour sequence is shared by all candidates").  The dynamic mask makes every candidate see
only the user prefix and itself, so inside the layer the candidates are pure queries:
libmtgr never loads candidate keys (R#9 diagonal term instead), i.e. the K candidates cost
`K x (n_s + n_r)` attention work on top of the prefix, not `(prefix + K)^2`.

`InferenceSession` is the serving wrapper around the same C ABI:
* forward only (`mtgr_hstu_layer_fwd` with `saved = NULL`), ping-pong activation buffers,
  one workspace;
* the whole L-layer forward is captured once per request shape into a CUDA graph and replayed
  (one launch per request instead of ~8 per layer);
* requests are copied into static device buffers (metadata + X) before each replay;
* a batch of several users is one request shape as well (throughput mode).

This module only marshals tensors; every step runs in libmtgr's kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api


class InferenceSession:
    """Graph-captured L-layer HSTU forward over one fixed jagged shape."""

    def __init__(self, cfg: api.LayerCfg, params: list, dtype: torch.dtype, device, seg4, ts=None):
        """params: per-layer device parameter dicts (`api.params_to_device`).  seg4 [B][4] host
        (nU, nS, nR, K per user) fixes the request shape; ts (host int64 [T]) the timestamps."""
        self.cfg, self.params, self.dtype, self.device = cfg, params, dtype, device
        seg4 = np.asarray(seg4, dtype=np.int32)
        T = int(seg4.astype(np.int64).sum())
        if ts is None:
            ts = np.zeros(T, dtype=np.int64)
        self.jb = api.JaggedBatch.build(seg4, ts, device)
        self.T, self.d = self.jb.total_tokens, cfg.d_model
        self.x = torch.zeros(max(self.T, 1), self.d, dtype=dtype, device=device)
        self.bufs = [torch.empty_like(self.x) for _ in range(2)]
        # forward-only scratch (no backward score scratch)
        self.ws = api._ws(api.layer_fwd_workspace_bytes(cfg, self.jb, dtype, inference=True), device)
        self.graph = None
        self.out = None
        # candidate rows of each user (the scored outputs): [offsets[u] + n_s + n_r, offsets[u+1])
        off = self.jb.host["offsets"]
        kv = self.jb.host["n_static"] + self.jb.host["n_rt"]
        self.cand_rows = np.concatenate([np.arange(off[u] + kv[u], off[u + 1]) for u in range(len(kv))]) \
            if len(kv) else np.zeros(0, np.int64)
        self._cand_idx = torch.from_numpy(self.cand_rows.astype(np.int64)).to(device)

    def _forward(self):
        cur = self.x
        for li, P in enumerate(self.params):
            out = self.bufs[li % 2]
            api.hstu_layer_fwd(self.cfg, self.jb, P, cur, out, saved=None, ws=self.ws)
            cur = out
        return cur

    def capture(self):
        """Warm up (first-call allocations, tensor-map encodes) and capture the forward."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self._forward()  # warm-up outside the graph
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = self._forward()
        return self

    def set_request(self, x: torch.Tensor, ts=None):
        """Copy a request's token features (and timestamps) into the static buffers."""
        assert x.shape == (self.T, self.d)
        self.x[:self.T].copy_(x, non_blocking=True)
        if ts is not None:
            self.jb.ts.copy_(torch.as_tensor(np.asarray(ts, np.int64)), non_blocking=True)

    def run(self) -> torch.Tensor:
        """Replay the captured forward; returns the full output [T][d] (a view of a static
        buffer, valid until the next replay)."""
        if self.graph is None:
            self.capture()
        self.graph.replay()
        return self.out[:self.T]

    def candidates(self) -> torch.Tensor:
        """The scored rows (every user's K candidate outputs), gathered [sum K][d]."""
        return self.out.index_select(0, self._cand_idx)
