"""Thin Python binding of libmtgr with the C ABI's names (argument marshalling only).

PyTorch supplies device memory, streams and process groups; every arithmetic step runs in
libmtgr's CUDA kernels.  Tensors must live on the current CUDA device.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (Jagged, LayerCfg, LayerParams, LayerGrads, HeadCfg, HeadParams, HeadGrads, TokenCfg,
                   MlpParams, TokenParams, TokenGrads, check, lib, MTGR_F32, MTGR_BF16)


def _dt(t: torch.dtype) -> int:
    if t == torch.float32:
        return MTGR_F32
    if t == torch.bfloat16:
        return MTGR_BF16
    raise TypeError(f"unsupported dtype {t}")


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _np(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ host integer artefacts

def build_jagged(seg4: np.ndarray, users=None):
    """mtgr_build_jagged: returns dict(offsets, n_static, n_rt, n_cand, group_id) numpy arrays."""
    seg4 = np.ascontiguousarray(seg4, dtype=np.int32).reshape(-1, 4)
    n = seg4.shape[0]
    us = None if users is None else np.ascontiguousarray(users, dtype=np.int32)
    m = n if us is None else us.shape[0]
    idx = np.arange(n) if us is None else us
    T = int(seg4[idx].astype(np.int64).sum()) if m else 0
    out = dict(offsets=np.zeros(m + 1, np.int32), n_static=np.zeros(m, np.int32),
               n_rt=np.zeros(m, np.int32), n_cand=np.zeros(m, np.int32),
               group_id=np.zeros(max(T, 1), np.uint8))
    check(lib().mtgr_build_jagged(_np(seg4), n, _np(us), m, _np(out["offsets"]),
                                  _np(out["n_static"]), _np(out["n_rt"]), _np(out["n_cand"]),
                                  _np(out["group_id"])))
    out["group_id"] = out["group_id"][:T]
    return out


def balance_lpt(cost, world: int, cap: int = 0):
    """mtgr_balance_lpt: returns (rank_of int32 [n], load int64 [world])."""
    cost = np.ascontiguousarray(cost, dtype=np.int64)
    rank_of = np.zeros(cost.shape[0], np.int32)
    load = np.zeros(world, np.int64)
    check(lib().mtgr_balance_lpt(_np(cost), cost.shape[0], world, cap, _np(rank_of), _np(load)))
    return rank_of, load


# ------------------------------------------------------------------ jagged batch on device

@dataclass
class JaggedBatch:
    """Device-resident jagged metadata (mtgr_jagged_t) of one rank's batch."""
    offsets: torch.Tensor
    n_static: torch.Tensor
    n_rt: torch.Tensor
    n_cand: torch.Tensor
    group_id: torch.Tensor
    ts: torch.Tensor
    inv_norm: torch.Tensor | None
    num_users: int
    total_tokens: int
    max_len: int
    host: dict = field(default_factory=dict)

    @staticmethod
    def build(seg4, ts, device, users=None, inv_norm=None):
        """seg4 [n][4] host; ts: host int64 [T] of the packed users (in `users` order)."""
        h = build_jagged(seg4, users)
        T = int(h["offsets"][-1])
        ts = np.ascontiguousarray(ts, dtype=np.int64)
        assert ts.shape == (T,), (ts.shape, T)
        L = np.diff(h["offsets"])
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return JaggedBatch(
            offsets=dev(h["offsets"]), n_static=dev(h["n_static"]), n_rt=dev(h["n_rt"]),
            n_cand=dev(h["n_cand"]), group_id=dev(h["group_id"]) if T else torch.zeros(1, dtype=torch.uint8, device=device),
            ts=dev(ts) if T else torch.zeros(1, dtype=torch.int64, device=device),
            inv_norm=None if inv_norm is None else dev(np.asarray(inv_norm, np.float32)),
            num_users=len(L), total_tokens=T, max_len=int(L.max()) if len(L) else 0,
            host=dict(h, ts=ts))

    def c(self) -> Jagged:
        return Jagged(self.num_users, self.total_tokens, self.max_len,
                      self.offsets.data_ptr(), self.n_static.data_ptr(), self.n_rt.data_ptr(),
                      self.n_cand.data_ptr(), self.group_id.data_ptr(), self.ts.data_ptr(),
                      None if self.inv_norm is None else self.inv_norm.data_ptr())


MASK_MODES = {"dynamic": 0, "causal": 1, "full": 2}  # include/mtgr.h MTGR_MASK_*


def layer_cfg(d_model, n_heads, num_groups=4, rab_buckets=0, eps=1e-6, qkvu_silu=True,
              mask_mode="dynamic", post_mlp_layers=1) -> LayerCfg:
    return LayerCfg(d_model, n_heads, num_groups, rab_buckets, eps, 1 if qkvu_silu else 0,
                    MASK_MODES[mask_mode], post_mlp_layers)


def validate_jagged(jb: JaggedBatch, num_groups: int):
    j = jb.c()
    check(lib().mtgr_validate_jagged(ctypes.byref(j), num_groups, _stream()))


def mask_dense(jb: JaggedBatch, user: int) -> torch.Tensor:
    L = int(jb.host["offsets"][user + 1] - jb.host["offsets"][user])
    out = torch.empty(max(L * L, 1), dtype=torch.uint8, device=jb.offsets.device)
    j = jb.c()
    check(lib().mtgr_mask_dense(ctypes.byref(j), user, _p(out), _stream()))
    return out[:L * L].view(L, L)


# ------------------------------------------------------------------ GLN

def gln_fwd(cfg: LayerCfg, jb: JaggedBatch, x, gamma, beta):
    y = torch.empty_like(x)
    mean = torch.empty(max(jb.total_tokens, 1), dtype=torch.float32, device=x.device)
    rstd = torch.empty_like(mean)
    j = jb.c()
    check(lib().mtgr_gln_fwd(ctypes.byref(cfg), ctypes.byref(j), _dt(x.dtype), _p(x), _p(gamma),
                             _p(beta), _p(y), _p(mean), _p(rstd), _stream()))
    return y, mean[:jb.total_tokens], rstd[:jb.total_tokens]


def gln_bwd(cfg: LayerCfg, jb: JaggedBatch, dy, x, mean, rstd, gamma):
    dx = torch.empty_like(x)
    dgamma = torch.empty_like(gamma)
    dbeta = torch.empty_like(gamma)
    j = jb.c()
    nb = lib().mtgr_gln_bwd_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j))
    ws = _ws(nb, x.device)
    check(lib().mtgr_gln_bwd(ctypes.byref(cfg), ctypes.byref(j), _dt(x.dtype), _p(dy), _p(x),
                             _p(mean), _p(rstd), _p(gamma), _p(dx), _p(dgamma), _p(dbeta),
                             _p(ws), ws.numel(), _stream()))
    return dx, dgamma, dbeta


# ------------------------------------------------------------------ attention

def attn_fwd(cfg: LayerCfg, jb: JaggedBatch, q, k, v, ld, u=None, rab_w=None):
    """q, k, v, u: tensors whose data_ptr is the start of the Q/K/V/U block (row stride ld)."""
    T, d = jb.total_tokens, cfg.d_model
    o = torch.empty(max(T, 1), d, dtype=q.dtype, device=q.device)
    y = torch.empty_like(o) if u is not None else None
    j = jb.c()
    ws = _ws(lib().mtgr_attn_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j), _dt(q.dtype)), q.device)
    check(lib().mtgr_hstu_attn_fwd(ctypes.byref(cfg), ctypes.byref(j), _dt(q.dtype), _p(q), _p(k),
                                   _p(v), ld, _p(u), _p(rab_w), _p(o), _p(y), _p(ws), ws.numel(),
                                   _stream()))
    return o[:T], (None if y is None else y[:T])


def attn_bwd(cfg: LayerCfg, jb: JaggedBatch, dO, q, k, v, ld, rab_w=None, silu_pre=None):
    T, d = jb.total_tokens, cfg.d_model
    dq = torch.empty(max(T, 1), d, dtype=q.dtype, device=q.device)
    dk = torch.empty_like(dq)
    dv = torch.empty_like(dq)
    drab = None
    if cfg.rab_buckets > 0:
        drab = torch.zeros(cfg.n_heads, cfg.rab_buckets, dtype=torch.float32, device=q.device)
    j = jb.c()
    ws = _ws(lib().mtgr_attn_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j), _dt(q.dtype)), q.device)
    check(lib().mtgr_hstu_attn_bwd(ctypes.byref(cfg), ctypes.byref(j), _dt(q.dtype), _p(dO), _p(q),
                                   _p(k), _p(v), ld, _p(rab_w), _p(silu_pre), _p(dq), _p(dk),
                                   _p(dv), d, _p(drab), _p(ws), ws.numel(), _stream()))
    return dq[:T], dk[:T], dv[:T], drab


# ------------------------------------------------------------------ layer

PARAM_KEYS = ("W1", "b1", "W2", "b2", "gamma1", "beta1", "gamma2", "beta2", "rab_w", "W3", "b3")
_C_NAMES = dict(W1="w1", b1="b1", W2="w2", b2="b2", gamma1="gamma1", beta1="beta1",
                gamma2="gamma2", beta2="beta2", rab_w="rab_w", W3="w3", b3="b3")


def params_to_device(p: dict, dtype: torch.dtype, device) -> dict:
    """W1/W2 in the activation dtype, everything else fp32 (mtgr_layer_params_t)."""
    out = {}
    for k, v in p.items():
        t = torch.as_tensor(np.asarray(v, dtype=np.float32))
        out[k] = t.to(device=device, dtype=dtype if k in ("W1", "W2", "W3") else torch.float32).contiguous()
    return out


def _cparams(p: dict) -> LayerParams:
    return LayerParams(*[(p[k].data_ptr() if p.get(k) is not None else None) for k in PARAM_KEYS])


def grad_numel(cfg: LayerCfg) -> int:
    d, G = cfg.d_model, cfg.num_groups
    return (5 * d * d + 5 * d + 4 * G * d + (cfg.n_heads * cfg.rab_buckets if cfg.rab_buckets > 0 else 0)
            + (d * d + d if cfg.post_mlp_layers == 2 else 0))


def alloc_grads(cfg: LayerCfg, device, flat: torch.Tensor | None = None) -> dict:
    """fp32 gradient views (mtgr_layer_grads_t) carved from one flat bucket (all-reduce unit)."""
    d, G = cfg.d_model, cfg.num_groups
    if flat is None:
        flat = torch.zeros(grad_numel(cfg), dtype=torch.float32, device=device)
    shapes = dict(W1=(4 * d, d), b1=(4 * d,), W2=(d, d), b2=(d,), gamma1=(G, d), beta1=(G, d),
                  gamma2=(G, d), beta2=(G, d))
    if cfg.rab_buckets > 0:
        shapes["rab_w"] = (cfg.n_heads, cfg.rab_buckets)
    if cfg.post_mlp_layers == 2:
        shapes["W3"], shapes["b3"] = (d, d), (d,)
    g, off = {}, 0
    for k, shp in shapes.items():
        n = int(np.prod(shp))
        g[k] = flat[off:off + n].view(*shp)
        off += n
    assert off == flat.numel()
    g["_flat"] = flat
    return g


def _cgrads(g: dict) -> LayerGrads:  # noqa: E302
    return LayerGrads(*[(g[k].data_ptr() if g.get(k) is not None else None) for k in PARAM_KEYS])


def layer_saved_bytes(cfg: LayerCfg, total_tokens: int, dtype: torch.dtype) -> int:
    return lib().mtgr_layer_saved_bytes(ctypes.byref(cfg), total_tokens, _dt(dtype))


def layer_workspace_bytes(cfg: LayerCfg, jb: JaggedBatch, dtype: torch.dtype) -> int:
    j = jb.c()
    return lib().mtgr_layer_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j), _dt(dtype))


def layer_fwd_workspace_bytes(cfg: LayerCfg, jb: JaggedBatch, dtype: torch.dtype, inference: bool) -> int:
    """Forward-only scratch (mtgr_layer_fwd_workspace_bytes): no backward score scratch; with
    inference = True it includes the per-layer intermediates that `saved` would hold."""
    j = jb.c()
    return lib().mtgr_layer_fwd_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j), _dt(dtype), 1 if inference else 0)


def hstu_layer_fwd(cfg, jb, params, x, z=None, saved=None, ws=None):
    z = torch.empty_like(x) if z is None else z
    if ws is None:
        ws = _ws(layer_fwd_workspace_bytes(cfg, jb, x.dtype, saved is None), x.device)
    j = jb.c()
    cp = _cparams(params)
    check(lib().mtgr_hstu_layer_fwd(ctypes.byref(cfg), ctypes.byref(j), _dt(x.dtype), ctypes.byref(cp),
                                    _p(x), _p(z), _p(saved), _p(ws), ws.numel(), _stream()))
    return z


def hstu_layer_bwd(cfg, jb, params, x, saved, dz, grads, dx=None, accumulate=False, ws=None):
    dx = torch.empty_like(x) if dx is None else dx
    if ws is None:
        ws = _ws(layer_workspace_bytes(cfg, jb, x.dtype), x.device)
    j = jb.c()
    cp = _cparams(params)
    cg = _cgrads(grads)
    check(lib().mtgr_hstu_layer_bwd(ctypes.byref(cfg), ctypes.byref(j), _dt(x.dtype), ctypes.byref(cp),
                                    _p(x), _p(saved), _p(dz), _p(dx), ctypes.byref(cg),
                                    1 if accumulate else 0, _p(ws), ws.numel(), _stream()))
    return dx


def scale_(g: torch.Tensor, s: float):
    check(lib().mtgr_scale_f32(_p(g), g.numel(), float(s), _stream()))
    return g


def gemm(A, B, M, N, K, lda, a_kmajor, ldb, b_kmajor, C=None, ldc=None, c_f32=False, bias=None,
         accumulate=False):
    """C = A B^T through the layer's GEMM kernels (mtgr_gemm)."""
    dt = _dt(A.dtype)
    if C is None:
        C = torch.empty(M, N, dtype=torch.float32 if c_f32 else A.dtype, device=A.device)
        ldc = N
    wsb = lib().mtgr_gemm_workspace_bytes(dt, M, N, K, 1 if c_f32 else 0)
    ws = _ws(wsb, A.device)
    check(lib().mtgr_gemm(dt, M, N, K, _p(A), lda, a_kmajor, _p(B), ldb, b_kmajor, _p(C), ldc,
                          1 if c_f32 else 0, _p(bias), 1 if accumulate else 0, _p(ws), ws.numel(),
                          _stream()))
    return C


# ------------------------------------------------------------------ encoder stack runner

class HstuStack:
    """L HSTU layers with the same jagged metadata, forward and backward.

    Owns the per-layer saved buffers, a shared workspace and fp32 gradient buffers.
    """

    def __init__(self, cfg: LayerCfg, params: list, dtype: torch.dtype, device):
        self.cfg, self.params, self.dtype, self.device = cfg, params, dtype, device
        n = grad_numel(cfg)
        # one flat fp32 buffer holding every layer's gradients; per-layer slices are the
        # all-reduce buckets of data-parallel training
        self.grad_flat = torch.zeros(n * len(params), dtype=torch.float32, device=device)
        self.grads = [alloc_grads(cfg, device, self.grad_flat[i * n:(i + 1) * n]) for i in range(len(params))]
        self._jb = None
        self.saved = self.xs = self.ws = None

    def bind(self, jb: JaggedBatch):
        """Allocate activations for a batch.  Buffers are re-used while they are large enough:
        the activations depend on T, the workspace also on num_users and max_len (stored-score
        scratch), so each is checked against this batch's own requirement."""
        self._jb = jb
        T, d = max(jb.total_tokens, 1), self.cfg.d_model
        sb = layer_saved_bytes(self.cfg, jb.total_tokens, self.dtype)
        if getattr(self, "saved", None) is None or self.saved[0].numel() < sb:
            self.saved = [_ws(sb, self.device) for _ in self.params]
        if getattr(self, "xs", None) is None or self.xs[1].shape[0] < T:
            self.xs = [None] + [torch.empty(T, d, dtype=self.dtype, device=self.device) for _ in self.params]
            self.dbuf = [torch.empty(T, d, dtype=self.dtype, device=self.device) for _ in range(2)]
        wb = layer_workspace_bytes(self.cfg, jb, self.dtype)
        if getattr(self, "ws", None) is None or self.ws.numel() < wb:
            self.ws = None  # release before allocating the larger one
            self.ws = _ws(wb, self.device)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        jb = self._jb
        assert x.is_contiguous() and x.dtype == self.dtype
        self.xs[0] = x  # layer-0 input is read in place (kept alive for the backward)
        for li, P in enumerate(self.params):
            with _nvtx(f"layer{li}.fwd"):
                hstu_layer_fwd(self.cfg, jb, P, self.xs[li], self.xs[li + 1], self.saved[li], self.ws)
        return self.xs[-1][:jb.total_tokens]

    def backward(self, dz: torch.Tensor, accumulate=False, on_layer_done=None) -> torch.Tensor:
        """Backward through the stack.  on_layer_done(li, grad_bucket) is called right after
        layer li's backward is enqueued (hook for overlapping its all-reduce)."""
        jb = self._jb
        cur = dz
        for li in range(len(self.params) - 1, -1, -1):
            out = self.dbuf[li % 2]
            with _nvtx(f"layer{li}.bwd"):
                hstu_layer_bwd(self.cfg, jb, self.params[li], self.xs[li], self.saved[li], cur,
                               self.grads[li], dx=out, accumulate=accumulate, ws=self.ws)
            if on_layer_done is not None:
                on_layer_done(li, self.grads[li]["_flat"])
            cur = out
        return cur[:jb.total_tokens]


# ------------------------------------------------------------------ tracing

_NVTX = os.environ.get("MTGR_NVTX") == "1"


@contextlib.contextmanager
def _nvtx(name: str):
    """NVTX range around a layer call when MTGR_NVTX=1 (the library wraps each kernel launch in
    its own range under the same switch); a no-op otherwise."""
    if not _NVTX:
        yield
        return
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()

# ------------------------------------------------------------------ candidate head

def head_params_to_device(p: dict, dtype: torch.dtype, device) -> dict:
    """w_a in the activation dtype; b_a, w_b, b_b fp32 (include/mtgr.h mtgr_head_params_t)."""
    out = {}
    for k, v in p.items():
        t = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float32))
        out[k] = t.to(device, dtype if k == "w_a" else torch.float32).contiguous()
    return out


def head_fwd_bwd(jb: JaggedBatch, params: dict, z: torch.Tensor, labels: torch.Tensor,
                 d_hidden: int | None = None, want_grad: bool = True, ws=None, grads_out: dict | None = None):
    """Candidate logit head + CTR/CTCVR BCE sums (mtgr_head_fwd_bwd).  labels: uint8 [T]
    (bit 0 click, bit 1 purchase).  Returns (logits [K][2], loss [2], dz or None, grads or None).
    grads_out: optional preallocated fp32 gradient tensors (e.g. views of an all-reduce bucket)."""
    d = z.shape[1]
    dh = d_hidden or params["w_a"].shape[0]
    cfg = HeadCfg(d, dh)
    K = int(jb.host["n_cand"].sum()) if jb.num_users else 0
    j = jb.c()
    dt = _dt(z.dtype)
    nbytes = lib().mtgr_head_workspace_bytes(ctypes.byref(cfg), ctypes.byref(j), K, dt)
    ws = _ws(nbytes, z.device) if ws is None else ws
    logits = torch.empty((max(K, 1), 2), dtype=torch.float32, device=z.device)
    loss = torch.empty(2, dtype=torch.float32, device=z.device)
    dz = torch.empty_like(z) if want_grad else None
    grads = None
    if want_grad and grads_out is not None:
        grads = grads_out
    elif want_grad:
        grads = {"w_a": torch.empty((dh, d), dtype=torch.float32, device=z.device),
                 "b_a": torch.empty(dh, dtype=torch.float32, device=z.device),
                 "w_b": torch.empty((2, dh), dtype=torch.float32, device=z.device),
                 "b_b": torch.empty(2, dtype=torch.float32, device=z.device)}
    P = HeadParams(*(params[k].data_ptr() for k in ("w_a", "b_a", "w_b", "b_b")))
    G = HeadGrads(*(grads[k].data_ptr() for k in ("w_a", "b_a", "w_b", "b_b"))) if want_grad else None
    check(lib().mtgr_head_fwd_bwd(ctypes.byref(cfg), ctypes.byref(j), K, dt, ctypes.byref(P),
                                  _p(z), _p(labels), _p(logits), _p(loss), _p(dz),
                                  ctypes.byref(G) if G is not None else None, _p(ws), ws.numel(),
                                  _stream()))
    return logits[:K], loss, dz, grads


# ------------------------------------------------------------------ token construction

class TokenEmbed:
    """Eq.4 token construction (mtgr_token_fwd / _bwd): U rows from the given embeddings, one
    Linear-SiLU-Linear MLP per item type (S, R, candidates).  `params`: {"s","r","c"} ->
    {"w1","b1","w2","b2"} on the device (w1, w2 in the activation dtype)."""

    def __init__(self, d_model: int, widths: dict, params: dict, dtype: torch.dtype, device):
        self.cfg = TokenCfg(d_model, widths["s"], widths["r"], widths["c"])
        self.d, self.dtype, self.device = d_model, dtype, device
        self.params = params
        self._cp = TokenParams(*(MlpParams(*(params[t][k].data_ptr() for k in ("w1", "b1", "w2", "b2")))
                                 for t in ("s", "r", "c")))

    @staticmethod
    def params_to_device(p: dict, dtype: torch.dtype, device) -> dict:
        out = {}
        for t, q in p.items():
            out[t] = {k: torch.as_tensor(np.ascontiguousarray(v, dtype=np.float32)).to(
                device, dtype if k in ("w1", "w2") else torch.float32).contiguous() for k, v in q.items()}
        return out

    def bind(self, jb: JaggedBatch, seg4: np.ndarray):
        """seg4 [B][4] host (n_U, n_S, n_r, K) of the batch's users, in batch order."""
        seg4 = np.asarray(seg4, dtype=np.int64)
        self.jb = jb
        self.n_user = torch.from_numpy(np.ascontiguousarray(seg4[:, 0], dtype=np.int32)).to(self.device)
        self.n_tot = (ctypes.c_int32 * 4)(*(int(seg4[:, i].sum()) for i in range(4)))
        dt = _dt(self.dtype)
        j = jb.c()
        self.saved = _ws(lib().mtgr_token_saved_bytes(ctypes.byref(self.cfg), self.n_tot, dt), self.device)
        self.ws = _ws(lib().mtgr_token_workspace_bytes(ctypes.byref(self.cfg), ctypes.byref(j), self.n_tot, dt),
                      self.device)

    def forward(self, feats: dict) -> torch.Tensor:
        self.feats = feats
        x = torch.empty((max(self.jb.total_tokens, 1), self.d), dtype=self.dtype, device=self.device)
        j = self.jb.c()
        check(lib().mtgr_token_fwd(ctypes.byref(self.cfg), ctypes.byref(j), _p(self.n_user), self.n_tot,
                                   _dt(self.dtype), ctypes.byref(self._cp), *(_p(feats.get(t)) for t in "usrc"),
                                   _p(x), _p(self.saved), _p(self.ws), self.ws.numel(), _stream()))
        return x[:self.jb.total_tokens]

    def grad_shapes(self) -> dict:
        return {t: {"w1": tuple(self.params[t]["w1"].shape), "b1": (self.d,), "w2": (self.d, self.d), "b2": (self.d,)}
                for t in ("s", "r", "c")}

    def backward(self, dx: torch.Tensor, want_dfeats: bool = True, out: dict | None = None,
                 grads_out: dict | None = None):
        """Returns (dfeats dict or None, grads {"s","r","c"} -> {"w1","b1","w2","b2"} fp32 sums).
        `out`: optional preallocated feature-gradient tensors (e.g. views of one buffer);
        `grads_out`: optional preallocated parameter-gradient tensors (views of a bucket)."""
        f = lambda *s: torch.empty(s, dtype=torch.float32, device=self.device)
        grads = grads_out if grads_out is not None else {
            t: {k: f(*shp) for k, shp in q.items()} for t, q in self.grad_shapes().items()}
        cg = TokenGrads(*(MlpParams(*(grads[t][k].data_ptr() for k in ("w1", "b1", "w2", "b2")))
                          for t in ("s", "r", "c")))
        dfe = {}
        if want_dfeats:
            dfe = {t: (out[t] if out is not None and t in out else torch.empty_like(v))
                   for t, v in self.feats.items() if v is not None}
        j = self.jb.c()
        check(lib().mtgr_token_bwd(ctypes.byref(self.cfg), ctypes.byref(j), _p(self.n_user), self.n_tot,
                                   _dt(self.dtype), ctypes.byref(self._cp),
                                   *(_p(self.feats.get(t)) for t in "src"), _p(self.saved), _p(dx),
                                   *(_p(dfe.get(t)) for t in "usrc"), ctypes.byref(cg), _p(self.ws),
                                   self.ws.numel(), _stream()))
        return (dfe if want_dfeats else None), grads


def launch_count() -> int:
    """Kernels libmtgr has launched in this process."""
    return int(lib().mtgr_launch_count())


def prof_enable(on: bool = True):
    lib().mtgr_prof_enable(1 if on else 0)


def prof_reset():
    lib().mtgr_prof_reset()


def prof_query() -> dict:
    """{kind: (launches, total_ms)} of CUDA-event-timed kernels since the last reset."""
    out = {}
    for k in range(lib().mtgr_prof_num_kinds()):
        n = ctypes.c_int64()
        ms = ctypes.c_double()
        check(lib().mtgr_prof_query(k, ctypes.byref(n), ctypes.byref(ms)))
        if n.value:
            out[lib().mtgr_prof_kind_name(k).decode()] = (int(n.value), float(ms.value))
    return out
