"""ctypes declarations of include/mtgr.h and the loader of the in-tree libmtgr.so.

Argument marshalling only: every step of the hot path runs inside libmtgr.  There is no
fallback — if the shared library is missing the import of the operations fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_float, c_int32, c_int64, c_size_t, c_void_p, c_char_p, c_uint8

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmtgr.so")
# A/B measurements only: another in-tree build of the same ABI (e.g. libmtgr_ab.so)
if os.environ.get("MTGR_LIBRARY"):
    LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.path.basename(os.environ["MTGR_LIBRARY"]))

MTGR_F32, MTGR_BF16 = 0, 1
STATUS = {0: "MTGR_OK", 1: "MTGR_E_ARG", 2: "MTGR_E_SHAPE", 3: "MTGR_E_LAYOUT", 4: "MTGR_E_DTYPE",
          5: "MTGR_E_WORKSPACE", 6: "MTGR_E_BUDGET", 7: "MTGR_E_UNSUPPORTED", 8: "MTGR_E_CUDA",
          9: "MTGR_E_INVALID"}


class MtgrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Jagged(ctypes.Structure):
    _fields_ = [("num_users", c_int32), ("total_tokens", c_int32), ("max_len", c_int32),
                ("offsets", c_void_p), ("n_static", c_void_p), ("n_rt", c_void_p),
                ("n_cand", c_void_p), ("group_id", c_void_p), ("ts", c_void_p),
                ("inv_norm", c_void_p)]


class LayerCfg(ctypes.Structure):
    _fields_ = [("d_model", c_int32), ("n_heads", c_int32), ("num_groups", c_int32),
                ("rab_buckets", c_int32), ("eps", c_float), ("qkvu_silu", c_int32),
                ("mask_mode", c_int32), ("post_mlp_layers", c_int32)]


_PNAMES = ("w1", "b1", "w2", "b2", "gamma1", "beta1", "gamma2", "beta2", "rab_w", "w3", "b3")


class LayerParams(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in _PNAMES]


class LayerGrads(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in _PNAMES]


class HeadCfg(ctypes.Structure):
    _fields_ = [("d_model", c_int32), ("d_hidden", c_int32)]


_HNAMES = ("w_a", "b_a", "w_b", "b_b")


class HeadParams(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in _HNAMES]


class HeadGrads(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in _HNAMES]


class TokenCfg(ctypes.Structure):
    _fields_ = [("d_model", c_int32), ("k_s", c_int32), ("k_r", c_int32), ("k_c", c_int32)]


_MNAMES = ("w1", "b1", "w2", "b2")


class MlpParams(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in _MNAMES]


class TokenParams(ctypes.Structure):
    _fields_ = [("s", MlpParams), ("r", MlpParams), ("c", MlpParams)]


class TokenGrads(ctypes.Structure):  # mtgr_mlp_grads_t has the same layout as MlpParams
    _fields_ = [("s", MlpParams), ("r", MlpParams), ("c", MlpParams)]


class HashTable(ctypes.Structure):
    _fields_ = [("keys", c_void_p), ("slots", c_void_p), ("cap_k", c_int64), ("values", c_void_p),
                ("counter", c_void_p), ("ts", c_void_p), ("slot_key", c_void_p), ("cap_v", c_int64),
                ("dim", c_int32), ("alloc", c_void_p), ("free_stack", c_void_p), ("seed", ctypes.c_uint64),
                ("init_scale", c_float)]


# name -> (restype, argtypes); mirrors include/mtgr.h
_S = c_int32  # mtgr_status_t
_P = c_void_p
SIGNATURES = {
    "mtgr_status_str": (c_char_p, [c_int32]),
    "mtgr_last_error": (c_char_p, []),
    "mtgr_version": (c_int32, []),
    "mtgr_build_jagged": (_S, [_P, c_int32, _P, c_int32, _P, _P, _P, _P, _P]),
    "mtgr_balance_lpt": (_S, [_P, c_int32, c_int32, c_int64, _P, _P]),
    "mtgr_validate_jagged": (_S, [POINTER(Jagged), c_int32, _P]),
    "mtgr_mask_dense": (_S, [POINTER(Jagged), c_int32, _P, _P]),
    "mtgr_gln_fwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, _P, _P, _P, _P, _P, _P, _P]),
    "mtgr_gln_bwd_workspace_bytes": (c_size_t, [POINTER(LayerCfg), POINTER(Jagged)]),
    "mtgr_gln_bwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, _P, _P, _P, _P, _P, _P, _P,
                          _P, _P, c_size_t, _P]),
    "mtgr_attn_workspace_bytes": (c_size_t, [POINTER(LayerCfg), POINTER(Jagged), c_int32]),
    "mtgr_hstu_attn_fwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, _P, _P, _P, c_int64,
                                _P, _P, _P, _P, _P, c_size_t, _P]),
    "mtgr_hstu_attn_bwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, _P, _P, _P, _P,
                                c_int64, _P, _P, _P, _P, _P, c_int64, _P, _P, c_size_t, _P]),
    "mtgr_layer_saved_bytes": (c_size_t, [POINTER(LayerCfg), c_int32, c_int32]),
    "mtgr_layer_workspace_bytes": (c_size_t, [POINTER(LayerCfg), POINTER(Jagged), c_int32]),
    "mtgr_layer_fwd_workspace_bytes": (c_size_t, [POINTER(LayerCfg), POINTER(Jagged), c_int32, c_int32]),
    "mtgr_hstu_layer_fwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, POINTER(LayerParams),
                                 _P, _P, _P, _P, c_size_t, _P]),
    "mtgr_hstu_layer_bwd": (_S, [POINTER(LayerCfg), POINTER(Jagged), c_int32, POINTER(LayerParams),
                                 _P, _P, _P, _P, POINTER(LayerGrads), c_int32, _P, c_size_t, _P]),
    "mtgr_scale_f32": (_S, [_P, c_int64, c_float, _P]),
    "mtgr_gemm": (_S, [c_int32, c_int32, c_int32, c_int32, _P, c_int64, c_int32, _P, c_int64,
                       c_int32, _P, c_int64, c_int32, _P, c_int32, _P, c_size_t, _P]),
    "mtgr_gemm_workspace_bytes": (c_size_t, [c_int32, c_int32, c_int32, c_int32, c_int32]),
    "mtgr_head_workspace_bytes": (c_size_t, [POINTER(HeadCfg), POINTER(Jagged), c_int32, c_int32]),
    "mtgr_head_fwd_bwd": (_S, [POINTER(HeadCfg), POINTER(Jagged), c_int32, c_int32, POINTER(HeadParams),
                               _P, _P, _P, _P, _P, POINTER(HeadGrads), _P, c_size_t, _P]),
    "mtgr_token_saved_bytes": (c_size_t, [POINTER(TokenCfg), _P, c_int32]),
    "mtgr_token_workspace_bytes": (c_size_t, [POINTER(TokenCfg), POINTER(Jagged), _P, c_int32]),
    "mtgr_token_fwd": (_S, [POINTER(TokenCfg), POINTER(Jagged), _P, _P, c_int32, POINTER(TokenParams),
                            _P, _P, _P, _P, _P, _P, _P, c_size_t, _P]),
    "mtgr_token_bwd": (_S, [POINTER(TokenCfg), POINTER(Jagged), _P, _P, c_int32, POINTER(TokenParams),
                            _P, _P, _P, _P, _P, _P, _P, _P, _P, POINTER(TokenGrads), _P, c_size_t, _P]),
    "mtgr_hash_init": (_S, [POINTER(HashTable), _P]),
    "mtgr_hash_find_or_insert": (_S, [POINTER(HashTable), _P, c_int32, c_int64, c_int32, _P, _P]),
    "mtgr_hash_gather": (_S, [POINTER(HashTable), _P, c_int32, c_int32, _P, _P]),
    "mtgr_hash_sgd": (_S, [POINTER(HashTable), _P, c_int32, c_int32, _P, c_float, _P]),
    "mtgr_hash_evict": (_S, [POINTER(HashTable), c_int64, _P]),
    "mtgr_hash_expand": (_S, [POINTER(HashTable), _P, _P, c_int64, _P]),
    "mtgr_unique_workspace_bytes": (c_size_t, [c_int32]),
    "mtgr_unique": (_S, [_P, c_int32, _P, _P, _P, _P, c_size_t, _P]),
    "mtgr_segment_sum": (_S, [c_int32, _P, _P, c_int32, c_int32, _P, c_int32, _P]),
    "mtgr_take_rows": (_S, [c_int32, _P, _P, c_int32, c_int32, _P, _P]),
    "mtgr_put_rows": (_S, [c_int32, _P, _P, c_int32, c_int32, _P, _P]),
    "mtgr_partition_ids": (_S, [_P, c_int32, c_int32, ctypes.c_uint64, _P, _P, _P, _P, _P, _P]),
    "mtgr_launch_count": (c_int64, []),
    "mtgr_prof_enable": (None, [c_int32]),
    "mtgr_prof_reset": (None, []),
    "mtgr_prof_num_kinds": (c_int32, []),
    "mtgr_prof_kind_name": (c_char_p, [c_int32]),
    "mtgr_prof_query": (_S, [c_int32, POINTER(c_int64), POINTER(ctypes.c_double)]),
}

_lib = None


def lib():
    """Load libmtgr.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libmtgr.so not found at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        msg = lib().mtgr_last_error().decode(errors="replace")
        raise MtgrError(status, msg)
