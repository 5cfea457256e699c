"""B200-native MTGR hot path: jagged Group-Layer-Norm + HSTU encoder layer (arXiv 2505.18654).

The compute lives in libmtgr.so (hand-written sm_100a CUDA behind the C ABI of
include/mtgr.h); this package is the thin ctypes binding with the same names.
"""
from ._lib import MtgrError, LIB_PATH, lib, SIGNATURES
from .api import (JaggedBatch, HstuStack, layer_cfg, build_jagged, balance_lpt, validate_jagged,
                  mask_dense, gln_fwd, gln_bwd, attn_fwd, attn_bwd, hstu_layer_fwd,
                  hstu_layer_bwd, layer_saved_bytes, layer_workspace_bytes, params_to_device,
                  alloc_grads, grad_numel, scale_, gemm, launch_count, prof_enable, prof_reset,
                  prof_query, head_params_to_device, head_fwd_bwd, TokenEmbed, MASK_MODES)

__all__ = ["MtgrError", "LIB_PATH", "lib", "SIGNATURES", "JaggedBatch", "HstuStack", "layer_cfg",
           "build_jagged", "balance_lpt", "validate_jagged", "mask_dense", "gln_fwd", "gln_bwd",
           "attn_fwd", "attn_bwd", "hstu_layer_fwd", "hstu_layer_bwd", "layer_saved_bytes",
           "layer_workspace_bytes", "params_to_device", "alloc_grads", "grad_numel", "scale_", "gemm", "launch_count", "prof_enable",
           "prof_reset", "prof_query", "head_params_to_device", "head_fwd_bwd", "TokenEmbed", "MASK_MODES"]
from .embed import HashEmbedding, ShardedEmbedding, unique, segment_sum, take_rows  # noqa: E402
from .model import MTGRModel  # noqa: E402
