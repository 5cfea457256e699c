"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the MTGR method (no mask, no norm, no
attention, no prefix sums, no balancing).  It only draws random numbers with
the shapes and distributions of the paper's workloads; both the
oracle (`oracle/`) and the CUDA path (`paper_2505_18654_b200/`) consume them.
"""
from .gen import (CONFIGS, T0, config, gen_segments, gen_user_ts, gen_user_x,
                  gen_user_dz, gen_layer_params, round_bf16, gen_user_labels, gen_head_params,
                  TOKEN_TYPES, token_widths, gen_user_features, gen_token_params,
                  EMB_DIM, features_per_token, gen_user_feature_ids)

__all__ = ["CONFIGS", "T0", "config", "gen_segments", "gen_user_ts", "gen_user_x",
           "gen_user_dz", "gen_layer_params", "round_bf16", "gen_user_labels", "gen_head_params",
           "TOKEN_TYPES", "token_widths", "gen_user_features", "gen_token_params",
           "EMB_DIM", "features_per_token", "gen_user_feature_ids"]
