"""MTGR float64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy float64 implementation of the hot path of
MTGR (arXiv 2505.18654, /root/reference/PAPER.md): Group-Layer Norm, the
dynamically masked pointwise-SiLU HSTU attention, the full layer forward and
backward, the token-count LPT balancer, the jagged batch builder and the
batch-size-weighted gradient aggregation.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_2505_18654_b200/`) and imports nothing from it; the only
module both sides use is the seeded input generator `synth/`.

Every function cites the PAPER.md passage (P:line) it follows.  Readings of
places where the paper is silent/ambiguous are listed in DESIGN.md §2 and
referenced here as R#n.

Parity pins (tests/test_oracle_*.py): Fig.2(c) worked mask (golden fixture),
textbook LayerNorm special case, closed forms (all-static user, L=2 hand
transcription), brute-force triple loops, central finite differences,
leakage / removal / permutation invariants, brute-force LPT optimum and
Graham's bound, pooled-gradient identity.
Parity unpinned against the paper (pinned only to our own definition): the
optional `rab` term (R#4), SiLU on Q/K/V/U (R#5), single-Linear post-gate MLP
(R#6), eps (R#14).
"""
from .mask import mask_dense, mask_causal, mask_full, mask_for, MASK_MODES, mask_rules_pairwise, rab_bucket
from .gln import gln_fwd, gln_bwd
from .layer import (silu, dsilu, LayerCache, layer_fwd_user, layer_bwd_user,
                    stack_fwd_user, stack_bwd_user, attn_fwd_user, attn_bwd_user)
from .balance import build_jagged, lpt, BudgetError, aggregate_sum, aggregate_weighted
from .jagged import layer_fwd_jagged, layer_bwd_jagged

__all__ = [
    "mask_dense", "mask_rules_pairwise", "rab_bucket", "gln_fwd", "gln_bwd", "silu", "dsilu",
    "LayerCache", "layer_fwd_user", "layer_bwd_user", "stack_fwd_user", "stack_bwd_user",
    "attn_fwd_user", "attn_bwd_user", "build_jagged", "lpt", "BudgetError",
    "aggregate_sum", "aggregate_weighted", "layer_fwd_jagged", "layer_bwd_jagged",
]
from .head import candidate_rows, bce_with_logits, head_fwd_bwd
from .token import mlp_fwd, mlp_bwd, tokens_user, tokens_user_bwd
from .embed import mix64, init_row, TableModel, unique_with_inverse
