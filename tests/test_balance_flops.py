"""FLOP-aware balancer cost: on a skewed batch the token-count LPT leaves the
attention work (~L_u n_s per user) unbalanced; LPT over per-user FLOPs balances what the GPUs
actually execute.  Host logic only (oracle LPT on both costs)."""
import numpy as np

import oracle
import synth
from paper_2505_18654_b200.dp import flop_cost, visible_pairs


def _flops(seg, ts, d):
    return np.array([30 * int(seg[u].sum()) * d + 12 * visible_pairs(seg[u], ts[u]) for u in range(len(seg))],
                    dtype=np.int64)


def test_visible_pairs_matches_the_dense_mask():
    cfg = synth.config("toy")
    seg = synth.gen_segments(cfg, 6)
    for u in range(len(seg)):
        ts = synth.gen_user_ts(cfg, u, seg[u])
        nU, nS, nR, K = (int(v) for v in seg[u])
        M = oracle.mask_dense(nU + nS, nR, K, ts)
        assert visible_pairs(seg[u], ts) == int(M.sum())


def test_flop_lpt_balances_flops_better_than_token_lpt():
    cfg = synth.config("large_skew", users=64)
    world = 8
    seg = synth.gen_segments(cfg, cfg["users"])
    ts = [synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))]
    work = _flops(seg, ts, cfg["d"])
    cost_f = flop_cost(seg, ts, cfg["d"])
    assert np.array_equal(cost_f, work)
    imb = {}
    for name, cost in (("tokens", seg.astype(np.int64).sum(1)), ("flops", cost_f)):
        rank_of, _ = oracle.lpt(cost, world)
        per_rank = np.bincount(rank_of, weights=work, minlength=world)
        imb[name] = per_rank.max() / per_rank.mean()
    assert imb["flops"] <= imb["tokens"] + 1e-12
    assert imb["flops"] <= 4 / 3  # Graham's bound for LPT on the balanced quantity
