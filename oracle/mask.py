"""Dynamic mask of MTGR (§4.2 "Dynamic Masking"; Fig.2(c) caption P:274).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Three rules:
  1. "The static sequence is visible to all tokens."
  2. "The visibility of the dynamic sequence adheres to causality, where each
     token is only visible to tokens that occur afterward, which include
     candidate tokens."
  3. "Candidate tokens (C, I) is visible to itself only."
Readings: R#8 static rows read static columns only (Fig.2(c)
white square); R#9 the diagonal is always visible; R#10 strict '<' on
timestamps (equal-time real-time tokens are invisible); R#12 the predicate
uses timestamps only, never token order.
"""
from __future__ import annotations

import numpy as np

STATIC, REALTIME, CANDIDATE = 0, 1, 2


def mask_dense(n_s: int, n_r: int, n_c: int, ts: np.ndarray) -> np.ndarray:
    """m[i, j] = 1 iff token i (reader, row) may read token j (column).  uint8 [L][L].

    User-local layout [static n_s | real-time n_r | candidates n_c] (Eq.3-4).
      i <  n_s : m_ij = [j < n_s]                                   (rule 1 + R#8)
      i >= n_s : m_ij = [j < n_s] or [i == j]
                         or [n_s <= j < n_s+n_r and ts_j < ts_i]     (rules 1-3, R#9, R#10)
    """
    L = n_s + n_r + n_c
    ts = np.asarray(ts, dtype=np.int64)
    assert ts.shape == (L,)
    i = np.arange(L)[:, None]          # reader (row)
    j = np.arange(L)[None, :]          # read token (column)
    static_col = j < n_s
    rt_col = (j >= n_s) & (j < n_s + n_r)
    earlier = ts[None, :] < ts[:, None]  # ts_j < ts_i
    m = np.where(i < n_s, static_col, static_col | (i == j) | (rt_col & earlier))
    m = m.astype(np.uint8)
    return m


def mask_causal(L: int) -> np.ndarray:
    """The plain causal mask over the packed order, m[i, j] = [j <= i]  (uint8 [L][L]).

    HSTU's mask, which MTGR replaces ("utilizes the causal mask for sequence
    modeling ... Using a simple causal mask in MTGR could result in information leakage");
    Table 4's "w/o dynamic mask" ablation.  Candidates read every earlier candidate.
    """
    i = np.arange(L)[:, None]
    j = np.arange(L)[None, :]
    return (j <= i).astype(np.uint8)


def mask_full(n_s: int, n_r: int, n_c: int) -> np.ndarray:
    """Table 4's "w/o dynamic mask" ablation read as FULL attention, the second reading
    SPEC lists: the dynamic mask is removed, "except candidate diagonal rule is
    retained to keep the task well-posed".  uint8 [L][L]:
        m_ij = [j < n_s + n_r]  or  [i == j]
    every static and real-time token is visible to every token (no timestamps consulted);
    candidate tokens are visible to themselves only (rule 3).
    """
    L = n_s + n_r + n_c
    i = np.arange(L)[:, None]
    j = np.arange(L)[None, :]
    return ((j < n_s + n_r) | (i == j)).astype(np.uint8)


MASK_MODES = ("dynamic", "causal", "full")


def mask_for(mode: str, n_s: int, n_r: int, n_c: int, ts) -> np.ndarray:
    """Mask of a user under `mode` (layer config mask_mode; include/mtgr.h MTGR_MASK_*)."""
    if mode == "dynamic":
        return mask_dense(n_s, n_r, n_c, ts)
    if mode == "causal":
        return mask_causal(n_s + n_r + n_c)
    if mode == "full":
        return mask_full(n_s, n_r, n_c)
    raise ValueError(mode)


def mask_rules_pairwise(kinds, ts) -> np.ndarray:
    """Rule interpreter: evaluates the three textual rules pairwise from token kinds.

    kinds[t] in {STATIC, REALTIME, CANDIDATE}; the layout order is NOT assumed
    (the rules speak of token kinds and times only).
    Column j visible to row i iff
      * j static and i static                 (rule 1, static square of Fig.2(c), R#8)
      * j static and i not static             (rule 1)
      * j real-time, i not static, j occurred before i   (rule 2, "occur afterward", R#10)
      * i == j                                (rule 3 for candidates, R#9 for all)
    Candidate columns are visible to nobody but themselves (rule 3).
    """
    n = len(kinds)
    m = np.zeros((n, n), dtype=np.uint8)
    for i in range(n):
        for j in range(n):
            if i == j:
                m[i, j] = 1
            elif kinds[j] == STATIC:
                m[i, j] = 1
            elif kinds[j] == REALTIME:
                m[i, j] = 1 if (kinds[i] != STATIC and ts[j] < ts[i]) else 0
            else:
                m[i, j] = 0
    return m


def rab_bucket(dt: np.ndarray, n_buckets: int) -> np.ndarray:
    """Relative-time bucket (R#4, not in the paper): min(NB-1, floor(log2(max(|dt|, 1))))."""
    a = np.maximum(np.abs(np.asarray(dt, dtype=np.int64)), 1)
    # floor(log2(a)) exactly for integers: a = m * 2^e with m in [0.5, 1)  ->  e - 1
    _, e = np.frexp(a.astype(np.float64))
    return np.minimum(n_buckets - 1, e.astype(np.int64) - 1)
