"""Dynamic hash embedding table and sharded lookup (§5) —
TEST INFRASTRUCTURE ONLY.

The observable semantics the GPU table must reproduce (slot numbers and bucket positions are
implementation choices and are not compared):
  * a key's row starts as init(seed, key) — the counter-based generator both sides implement
    (splitmix64, below; "each side implements the same counter-based generator");
  * an SGD step subtracts lr times the summed gradient of every occurrence of the key;
  * eviction ("auxiliary metadata (e.g., counters and timestamps) required for eviction
    policies") removes every key whose last access is older than a threshold; a later lookup
    re-inserts it with a fresh init row;
  * expanding the key structure changes no row;
  * the sharded lookup with two-stage ID unique returns exactly the rows a single table
    would, whatever the number of ranks.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 output function applied to z (Steele, Lea, Flood 2014)."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def init_row(seed: int, key: int, dim: int, scale: float) -> np.ndarray:
    """init_scale * U(-1, 1), column c from mix64(seed ^ (mix64(key) + c)): 24 high bits -> [0, 1),
    computed in float32 as the kernel does (2u - 1 is exact, one rounding for the scale)."""
    hk = mix64(key & M64)
    out = np.empty(dim, dtype=np.float32)
    for c in range(dim):
        h = mix64(seed ^ ((hk + c) & M64))
        u = np.float32(h >> 40) * np.float32(1.0 / 16777216.0)
        out[c] = np.float32(scale) * (np.float32(2.0) * u - np.float32(1.0))
    return out


class TableModel:
    """Reference semantics of one table: key -> (row, last access)."""

    def __init__(self, dim: int, seed: int = 0, scale: float = 0.05):
        self.dim, self.seed, self.scale = dim, seed, scale
        self.rows: dict[int, np.ndarray] = {}
        self.last: dict[int, int] = {}

    def lookup(self, ids, now: int = 0, insert: bool = True):
        out = np.zeros((len(ids), self.dim), dtype=np.float64)
        for i, k in enumerate(int(v) for v in ids):
            if k not in self.rows:
                if not insert:
                    continue
                self.rows[k] = init_row(self.seed, k, self.dim, self.scale).astype(np.float64)
            self.last[k] = now
            out[i] = self.rows[k]
        return out

    def sgd(self, ids, grads, lr: float):
        for k, g in zip((int(v) for v in ids), np.asarray(grads, np.float64)):
            self.rows[k] = self.rows[k] - lr * g

    def evict(self, ts_before: int):
        for k in [k for k, t in self.last.items() if t < ts_before]:
            del self.rows[k], self.last[k]


def unique_with_inverse(ids):
    """Distinct ids and the inverse map (np.unique: sorted order)."""
    u, inv = np.unique(np.asarray(ids, dtype=np.int64), return_inverse=True)
    return u, inv
