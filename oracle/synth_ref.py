"""Host restatement of the GPU input generators (csrc/gen.cu).

TEST INFRASTRUCTURE ONLY (see oracle/port.py).  Regenerates the R-MAT edge
lists and uniform vectors bit for bit from the same counter-based hash, so
parity tests can build the CPU oracle's input without trusting the GPU.

hash(seed, e, l) = mix64(mix64(seed) ^ (e*64 + l)), mix64 = splitmix64
finaliser, U = (hash >> 11) * 2^-53.
"""

from __future__ import annotations

import numpy as np

M1 = np.uint64(0x9E3779B97F4A7C15)
M2 = np.uint64(0xBF58476D1CE4E5B9)
M3 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    with np.errstate(over="ignore"):  # uint64 arithmetic wraps by design
        z = np.asarray(z, dtype=np.uint64) + M1
        z = (z ^ (z >> np.uint64(30))) * M2
        z = (z ^ (z >> np.uint64(27))) * M3
        return z ^ (z >> np.uint64(31))


def u01(seed_mixed, e, level):
    with np.errstate(over="ignore"):
        h = mix64(np.uint64(seed_mixed) ^ (np.asarray(e, dtype=np.uint64) * np.uint64(64) + np.uint64(level)))
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(n, seed, lo=-1.0, hi=1.0):
    sm = mix64(np.uint64(seed))
    return lo + (hi - lo) * u01(sm, np.arange(n, dtype=np.uint64), 0)


def rmat_draws(scale, draws, seed, a=0.57, b=0.19, c=0.19, lo=0, hi=None):
    """Rows, cols and values of draws [lo, hi) (before deduplication)."""
    hi = draws if hi is None else hi
    sm = mix64(np.uint64(seed))
    e = np.arange(lo, hi, dtype=np.uint64)
    ab, abc = a + b, a + b + c
    row = np.zeros(e.size, dtype=np.int64)
    col = np.zeros(e.size, dtype=np.int64)
    for level in range(scale):
        u = u01(sm, e, level)
        rb = (u >= ab).astype(np.int64)
        cb = (((u >= a) & (u < ab)) | (u >= abc)).astype(np.int64)
        row = (row << 1) | rb
        col = (col << 1) | cb
    val = 1.0 - u01(sm, e, 63)
    return row, col, val


def rmat(scale, edge_factor, seed, a=0.57, b=0.19, c=0.19):
    """Deduplicated (first draw kept) edge list in draw order."""
    draws = edge_factor << scale
    rows, cols, vals = [], [], []
    chunk = 1 << 22
    for lo in range(0, draws, chunk):
        r, cc, v = rmat_draws(scale, draws, seed, a, b, c, lo, min(draws, lo + chunk))
        rows.append(r)
        cols.append(cc)
        vals.append(v)
    row = np.concatenate(rows) if rows else np.empty(0, np.int64)
    col = np.concatenate(cols) if cols else np.empty(0, np.int64)
    val = np.concatenate(vals) if vals else np.empty(0)
    key = (row << scale) | col
    _, first = np.unique(key, return_index=True)
    first.sort()
    return row[first], col[first], val[first]
