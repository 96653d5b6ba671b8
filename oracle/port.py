"""CPU oracle: a numpy restatement of the reference's hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import this
module, and only as the checker or the timed CPU baseline — never as part
of the product path (the product, ``paper_1805_11938_b200``, has no CPU
fallback).

Each function restates the algorithm of the reference package ``spmvkit``
(/root/reference/pkg/src/spmvkit/, cited file:line) in plain numpy.  The
arithmetic the reference delegates to numpy 2.3 (lexsort, add.reduceat =
first + pairwise(rest), bincount = sequential from 0.0, add.reduce =
0 + pairwise(all)) is used the same way here, so results agree bit for bit.

Parity pin: this module is checked against (1) the reference's own golden
vectors (Table-1 demo arrays, tests/test_oracle.py) and (2) fixtures that
the reference itself produced in this container
(tests/golden/make_golden.py -> tests/golden/*.npz).

Host-side threading mirrors the reference's task runtime (kernels.py:42-66):
``workers`` threads over row blocks / tiles, partials folded in ascending
task order, so the timed CPU baseline has the reference's structure.
"""

from __future__ import annotations

import concurrent.futures
import os
from dataclasses import dataclass

import numpy as np

TAGS = ("csr", "csr5", "ell", "sell", "hyb")
DEFAULT_MAX_GRID_CELLS = 1 << 26


class GridTooLarge(RuntimeError):
    """Stands for spmvkit.formats.ConversionError."""


# --------------------------------------------------------------------- COO --
def canonicalize(row, col, data, n_rows, n_cols):
    """coo.py:86-125 — lexsort (row, col), reduceat sums, drop == 0.0."""
    row = np.asarray(row, dtype=np.int64).ravel()
    col = np.asarray(col, dtype=np.int64).ravel()
    data = np.asarray(data, dtype=np.float64).ravel()
    if not (row.shape == col.shape == data.shape):
        raise ValueError("triplet arrays disagree in length")
    if row.size == 0:
        return row.copy(), col.copy(), data.copy()
    bad = (row < 0) | (row >= n_rows) | (col < 0) | (col >= n_cols)
    if bad.any():
        i = int(np.argmax(bad))
        raise ValueError(f"entry {i} at ({row[i]}, {col[i]}) is outside {n_rows}x{n_cols}")
    order = np.lexsort((col, row))
    r, c, v = row[order], col[order], data[order]
    new = np.ones(r.size, dtype=bool)
    new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    heads = np.nonzero(new)[0]
    sums = np.add.reduceat(v, heads)
    nz = sums != 0.0
    return r[heads][nz], c[heads][nz], sums[nz]


def row_counts(row, n_rows):
    """coo.py:144-146."""
    return np.bincount(np.asarray(row, dtype=np.int64), minlength=n_rows).astype(np.int64)


def dense_spmv_oracle(row, col, data, n_rows, x):
    """coo.py:128-141 — y_i accumulated entry by entry in (row, col) order.

    Vectorised over rows: slot j of every row is added in step j, which is
    the same per-row sequence of roundings as the reference's loop."""
    row = np.asarray(row, dtype=np.int64)
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(n_rows, dtype=np.float64)
    if row.size == 0:
        return y
    counts = row_counts(row, n_rows)
    ptr = np.concatenate([[0], np.cumsum(counts)])
    prod = np.asarray(data, dtype=np.float64) * x[np.asarray(col, dtype=np.int64)]
    rows = np.nonzero(counts)[0]
    j = 0
    while rows.size:
        y[rows] += prod[ptr[rows] + j]
        j += 1
        rows = rows[counts[rows] > j]
    return y


# ----------------------------------------------------------------- formats --
def to_csr(row, col, data, n_rows):
    """formats.py:183-188."""
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(row_counts(row, n_rows), out=ptr[1:])
    return ptr, np.asarray(col, dtype=np.int64).copy(), np.asarray(data, dtype=np.float64).copy()


def csr5_stored_positions(nnz, omega, sigma):
    """Stored slot of every CSR-order entry (formats.py:204-209), closed form
    base + gi*q + min(gi, rem) + gj (q, rem from the tile's fill m)."""
    tile = omega * sigma
    k = np.arange(nnz, dtype=np.int64)
    base = (k // tile) * tile
    p = k - base
    m = np.minimum(tile, nnz - base)
    q, rem = m // sigma, m % sigma
    gi, gj = p % sigma, p // sigma
    return base + gi * q + np.minimum(gi, rem) + gj


@dataclass
class Csr5:
    ptr: np.ndarray
    omega: int
    sigma: int
    num_tiles: int
    tile_ptr: np.ndarray
    bit_flag: np.ndarray
    y_off: np.ndarray
    seg_off: np.ndarray
    indices: np.ndarray
    data: np.ndarray


def to_csr5(ptr, indices, data, n_rows, omega, sigma):
    """formats.py:196-250 restated without the per-tile Python loop."""
    if omega < 1 or sigma < 1:
        raise ValueError(f"omega and sigma must be >= 1, got {omega}, {sigma}")
    nnz = int(indices.size)
    tile = omega * sigma
    T = -(-nnz // tile)
    counts = np.diff(ptr)
    flags = np.zeros(nnz, dtype=bool)
    flags[ptr[:-1][counts > 0]] = True
    flags[np.arange(0, nnz, tile)] = True
    tile_ptr = np.empty(T + 1, dtype=np.int64)
    tile_ptr[:T] = np.searchsorted(ptr, np.arange(T, dtype=np.int64) * tile, side="right") - 1
    tile_ptr[T] = n_rows
    # per (tile, column) flag counts -> y_off (exclusive), top flags -> seg_off
    k = np.arange(nnz, dtype=np.int64)
    cell = (k // tile) * omega + (k % tile) // sigma
    per_col = np.bincount(cell[flags], minlength=T * omega).reshape(T, omega)
    y_off = np.zeros((T, omega), dtype=np.int64)
    if omega > 1:
        y_off[:, 1:] = np.cumsum(per_col, axis=1)[:, :-1]
    tops = np.arange(T * omega, dtype=np.int64).reshape(T, omega)
    top_pos = (tops // omega) * tile + (tops % omega) * sigma
    exists = top_pos < nnz
    open_top = exists & ~flags[np.minimum(top_pos, max(nnz - 1, 0))] if nnz else exists
    seg_off = np.zeros((T, omega), dtype=np.int64)
    run = np.zeros(T, dtype=np.int64)
    for j in range(omega - 1, -1, -1):
        seg_off[:, j] = run
        run = np.where(open_top[:, j], run + 1, 0)
    pos = csr5_stored_positions(nnz, omega, sigma)
    bit_flag = np.empty(nnz, dtype=bool)
    bit_flag[pos] = flags
    ind = np.empty(nnz, dtype=np.int64)
    ind[pos] = indices
    val = np.empty(nnz, dtype=np.float64)
    val[pos] = data
    return Csr5(ptr, omega, sigma, T, tile_ptr, bit_flag, y_off, seg_off, ind, val)


def _grids(n_rows, k, counts, ptr, cols, vals, max_cells):
    """formats.py:253-278 — left-justified grids, pad = last valid col / 0."""
    if n_rows * k > max_cells:
        raise GridTooLarge(f"padded grid of {n_rows}x{k} = {n_rows * k} cells exceeds the {max_cells}-cell limit")
    last = np.zeros(n_rows, dtype=np.int64)
    has = counts > 0
    last[has] = cols[ptr[1:][has] - 1]
    gi = np.repeat(last[:, None], k, axis=1)
    gd = np.zeros((n_rows, k), dtype=np.float64)
    if cols.size:
        rr = np.repeat(np.arange(n_rows), counts)
        ss = np.arange(cols.size) - np.repeat(ptr[:-1], counts)
        gi[rr, ss] = cols
        gd[rr, ss] = vals
    return gi, gd


def to_ell(ptr, indices, data, n_rows, max_cells=DEFAULT_MAX_GRID_CELLS):
    """formats.py:281-288 -> (k, indices (n,k), data (n,k), row_nnz)."""
    counts = np.diff(ptr)
    k = int(counts.max()) if n_rows else 0
    gi, gd = _grids(n_rows, k, counts, ptr, indices, data, max_cells)
    return k, gi, gd, counts


@dataclass
class Sell:
    c: int
    sigma: int
    perm: np.ndarray
    widths: np.ndarray
    data: list
    indices: list
    row_nnz_perm: np.ndarray
    slice_off: np.ndarray
    flat_indices: np.ndarray
    flat_data: np.ndarray


def to_sell(ptr, indices, data, n_rows, c, sigma=0, max_cells=DEFAULT_MAX_GRID_CELLS):
    """formats.py:291-344 (slices as Fortran-order (rows, width) arrays)."""
    if c < 1:
        raise ValueError(f"slice height c must be >= 1, got {c}")
    if sigma < 0 or (sigma > 0 and sigma % c != 0):
        raise ValueError(f"sorting window sigma must be 0 or a positive multiple of c, got sigma={sigma}, c={c}")
    counts = np.diff(ptr)
    if sigma > 0:
        window = np.arange(n_rows) // sigma
        perm = np.lexsort((-counts, window)).astype(np.int64)  # stable: ties keep row order
    else:
        perm = np.arange(n_rows, dtype=np.int64)
    cp = counts[perm]
    S = -(-n_rows // c)
    widths = np.zeros(S, dtype=np.int64)
    if n_rows:
        pad = np.zeros(S * c, dtype=np.int64)
        pad[:n_rows] = cp
        widths = pad.reshape(S, c).max(axis=1)
    rows_in = np.minimum(c, n_rows - np.arange(S) * c)
    total = int((rows_in * widths).sum())
    if total > max_cells:
        raise GridTooLarge(f"sliced grids of {total} cells exceed the {max_cells}-cell limit")
    # One flat buffer = concatenation of the slices' Fortran-order ravels:
    # cell (slice s, column j, local row l) at off[s] + j*rows_s + l.
    off = np.zeros(S + 1, dtype=np.int64)
    np.cumsum(rows_in * widths, out=off[1:])
    cell_slice = np.repeat(np.arange(S), rows_in * widths)
    cell = np.arange(total, dtype=np.int64)
    cell_row = cell_slice * c + (cell - off[cell_slice]) % np.maximum(rows_in[cell_slice], 1)
    last = np.zeros(n_rows, dtype=np.int64)  # pad index: last valid column, 0 if empty
    has = cp > 0
    last[has] = indices[ptr[perm[has] + 1] - 1]
    flat_i = last[cell_row] if total else np.empty(0, np.int64)
    flat_d = np.zeros(total, dtype=np.float64)
    pptr = np.concatenate([[0], np.cumsum(cp)]).astype(np.int64)
    slot = np.arange(int(pptr[-1])) - np.repeat(pptr[:-1], cp)
    prow = np.repeat(np.arange(n_rows), cp)
    src = ptr[perm][prow] + slot
    s_of = prow // c
    dst = off[s_of] + slot * rows_in[s_of] + (prow - s_of * c)
    flat_i[dst] = indices[src]
    flat_d[dst] = data[src]
    ds = [flat_d[off[s]:off[s + 1]].reshape((int(rows_in[s]), int(widths[s])), order="F") for s in range(S)]
    ids = [flat_i[off[s]:off[s + 1]].reshape((int(rows_in[s]), int(widths[s])), order="F") for s in range(S)]
    return Sell(c, sigma, perm, widths, ds, ids, cp, off, flat_i, flat_d)


def hyb_typical_k(counts):
    """formats.py:347-358 — the (n//3 + 1)-th largest count, floored at 1."""
    counts = np.asarray(counts)
    n = counts.size
    if n == 0:
        raise ValueError("typical width is undefined for a matrix with no rows")
    kth = np.sort(counts)[n - 1 - n // 3]
    return max(int(kth), 1)


def to_hyb(row, col, data, n_rows, max_cells=DEFAULT_MAX_GRID_CELLS):
    """formats.py:361-397 -> (K, ell_idx, ell_data, ell_row_nnz, tail (r, c, v))."""
    counts = row_counts(row, n_rows)
    if col.size == 0:
        z = np.empty((n_rows, 0))
        e = np.empty(0, dtype=np.int64)
        return 0, z.astype(np.int64), z, counts, (e, e.copy(), np.empty(0))
    K = hyb_typical_k(counts)
    ptr, ind, val = to_csr(row, col, data, n_rows)
    slot = np.arange(col.size) - np.repeat(ptr[:-1], counts)
    keep = slot < K
    ec = np.minimum(counts, K)
    eptr = np.concatenate([[0], np.cumsum(ec)])
    gi, gd = _grids(n_rows, K, ec, eptr, ind[keep], val[keep], max_cells)
    return K, gi, gd, ec, (np.asarray(row)[~keep], np.asarray(col)[~keep], np.asarray(data)[~keep])


# ----------------------------------------------------------------- kernels --
_POOLS: dict[int, concurrent.futures.ThreadPoolExecutor] = {}


def _map(fn, items, workers):
    if workers <= 1 or len(items) <= 1:
        return [fn(*it) for it in items]
    pool = _POOLS.get(workers)
    if pool is None:
        pool = _POOLS[workers] = concurrent.futures.ThreadPoolExecutor(max_workers=workers)
    return list(pool.map(lambda it: fn(*it), items))


def row_blocks(n_rows, workers):
    """kernels.py:61-66."""
    if n_rows == 0:
        return []
    b = max(1, n_rows // (4 * max(workers, 1)))
    return [(lo, min(lo + b, n_rows)) for lo in range(0, n_rows, b)]


def spmv_csr(ptr, indices, data, n_rows, x, workers=1):
    """kernels.py:76-95: per block, products then reduceat over row starts."""
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(n_rows, dtype=np.float64)

    def block(lo, hi):
        a, b = ptr[lo], ptr[hi]
        prod = data[a:b] * x[indices[a:b]]
        cnt = np.diff(ptr[lo:hi + 1])
        live = np.nonzero(cnt)[0]
        if live.size:
            y[lo + live] = np.add.reduceat(prod, ptr[lo:hi][live] - a)

    _map(block, row_blocks(n_rows, workers), workers)
    return y


def spmv_ell(k, gi, gd, x, workers=1):
    """kernels.py:98-116: slot-by-slot accumulation (pads included)."""
    x = np.asarray(x, dtype=np.float64)
    n = gi.shape[0]
    y = np.zeros(n, dtype=np.float64)

    def block(lo, hi):
        acc = np.zeros(hi - lo)
        for j in range(k):
            acc += gd[lo:hi, j] * x[gi[lo:hi, j]]
        y[lo:hi] = acc

    _map(block, row_blocks(n, workers), workers)
    return y


def spmv_sell(m: Sell, n_rows, x, workers=1):
    """kernels.py:119-136."""
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(n_rows, dtype=np.float64)
    if n_rows == 0:
        return y
    # Column j of every slice at once: each row still accumulates its slots
    # in order 0..w-1 (pads included), the reference's per-slice recurrence.
    S = len(m.data)
    rows_in = np.minimum(m.c, n_rows - np.arange(S) * m.c)
    p = np.arange(n_rows)
    s_of = p // m.c
    w_of = m.widths[s_of]
    base = m.slice_off[s_of] + (p - s_of * m.c)
    stride = rows_in[s_of]
    acc = np.zeros(n_rows)
    live = np.nonzero(w_of > 0)[0]
    j = 0
    while live.size:
        o = base[live] + j * stride[live]
        acc[live] += m.flat_data[o] * x[m.flat_indices[o]]
        j += 1
        live = live[w_of[live] > j]
    y[m.perm] = acc
    return y


def csr5_tile_partials(m: Csr5, x, t):
    """kernels.py:139-164: undo stored order, reduceat over flags, rows via ptr."""
    tile = m.omega * m.sigma
    base = t * tile
    cnt = min(tile, m.indices.size - base)
    sl = slice(base, base + cnt)
    p = np.arange(cnt, dtype=np.int64)
    q, rem = cnt // m.sigma, cnt % m.sigma
    gi, gj = p % m.sigma, p // m.sigma
    stored = gi * q + np.minimum(gi, rem) + gj  # CSR-order p -> stored slot
    prod = (m.data[sl] * x[m.indices[sl]])[stored]
    fl = m.bit_flag[sl][stored]
    starts = np.nonzero(fl)[0]
    sums = np.add.reduceat(prod, starts)
    rows = np.searchsorted(m.ptr, base + starts, side="right") - 1
    return rows, sums


def spmv_csr5(m: Csr5, n_rows, x, workers=1):
    """kernels.py:167-174: partials folded in ascending tile order."""
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(n_rows, dtype=np.float64)
    parts = _map(lambda t: csr5_tile_partials(m, x, t), [(t,) for t in range(m.num_tiles)], workers)
    for rows, sums in parts:
        y[rows] += sums
    return y


def spmv_hyb(K, gi, gd, tail, n_rows, x, workers=1):
    """kernels.py:177-199: ELL part, then bincount tail ranges in order."""
    x = np.asarray(x, dtype=np.float64)
    y = spmv_ell(K, gi, gd, x, workers)
    tr, tc, tv = tail
    n = tr.size
    if n:
        chunk = -(-n // max(workers, 1))
        ranges = [(lo, min(lo + chunk, n)) for lo in range(0, n, chunk)]
        parts = _map(lambda lo, hi: np.bincount(tr[lo:hi], weights=tv[lo:hi] * x[tc[lo:hi]], minlength=n_rows),
                     ranges, workers)
        for part in parts:
            y += part
    return y


# ---------------------------------------------------------------- features --
def extract_features(row, n_rows, n_cols):
    """features.py:69-84 (8 values, fixed order)."""
    if n_rows == 0 or n_cols == 0:
        raise ValueError(f"features are undefined for a {n_rows}x{n_cols} matrix")
    counts = row_counts(row, n_rows)
    avg = float(counts.mean())
    std = float(counts.std())
    nnz = int(counts.sum())
    return (n_rows, n_cols, nnz / (n_rows * n_cols), int(counts.min()), int(counts.max()), avg, std,
            std / avg if avg > 0 else 0.0)


def extra_features(row, col, n_rows, n_cols):
    """North-star extras (no reference counterpart): bandwidth, diagonal density."""
    row = np.asarray(row, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    bw = int(np.abs(row - col).max()) if row.size else 0
    mn = min(n_rows, n_cols)
    diag = int(np.count_nonzero(row == col))
    return {"bandwidth": bw, "diag_density": diag / mn if mn else 0.0}


# -------------------------------------------------------------- byte model --
def spmv_bytes(tag, n_rows, n_cols, **kw):
    """bench.py:139-170 byte model (8 B values, 4 B indices, 1 B flags)."""
    vec = 8 * n_cols + 8 * n_rows
    if tag == "csr":
        return 12 * kw["nnz"] + 4 * (n_rows + 1) + vec
    if tag == "csr5":
        T = kw["num_tiles"]
        return 12 * kw["nnz"] + 4 * (n_rows + 1) + 4 * (T + 1) + kw["nnz"] + 8 * kw["omega"] * T + vec
    if tag == "ell":
        return 12 * n_rows * kw["k"] + vec
    if tag == "sell":
        return 12 * kw["cells"] + 4 * kw["n_slices"] + (4 * n_rows if kw["sigma"] > 0 else 0) + vec
    if tag == "hyb":
        return 12 * n_rows * kw["k"] + 16 * kw["tail_nnz"] + vec
    raise ValueError(tag)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
