"""Seeded synthetic matrices for the five benchmark configurations
(BASELINE.json ``configs``).  The paper's SuiteSparse corpus
is not available offline, so these generators stand in for it with the
configs' shapes, sizes and value distributions.

C1-C3 are built on the host with numpy (input setup, not the hot path) and
canonicalized on the GPU.  R-MAT (C4, C5) is generated on the GPU by a
counter-based hash (csrc/gen.cu); ``oracle/synth_ref.py`` regenerates the
same edge list on the host bit for bit for parity checks.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import LIB, check, ptr
from .coo import CooMatrix, canonicalize

__all__ = [
    "CONFIGS",
    "banded",
    "laplace2d",
    "rmat_coo",
    "rmat_triplets",
    "stencil27",
    "uniform_vector",
]

RMAT_ABC = (0.57, 0.19, 0.19)

CONFIGS = {
    "C1": dict(kind="laplace2d", g=512, seed=101),
    "C2": dict(kind="banded", n=1 << 20, per_row=8, half=64, seed=102),
    "C3": dict(kind="stencil27", g=88, seed=103),
    "C4": dict(kind="rmat", scale=21, edge_factor=10, seed=104),
    "C5": dict(kind="rmat", scale=25, edge_factor=16, seed=105),
}


def laplace2d(g: int = 512, seed: int = 101):
    """2-D 5-point Laplacian on a g x g grid: 4 on the diagonal, -1 to the
    in-grid neighbours (config 1).  Returns host (row, col, val, n)."""
    n = g * g
    i = np.arange(n, dtype=np.int64)
    r, c = i // g, i % g
    rows = [i]
    cols = [i]
    vals = [np.full(n, 4.0)]
    for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (r + dr >= 0) & (r + dr < g) & (c + dc >= 0) & (c + dc < g)
        rows.append(i[ok])
        cols.append(i[ok] + dr * g + dc)
        vals.append(np.full(int(ok.sum()), -1.0))
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), n


def banded(n: int = 1 << 20, per_row: int = 8, half: int = 64, seed: int = 102):
    """Each row gets `per_row` distinct columns drawn without replacement from
    [i-half, i+half] clipped to the matrix; values N(0, 1) (config 2)."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    w = 2 * half + 1
    chunk = 1 << 15
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        i = np.arange(lo, hi, dtype=np.int64)
        start = np.clip(i - half, 0, None)
        stop = np.minimum(i + half, n - 1)
        width = stop - start + 1
        keys = rng.random((hi - lo, w))
        keys[np.arange(w)[None, :] >= width[:, None]] = 2.0  # outside the clipped window
        pick = np.argpartition(keys, per_row - 1, axis=1)[:, :per_row]
        rows.append(np.repeat(i, per_row))
        cols.append((start[:, None] + pick).ravel())
    row = np.concatenate(rows)
    col = np.concatenate(cols)
    val = rng.standard_normal(row.size)
    return row, col, val, n


def stencil27(g: int = 88, seed: int = 103):
    """3-D 27-point stencil on a g^3 grid; off-diagonal U[-1, 1], diagonal
    1 + sum |off-diagonal| (strictly diagonally dominant) (config 3)."""
    rng = np.random.default_rng(seed)
    n = g ** 3
    i = np.arange(n, dtype=np.int64)
    z, y, x = i // (g * g), (i // g) % g, i % g
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dz == dy == dx == 0:
                    continue
                ok = (z + dz >= 0) & (z + dz < g) & (y + dy >= 0) & (y + dy < g) & (x + dx >= 0) & (x + dx < g)
                rows.append(i[ok])
                cols.append(i[ok] + dz * g * g + dy * g + dx)
    row = np.concatenate(rows)
    col = np.concatenate(cols)
    val = rng.uniform(-1.0, 1.0, size=row.size)
    diag = 1.0 + np.bincount(row, weights=np.abs(val), minlength=n)
    return np.concatenate([row, i]), np.concatenate([col, i]), np.concatenate([val, diag]), n


def host_coo(name: str, device=None) -> CooMatrix:
    """C1-C3 as canonical GPU COO (host-generated triplets)."""
    cfg = dict(CONFIGS[name])
    kind = cfg.pop("kind")
    row, col, val, n = {"laplace2d": laplace2d, "banded": banded, "stencil27": stencil27}[kind](**cfg)
    return canonicalize(row, col, val, n, n, device=device)


def rmat_triplets(scale: int, edge_factor: int, seed: int, device=None, abc=RMAT_ABC):
    """R-MAT edge list on the GPU: (row, col, val) int32/int32/float64
    tensors, duplicates removed keeping the first draw, unsorted (draw
    order).  n = 2^scale, draws = edge_factor * n."""
    dev = torch.device(device) if device is not None else _lib.require_cuda()
    draws = edge_factor << scale
    plan = ctypes.c_void_p()
    nnz = ctypes.c_int64()
    with torch.cuda.device(dev):
        s = _lib.stream(dev)
        check(LIB.spmvb_rmat_begin(scale, draws, abc[0], abc[1], abc[2], seed, ctypes.byref(plan),
                                   ctypes.byref(nnz), s))
        m = int(nnz.value)
        r = torch.empty(m, dtype=torch.int32, device=dev)
        c = torch.empty(m, dtype=torch.int32, device=dev)
        v = torch.empty(m, dtype=torch.float64, device=dev)
        check(LIB.spmvb_rmat_finish(plan, ptr(r), ptr(c), ptr(v), s))
    return r, c, v


def rmat_coo(scale: int, edge_factor: int, seed: int, device=None) -> CooMatrix:
    r, c, v = rmat_triplets(scale, edge_factor, seed, device)
    n = 1 << scale
    return canonicalize(r, c, v, n, n, device=r.device)


def uniform_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0, device=None) -> torch.Tensor:
    """x ~ U[lo, hi) from the counter hash (same values as oracle.synth_ref.uniform)."""
    dev = torch.device(device) if device is not None else _lib.require_cuda()
    x = torch.empty(n, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(LIB.spmvb_fill_uniform(ptr(x), n, lo, hi, seed, _lib.stream(dev)))
    return x
