"""Degree-ordered shadow layout for iterative SpMV on square matrices.

Not part of the reference's API: an internal layout behind the power
iteration (BASELINE configs C3-C5 iterate x <- A x / ||A x||).  The
reference's arrays (``to_csr5`` etc.) are never changed; this module builds
a second, relabelled copy ``P A P^T`` and runs the iteration on
``x' = P x``, so ``P^T x'_k`` is the same iterate as the plain iteration's
``x_k`` (within the SpMV tolerance: only the order of the row sums differs).

The relabelling (csrc/relabel.cu) sorts ids by (row is empty, -row degree,
-column degree) (or by row + column degree), stable by id.  On R-MAT it packs
the hot columns of x into
the first cache lines (more L1/L2 hits per gathered 128-byte line; the C5
SpMV is bound by the rate of distinct lines its random x gathers touch) and
puts every empty row last, so the CSR5 kernel needs no row indirection and
zeroes the empty tail with plain stores.  Measured (scripts/relabel_probe.py,
profiles/r02_relabel_probe_c{4,5}.txt): C5 CSR5 SpMV 2.84 -> 2.45 ms, C4 107.5 ->
97.3 us.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import LIB, check, ptr
from .coo import canonicalize
from .formats import CsrMatrix, FormatTag, convert, to_csr
from .kernels import SpmvOperator, bind, spmv

__all__ = ["DegreeOrder", "RelabelledMatrix", "power_iteration"]


def _as_csr(a) -> CsrMatrix:
    return a if isinstance(a, CsrMatrix) else to_csr(a)


_KEYS = {"sum": 0, "row": 1}


class DegreeOrder:
    """The symmetric permutation of a square matrix: ``perm[new] = old``,
    ``new_id[old] = new`` (int32 device tensors); rows ``[0, n_nonempty)``
    of ``P A P^T`` are the non-empty ones.  ``key``: ``"row"`` (default)
    orders by row degree, then column degree, so the rows come in exact
    descending length (SELL slices then pad least: degree-ordered C5 SELL-32
    2.22 -> 2.20 ms, sigma 0 2.41 -> 2.27 ms); ``"sum"`` by row + column
    degree (CSR5 is the same either way; profiles/r02_relabel_formats2.txt)."""

    def __init__(self, a, key: str = "row", parts: int = 1):
        if key not in _KEYS:
            raise ValueError(f"key must be one of {sorted(_KEYS)}, got {key!r}")
        if parts < 1:
            raise ValueError(f"parts must be >= 1, got {parts}")
        self.key = key
        self.parts = int(parts)
        csr = _as_csr(a)
        if csr.n_rows != csr.n_cols:
            raise ValueError(f"relabelling needs a square matrix, got {csr.n_rows}x{csr.n_cols}")
        dev = csr.device
        n = csr.n_rows
        self.n = n
        self.perm = torch.empty(n, dtype=torch.int32, device=dev)
        self.new_id = torch.empty(n, dtype=torch.int32, device=dev)
        cnt = ctypes.c_int64()
        with torch.cuda.device(dev):
            check(LIB.spmvb_degree_order(n, ptr(csr.ptr), ptr(csr.indices), csr.nnz, _KEYS[key], ptr(self.perm),
                                         ptr(self.new_id), ctypes.byref(cnt), _lib.stream(dev)))
        self.n_nonempty = int(cnt.value)
        self.part_bounds = [0, n]
        if self.parts > 1:
            self._deal(self.parts)

    def _deal(self, P: int) -> None:
        """Multi-GPU form (``parts`` = P): the degree-sorted ids are dealt
        round-robin to P contiguous blocks -- sorted position i goes to block
        i mod P, in sorted order within the block -- so every block (one
        rank's row block, ``part_bounds``) holds the same mix of hub and
        light rows, nnz-balanced to within one row's length, with its own
        hot columns first and its empty rows last.  A plain degree order cut
        into nnz-balanced blocks would hand rank 0 all the hub rows, whose x
        gathers miss L2 the most (the C5 SELL wide slices run at ~90 G
        gathers/s against ~340 for the rest)."""
        n, dev = self.n, self.device
        i = torch.arange(n, dtype=torch.int64, device=dev)
        counts = [(n - r + P - 1) // P for r in range(P)]
        offs = [0]
        for c_ in counts:
            offs.append(offs[-1] + c_)
        pos = torch.tensor(offs[:-1], dtype=torch.int64, device=dev)[i % P] + i // P
        perm = torch.empty_like(self.perm)
        perm[pos] = self.perm
        self.perm = perm
        self.new_id[perm.long()] = torch.arange(n, dtype=torch.int32, device=dev)
        self.part_bounds = offs
        self.n_nonempty = None  # the non-empty rows are a prefix of each block, not of the whole

    @property
    def device(self) -> torch.device:
        return self.perm.device

    def matrix(self, a) -> CsrMatrix:
        """``P A P^T`` as CSR (relabelled triplets, then the GPU canonicalize)."""
        csr = _as_csr(a)
        if csr.n_rows != self.n or csr.n_cols != self.n:
            raise ValueError("matrix shape does not match the relabelling")
        dev = csr.device
        nnz = csr.nnz
        row = torch.empty(nnz, dtype=torch.int32, device=dev)
        col = torch.empty(nnz, dtype=torch.int32, device=dev)
        val = torch.empty(nnz, dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            check(LIB.spmvb_relabel_csr(self.n, ptr(csr.ptr), ptr(csr.indices), ptr(csr.data), nnz,
                                        ptr(self.new_id), ptr(row), ptr(col), ptr(val), _lib.stream(dev)))
        coo = canonicalize(row, col, val, self.n, self.n, device=dev)
        del row, col, val
        return to_csr(coo)

    def _gather(self, src: torch.Tensor, idx: torch.Tensor, out: torch.Tensor | None) -> torch.Tensor:
        src = src.reshape(-1)
        if not src.is_cuda or src.dtype != torch.float64 or src.numel() != self.n:
            raise ValueError(f"expected a float64 CUDA vector of length {self.n}")
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, device=src.device)
        with torch.cuda.device(src.device):
            check(LIB.spmvb_gather_f64(ptr(src.contiguous()), 0, ptr(idx), self.n, ptr(out),
                                       _lib.stream(src.device)))
        return out

    def to_new(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """``x' = P x`` (x'[new] = x[perm[new]])."""
        return self._gather(x, self.perm, out)

    def to_old(self, xp: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """``x = P^T x'`` (x[old] = x'[new_id[old]])."""
        return self._gather(xp, self.new_id, out)


class RelabelledMatrix:
    """A format matrix of ``P A P^T`` (``convert(tag, ...)`` of the
    relabelled CSR) with its ``DegreeOrder``; ``spmv`` works in the new ids."""

    def __init__(self, tag, a, **convert_kw):
        csr = _as_csr(a)
        self.tag = FormatTag(tag)
        self.order = DegreeOrder(csr)
        shadow = self.order.matrix(csr)
        self.inner = convert(self.tag, shadow, **convert_kw)
        if self.tag in (FormatTag.CSR, FormatTag.HYB):
            self.inner.chunk_plan()
        self.n_rows = self.n_cols = csr.n_rows
        self.nnz = csr.nnz

    def spmv(self, xp: torch.Tensor, out: torch.Tensor | None = None, scale=None) -> torch.Tensor:
        """``y' = scale * (P A P^T) x'`` on device vectors in the new ids."""
        return spmv(self.tag, self.inner, xp, out=out, scale=scale)

    def bind(self, xp: torch.Tensor, out: torch.Tensor, scale=None):
        """A prepared ``spmv(xp, out, scale)`` (kernels.bind) in the new ids."""
        return bind(self.tag, self.inner, xp, out, scale)

    __call__ = spmv

    def spmv_original(self, x: torch.Tensor) -> torch.Tensor:
        """``A x`` in the original ids (two permutation gathers around the SpMV)."""
        return self.order.to_old(self.spmv(self.order.to_new(x)))


# the candidates tag="auto" times (the bench's shadow-layout candidates)
AUTO_CANDIDATES = {
    FormatTag.CSR: {},
    FormatTag.CSR5: dict(omega=32, sigma=8),
    FormatTag.SELL: dict(sell_c=32, sell_sigma=0, max_cells=1 << 34),
    FormatTag.HYB: dict(max_cells=1 << 34),
}


def power_iteration(a, x0, steps: int, tag="auto", *, relabel: bool = True, graph: bool = False, **convert_kw):
    """``steps`` iterations of x <- A x / ||A x|| on one GPU; returns the
    unit-norm iterate and ``||A x_{k-1}||`` (the eigenvalue estimate), x in
    the original ids.  ``relabel`` runs them on the
    degree-ordered shadow layout (one permutation of x0 before, one of the
    result after); ``graph`` replays the steps from a CUDA graph
    (dist.PowerIteration.run).  ``tag="auto"`` converts the matrix the steps
    run on to each of AUTO_CANDIDATES, times one SpMV of each and keeps the
    fastest (model.select_format_measured): SELL-32 on a degree-ordered
    R-MAT, ELL/SELL on stencils."""
    from .dist import PowerIteration
    from .model import select_format_measured

    csr = _as_csr(a)
    dev = csr.device
    x0 = torch.as_tensor(x0, dtype=torch.float64).to(dev).reshape(-1)
    if relabel:
        order = DegreeOrder(csr)
        shadow = order.matrix(csr)
        if tag == "auto":
            tag, m, _ = select_format_measured(shadow, list(AUTO_CANDIDATES), params=AUTO_CANDIDATES)
        else:
            m = convert(tag, shadow, **convert_kw)
        del shadow
        pi = PowerIteration(SpmvOperator(tag, m), [0, csr.n_rows], 0, 1, dev, order.to_new(x0))
        pi.run(steps, graph=graph)
        return order.to_old(pi.normalized()), pi.eigenvalue_estimate()
    if tag == "auto":
        cands = dict(AUTO_CANDIDATES, **{FormatTag.ELL: {}})
        tag, m, _ = select_format_measured(csr, list(cands), params=cands)
    else:
        m = convert(tag, csr, **convert_kw)
    pi = PowerIteration(SpmvOperator(tag, m), [0, csr.n_rows], 0, 1, dev, x0)
    pi.run(steps, graph=graph)
    return pi.normalized(), pi.eigenvalue_estimate()
