"""Sparse storage formats on the GPU: CSR, CSR5, ELL, SELL(-C-sigma), HYB.

Mirrors spmvkit.formats (/root/reference/pkg/src/spmvkit/formats.py): same
class names, fields, converters, parameters, defaults and error behaviour.
Arrays are CUDA tensors (int32 indices, float64 values).  Where the
reference stores a C-order grid, the GPU stores the layout its kernel reads
coalesced and the attribute returns the reference's *logical* view:

* ``EllMatrix.indices/.data`` are (n_rows, k) views of column-major grids.
* ``SellMatrix.indices/.data`` are sequences of per-slice (rows, width)
  views of one flat buffer holding each slice column-major, exactly the
  reference's Fortran-order slices (formats.py:326-341).
* ``Csr5Matrix.y_off/.seg_off`` are (num_tiles, omega) int32 tensors;
  ``bit_flag`` is a bool tensor in stored order.

Every conversion runs on the device (csrc/formats.cu, csrc/coo.cu).
Kernel-side auxiliary data (CSR chunk first-row tables, CSR5 tile words,
the non-empty row list) is derived at conversion time or lazily on first
use, like a cuSPARSE analysis buffer; it is not part of the reference
arrays and does not change them.
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np
import torch

from . import _lib
from ._lib import LIB, ConversionError, check, ptr
from .coo import CooMatrix, _empty, canonicalize

__all__ = [
    "DEFAULT_MAX_GRID_CELLS",
    "ConversionError",
    "Csr5Matrix",
    "CsrMatrix",
    "EllMatrix",
    "FormatMatrix",
    "FormatTag",
    "HybMatrix",
    "SellMatrix",
    "convert",
    "hyb_typical_k",
    "to_coo",
    "to_csr",
    "to_csr5",
    "to_ell",
    "to_hyb",
    "to_sell",
]

DEFAULT_MAX_GRID_CELLS = 1 << 26  # formats.py:58


class FormatTag(str, Enum):
    """The benchmarked storage formats, in tie-breaking declaration order."""

    CSR = "csr"
    CSR5 = "csr5"
    ELL = "ell"
    SELL = "sell"
    HYB = "hyb"


SELL_HUB_PIECES = 32  # include/spmvb.h SPMVB_SELL_HUB_PIECES


def _i32(n, dev):
    return torch.empty(int(n), dtype=torch.int32, device=dev)


def _i64(n, dev):
    return torch.empty(int(n), dtype=torch.int64, device=dev)


def _f64(n, dev):
    return torch.empty(int(n), dtype=torch.float64, device=dev)


def _row_stats(ptr_t: torch.Tensor, n_rows: int) -> tuple[int, int, int]:
    out = (ctypes.c_int64 * 3)()
    with torch.cuda.device(ptr_t.device):
        check(LIB.spmvb_csr_row_stats(ptr(ptr_t), n_rows, out, _lib.stream(ptr_t.device)))
    return int(out[0]), int(out[1]), int(out[2])


class _ChunkPlan:
    """Per-chunk first-row table for the chunked CSR kernel, built once."""

    def __init__(self, ptr_t: torch.Tensor, n_rows: int, nnz: int):
        dev = ptr_t.device
        self.chunk = int(LIB.spmvb_csr_chunk_size())
        self.chunks = int(LIB.spmvb_csr_chunks(nnz))
        self.chunk_row = _i32(self.chunks + 1, dev)
        self.nz_rows = None
        self.n_nz = n_rows
        if n_rows:
            with torch.cuda.device(dev):
                s = _lib.stream(dev)
                self.n_nz = _row_stats(ptr_t, n_rows)[2]
                if self.n_nz < n_rows:
                    self.nz_rows = _i32(self.n_nz, dev)
                    if self.n_nz:
                        check(LIB.spmvb_csr_nonempty_rows(ptr(ptr_t), n_rows, ptr(self.nz_rows), s))
                check(LIB.spmvb_csr_chunk_plan(n_rows, nnz, ptr(ptr_t), ptr(self.nz_rows), self.n_nz,
                                               ptr(self.chunk_row), s))

    def scratch(self, dev):
        return _i32(max(self.chunks, 1), dev), _f64(max(self.chunks, 1), dev)

    @property
    def nbytes(self) -> int:
        return 4 * (self.chunks + 1) + (4 * self.n_nz if self.nz_rows is not None else 0)


class CsrMatrix:
    """Row-pointer compressed rows (formats.py:75-85)."""

    def __init__(self, n_rows: int, n_cols: int, ptr: torch.Tensor, indices: torch.Tensor, data: torch.Tensor):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.ptr = ptr
        self.indices = indices
        self.data = data
        self._chunks: _ChunkPlan | None = None

    def chunk_plan(self) -> _ChunkPlan:
        if self._chunks is None:
            self._chunks = _ChunkPlan(self.ptr, self.n_rows, self.nnz)
        return self._chunks

    @property
    def nnz(self) -> int:
        return int(self.data.shape[0])

    @property
    def device(self) -> torch.device:
        return self.ptr.device

    def __repr__(self) -> str:
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


class Csr5Matrix:
    """CSR plus the tiled arrays and descriptor (formats.py:88-107)."""

    def __init__(self, n_rows, n_cols, ptr, omega, sigma, num_tiles, tile_ptr, bit_flag, y_off, seg_off, indices,
                 data, tile_aux, nonempty_rows, n_nonempty):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.ptr = ptr
        self.omega = int(omega)
        self.sigma = int(sigma)
        self.num_tiles = int(num_tiles)
        self.tile_ptr = tile_ptr
        self.bit_flag = bit_flag
        self.y_off = y_off
        self.seg_off = seg_off
        self.indices = indices
        self.data = data
        # kernel-side auxiliary data (not reference arrays)
        self.tile_aux = tile_aux
        self.nonempty_rows = nonempty_rows
        self.n_nonempty = int(n_nonempty)
        self.flag_bits = None  # bit_flag packed one bit per entry (set by to_csr5)
        self._ranges = {}

    @property
    def nnz(self) -> int:
        return int(self.data.shape[0])

    @property
    def device(self) -> torch.device:
        return self.ptr.device

    def range_plan(self, n_ranges: int) -> tuple[np.ndarray, np.ndarray]:
        """(tile_bounds, row_bounds) of ``n_ranges`` tile ranges that each start
        at a row-start tile (spmvb_csr5_range_bounds); cached per count.  The
        host-buffer SpMV streams each range's finished rows back while the
        next range computes."""
        n_ranges = max(1, int(n_ranges))
        if n_ranges not in self._ranges:
            tb = np.zeros(n_ranges + 1, dtype=np.int64)
            rb = np.zeros(n_ranges + 1, dtype=np.int64)
            with torch.cuda.device(self.device):
                check(LIB.spmvb_csr5_range_bounds(self.nnz, self.omega, self.sigma, ptr(self.tile_ptr),
                                                  ptr(self.tile_aux), n_ranges, tb.ctypes.data, rb.ctypes.data,
                                                  _lib.stream(self.device)))
            self._ranges[n_ranges] = (tb, rb)
        return self._ranges[n_ranges]

    def __repr__(self) -> str:
        return f"Csr5Matrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, omega={self.omega}, sigma={self.sigma})"


class EllMatrix:
    """Fixed-width padded rows; ``k`` is the widest row (formats.py:110-123).

    ``grid_indices``/``grid_data`` are the (k, n_rows) column-major device
    grids the kernel streams; ``indices``/``data`` are their (n_rows, k)
    logical views.
    """

    def __init__(self, n_rows, n_cols, k, grid_indices, grid_data, row_nnz):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.k = int(k)
        self.grid_indices = grid_indices
        self.grid_data = grid_data
        self.row_nnz = row_nnz

    @property
    def indices(self) -> torch.Tensor:
        return self.grid_indices.t()

    @property
    def data(self) -> torch.Tensor:
        return self.grid_data.t()

    @property
    def nnz(self) -> int:
        return int(self.row_nnz.sum().item()) if self.n_rows else 0

    @property
    def device(self) -> torch.device:
        return self.grid_data.device

    def __repr__(self) -> str:
        return f"EllMatrix({self.n_rows}x{self.n_cols}, k={self.k})"


class _SliceViews:
    """Read-only sequence of per-slice (rows, width) views of a flat buffer."""

    def __init__(self, flat: torch.Tensor, owner: "SellMatrix"):
        self._flat = flat
        self._owner = owner

    def __len__(self) -> int:
        return self._owner.n_slices

    def __getitem__(self, s):
        if isinstance(s, slice):
            return [self[i] for i in range(*s.indices(len(self)))]
        n = len(self)
        if s < 0:
            s += n
        if not 0 <= s < n:
            raise IndexError("slice index out of range")
        off, widths = self._owner._host_layout()
        c, n_rows = self._owner.c, self._owner.n_rows
        rows = min(c, n_rows - s * c)
        w = int(widths[s])
        return self._flat[int(off[s]) : int(off[s]) + rows * w].view(w, rows).t()

    def __iter__(self):
        for s in range(len(self)):
            yield self[s]


class SellMatrix:
    """Sliced ELL with optional sigma-window sorting (formats.py:126-153)."""

    def __init__(self, n_rows, n_cols, c, sigma, perm, widths, slice_off, flat_indices, flat_data, row_nnz_perm):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.c = int(c)
        self.sigma = int(sigma)
        self.perm = perm
        self.widths = widths
        self.slice_off = slice_off
        self.flat_indices = flat_indices
        self.flat_data = flat_data
        self.row_nnz_perm = row_nnz_perm
        self._host = None
        self._wide = None
        self._ranges = {}

    def wide_cols(self) -> int:
        """Slices up to this width are summed one thread per row (sequential,
        bit-identical); wider ones by a CTA per ~32K-cell piece.  256 (the
        header's SPMVB_SELL_WIDE_COLS) unless the matrix is big enough for
        4096-slot per-thread rows to hide behind the rest of the grid (at
        least ~1200 cells per resident thread) and its wide slices all come
        first (degree-ordered C5: 2.20 -> 2.09 ms at 4096; C4 stays at 256,
        where 1024 would serialise it: 135 -> 222 us;
        profiles/r02_sell_ab2.txt)."""
        w = 256
        wide = torch.nonzero(self.widths > w)
        # only when the wide slices come first (rows in descending length, a
        # degree-ordered matrix): their long threads then start with the grid
        # instead of trailing it (reference-layout C5 would lose 3.23 -> 3.43 ms)
        if wide.numel() == 0 or int(wide[-1].item()) >= self.n_slices // 4:
            return w
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        per_thread = self.total_cells / max(sms * 2048, 1)
        # measured: the whole degree-ordered C5 (~1750 cells per resident
        # thread) gains from 4096 (2.20 -> 2.09 ms); its dealt 1/2 .. 1/8
        # shards (870 .. 220) do not, and 512 costs 1/8 a quarter
        # (0.31 -> 0.39 ms, profiles/r02_sell_shard_wide_probe.txt)
        return 4096 if per_thread >= 1200 else w

    def wide_plan(self):
        """(wide slice list, count, widest remaining slice, first piece per
        wide slice, piece count, wide_cols): slices wider than wide_cols()
        are cut into ~32K-cell pieces, a CTA each (kernel-side, built once)."""
        if self._wide is None:
            n_slices = self.n_slices
            wide_cols = self.wide_cols()
            lst = _i32(max(n_slices, 1), self.device)
            first = _i32(max(n_slices, 1), self.device)
            cnt, mx, npieces = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            with torch.cuda.device(self.device):
                check(LIB.spmvb_sell_wide_plan(self.n_rows, self.c, ptr(self.widths), wide_cols, ptr(lst),
                                               ctypes.byref(cnt), ctypes.byref(mx), ptr(first),
                                               ctypes.byref(npieces), _lib.stream(self.device)))
            n_wide, n_pieces = int(cnt.value), int(npieces.value)
            hub = _i32(1, self.device)
            n_hub = 0
            if n_wide:  # wide slices of more than SPMVB_SELL_HUB_PIECES (32) pieces: summed a warp per row
                ends = torch.cat([first[1:n_wide].long(),
                                  torch.tensor([n_pieces], dtype=torch.int64, device=self.device)])
                hubs = torch.nonzero(ends - first[:n_wide].long() > SELL_HUB_PIECES).flatten().to(torch.int32)
                n_hub = int(hubs.numel())
                if n_hub:
                    hub = hubs
            self._wide = (lst, n_wide, int(mx.value), first, n_pieces, wide_cols, self._empty_tail(), hub, n_hub)
        return self._wide

    def range_plan(self, k: int):
        """About ``k`` slice ranges of roughly equal cells, aligned to the
        sigma sorting windows (so each range's rows are one contiguous block
        of y): a list of (s_begin, s_end, i_begin, i_end, pc_begin, pc_end,
        row_begin, row_end, h_begin, h_end) for ``kernels.spmv_sell_range``;
        cached."""
        key = int(k)
        if key in self._ranges:
            return self._ranges[key]
        wide, n_wide, _, first, n_pieces = self.wide_plan()[:5]
        hub, n_hub = self.wide_plan()[7:9]
        hl = hub[:n_hub].cpu().numpy() if n_hub else np.empty(0, np.int32)
        S = self.n_slices
        align = max(self.sigma // self.c, 1) if self.sigma > 0 else 1
        off = self.slice_off.cpu().numpy()
        total = int(off[-1]) if S else 0
        cuts = [0]
        for j in range(1, max(key, 1)):
            sj = int(np.searchsorted(off, total * j / key, side="left"))
            sj = min((sj // align) * align, S)
            if sj > cuts[-1]:
                cuts.append(sj)
        if S > cuts[-1]:
            cuts.append(S)
        wl = wide[:n_wide].cpu().numpy() if n_wide else np.empty(0, np.int32)
        fp = first[:n_wide].cpu().numpy() if n_wide else np.empty(0, np.int32)
        plan = []
        for s0, s1 in zip(cuts[:-1], cuts[1:]):
            i0, i1 = int(np.searchsorted(wl, s0)), int(np.searchsorted(wl, s1))
            pc0 = int(fp[i0]) if i0 < n_wide else n_pieces
            pc1 = int(fp[i1]) if i1 < n_wide else n_pieces
            h0, h1 = int(np.searchsorted(hl, i0)), int(np.searchsorted(hl, i1))
            plan.append((s0, s1, i0, i1, pc0, pc1, s0 * self.c, min(s1 * self.c, self.n_rows), h0, h1))
        self._ranges[key] = plan
        return plan

    def _empty_tail(self) -> int:
        """First permuted row of the trailing all-empty slices if perm is the
        identity from there on (a degree-ordered matrix), else n_rows."""
        n = self.n_rows
        if n == 0:
            return 0
        nz = torch.nonzero(self.widths > 0)
        tail = min((int(nz[-1].item()) + 1) * self.c, n) if nz.numel() else 0
        if tail < n and self.sigma > 0:
            ident = torch.arange(tail, n, dtype=self.perm.dtype, device=self.device)
            if not torch.equal(self.perm[tail:], ident):
                return n
        return tail

    def _host_layout(self):
        if self._host is None:
            self._host = (self.slice_off.cpu().numpy(), self.widths.cpu().numpy())
        return self._host

    @property
    def data(self) -> _SliceViews:
        return _SliceViews(self.flat_data, self)

    @property
    def indices(self) -> _SliceViews:
        return _SliceViews(self.flat_indices, self)

    @property
    def n_slices(self) -> int:
        return int(self.widths.shape[0])

    @property
    def total_cells(self) -> int:
        return int(self.flat_data.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.row_nnz_perm.sum().item()) if self.n_rows else 0

    @property
    def device(self) -> torch.device:
        return self.perm.device

    def __repr__(self) -> str:
        return f"SellMatrix({self.n_rows}x{self.n_cols}, c={self.c}, sigma={self.sigma}, cells={self.total_cells})"


class HybMatrix:
    """ELL part of width K plus a canonical COO tail (formats.py:156-177).

    ``tail_ptr`` (kernel-side) is the tail's per-row offset array, so the
    tail is reduced by the chunked CSR kernel without atomics.
    """

    def __init__(self, ell: EllMatrix, coo_tail: CooMatrix, tail_ptr: torch.Tensor):
        self.ell = ell
        self.coo_tail = coo_tail
        self.tail_ptr = tail_ptr
        self._chunks: _ChunkPlan | None = None

    def chunk_plan(self) -> _ChunkPlan:
        if self._chunks is None:
            self._chunks = _ChunkPlan(self.tail_ptr, self.n_rows, self.coo_tail.nnz)
        return self._chunks

    n_rows = property(lambda self: self.ell.n_rows)
    n_cols = property(lambda self: self.ell.n_cols)
    k = property(lambda self: self.ell.k)

    @property
    def nnz(self) -> int:
        return self.ell.nnz + self.coo_tail.nnz

    @property
    def device(self) -> torch.device:
        return self.tail_ptr.device

    def __repr__(self) -> str:
        return f"HybMatrix({self.n_rows}x{self.n_cols}, K={self.k}, tail={self.coo_tail.nnz})"


FormatMatrix = CsrMatrix | Csr5Matrix | EllMatrix | SellMatrix | HybMatrix


# ---------------------------------------------------------------------------
# Converters
# ---------------------------------------------------------------------------
def _as_csr(a) -> CsrMatrix:
    return a if isinstance(a, CsrMatrix) else to_csr(a)


def to_csr(a: CooMatrix) -> CsrMatrix:
    """Compress canonical COO rows into a row pointer (formats.py:183-188)."""
    dev = a.device
    p = _i32(a.n_rows + 1, dev)
    col = _i32(a.nnz, dev)
    val = _f64(a.nnz, dev)
    with torch.cuda.device(dev):
        check(
            LIB.spmvb_coo_to_csr(
                ptr(a.row), ptr(a.col), ptr(a.data), a.nnz, a.n_rows, ptr(p), ptr(col), ptr(val), _lib.stream(dev)
            )
        )
    return CsrMatrix(a.n_rows, a.n_cols, p, col, val)


def to_csr5(a, omega: int, sigma: int) -> Csr5Matrix:
    """CSR5 tiles + descriptor (formats.py:196-250), bit-exact arrays."""
    if omega < 1 or sigma < 1:
        raise ValueError(f"omega and sigma must be >= 1, got {omega}, {sigma}")
    csr = _as_csr(a)
    dev = csr.device
    nnz = csr.nnz
    tile = omega * sigma
    num_tiles = -(-nnz // tile)
    tile_ptr = _i32(num_tiles + 1, dev)
    bit_flag = torch.empty(nnz, dtype=torch.bool, device=dev)
    y_off = torch.zeros((num_tiles, omega), dtype=torch.int32, device=dev)
    seg_off = torch.zeros((num_tiles, omega), dtype=torch.int32, device=dev)
    col = _i32(nnz, dev)
    val = _f64(nnz, dev)
    aux = torch.empty(num_tiles, dtype=torch.int32, device=dev)  # uint32 words
    with torch.cuda.device(dev):
        s = _lib.stream(dev)
        check(
            LIB.spmvb_csr_to_csr5(
                csr.n_rows, nnz, ptr(csr.ptr), ptr(csr.indices), ptr(csr.data), omega, sigma, ptr(tile_ptr),
                ptr(bit_flag), ptr(y_off), ptr(seg_off), ptr(col), ptr(val), ptr(aux), s,
            )
        )
        _, _, nonempty = _row_stats(csr.ptr, csr.n_rows)
        rows = None
        if nnz and nonempty < csr.n_rows:
            rows = _i32(nonempty, dev)
            check(LIB.spmvb_csr_nonempty_rows(ptr(csr.ptr), csr.n_rows, ptr(rows), s))
            if int(rows[-1].item()) == nonempty - 1:
                # the non-empty rows are the prefix [0, nonempty) (e.g. the
                # degree-ordered layout of relabel.py): no row lookup, the
                # empty tail is zeroed without ptr tests (spmvb.h)
                rows = None
        # kernel-side: the flags packed one bit per entry (64 B per 512-entry tile)
        bits = _i32((nnz + 31) // 32, dev)
        check(LIB.spmvb_csr5_pack_flags(nnz, ptr(bit_flag), ptr(bits), s))
    m = Csr5Matrix(csr.n_rows, csr.n_cols, csr.ptr, omega, sigma, num_tiles, tile_ptr, bit_flag, y_off, seg_off,
                   col, val, aux, rows, nonempty)
    m.flag_bits = bits
    return m


def to_ell(a, max_cells: int = DEFAULT_MAX_GRID_CELLS) -> EllMatrix:
    """Padded (n_rows, k) grid, k = widest row (formats.py:281-288)."""
    csr = _as_csr(a)
    dev = csr.device
    n = csr.n_rows
    k = _row_stats(csr.ptr, n)[1] if n else 0
    if n * k > max_cells:  # checked before allocation, as formats.py:263-267
        raise ConversionError(
            f"padded grid of {n}x{k} = {n * k} cells exceeds the {max_cells}-cell limit"
        )
    gi = torch.empty((k, n), dtype=torch.int32, device=dev)
    gd = torch.empty((k, n), dtype=torch.float64, device=dev)
    row_nnz = _i64(n, dev)
    with torch.cuda.device(dev):
        check(
            LIB.spmvb_csr_to_ell(
                n, ptr(csr.ptr), ptr(csr.indices), ptr(csr.data), k, max_cells, ptr(gi), ptr(gd), ptr(row_nnz),
                _lib.stream(dev),
            )
        )
    return EllMatrix(n, csr.n_cols, k, gi, gd, row_nnz)


def to_sell(a, c: int, sigma: int = 0, max_cells: int = DEFAULT_MAX_GRID_CELLS) -> SellMatrix:
    """Sliced ELL, optional sigma-window descending sort (formats.py:291-344)."""
    if c < 1:
        raise ValueError(f"slice height c must be >= 1, got {c}")
    if sigma < 0 or (sigma > 0 and sigma % c != 0):
        raise ValueError(
            f"sorting window sigma must be 0 or a positive multiple of c, got sigma={sigma}, c={c}"
        )
    csr = _as_csr(a)
    dev = csr.device
    n = csr.n_rows
    n_slices = -(-n // c)
    perm = _i32(n, dev)
    widths = _i64(n_slices, dev)
    slice_off = _i64(n_slices + 1, dev)
    row_nnz_perm = _i64(n, dev)
    total = ctypes.c_int64()
    with torch.cuda.device(dev):
        s = _lib.stream(dev)
        check(
            LIB.spmvb_sell_plan(
                n, ptr(csr.ptr), c, sigma, max_cells, ptr(perm), ptr(widths), ptr(slice_off), ptr(row_nnz_perm),
                ctypes.byref(total), s,
            )
        )
        cells = int(total.value)
        fi = _i32(cells, dev)
        fd = _f64(cells, dev)
        check(
            LIB.spmvb_sell_fill(
                n, ptr(csr.ptr), ptr(csr.indices), ptr(csr.data), c, ptr(perm), ptr(widths), ptr(slice_off),
                ptr(fi), ptr(fd), s,
            )
        )
    return SellMatrix(n, csr.n_cols, c, sigma, perm, widths, slice_off, fi, fd, row_nnz_perm)


def hyb_typical_k(row_nnz) -> int:
    """Largest K reached by strictly more than a third of the rows, else 1.

    formats.py:347-358, computed on the GPU from the per-row counts."""
    if isinstance(row_nnz, torch.Tensor) and row_nnz.is_cuda:
        counts = row_nnz.reshape(-1).to(torch.int64).contiguous()
    else:
        arr = np.asarray(row_nnz, dtype=np.int64).ravel()
        counts = torch.from_numpy(np.ascontiguousarray(arr)).to(_lib.require_cuda())
    n = int(counts.shape[0])
    if n == 0:
        raise ValueError("typical width is undefined for a matrix with no rows")
    out = ctypes.c_int64()
    with torch.cuda.device(counts.device):
        check(LIB.spmvb_typical_k_counts(ptr(counts), n, ctypes.byref(out), _lib.stream(counts.device)))
    return int(out.value)


def to_hyb(a, max_cells: int = DEFAULT_MAX_GRID_CELLS) -> HybMatrix:
    """ELL part of width K = hyb_typical_k plus the overflow COO tail (formats.py:361-397)."""
    csr = _as_csr(a)
    dev = csr.device
    n = csr.n_rows
    if csr.nnz == 0:
        counts = torch.zeros(n, dtype=torch.int64, device=dev)
        ell = EllMatrix(n, csr.n_cols, 0, torch.empty((0, n), dtype=torch.int32, device=dev),
                        torch.empty((0, n), dtype=torch.float64, device=dev), counts)
        return HybMatrix(ell, _empty(n, csr.n_cols, dev), torch.zeros(n + 1, dtype=torch.int32, device=dev))
    k = ctypes.c_int64()
    tail_nnz = ctypes.c_int64()
    tail_ptr = _i32(n + 1, dev)
    with torch.cuda.device(dev):
        s = _lib.stream(dev)
        check(LIB.spmvb_hyb_typical_k(ptr(csr.ptr), n, ctypes.byref(k), s))
        K = int(k.value)
        if n * K > max_cells:
            raise ConversionError(f"padded grid of {n}x{K} = {n * K} cells exceeds the {max_cells}-cell limit")
        check(LIB.spmvb_hyb_plan(n, ptr(csr.ptr), K, max_cells, ptr(tail_ptr), ctypes.byref(tail_nnz), s))
        t = int(tail_nnz.value)
        gi = torch.empty((K, n), dtype=torch.int32, device=dev)
        gd = torch.empty((K, n), dtype=torch.float64, device=dev)
        ell_nnz = _i64(n, dev)
        tr, tc, tv = _i32(t, dev), _i32(t, dev), _f64(t, dev)
        check(
            LIB.spmvb_hyb_fill(
                n, ptr(csr.ptr), ptr(csr.indices), ptr(csr.data), K, ptr(tail_ptr), ptr(gi), ptr(gd), ptr(ell_nnz),
                ptr(tr), ptr(tc), ptr(tv), s,
            )
        )
    ell = EllMatrix(n, csr.n_cols, K, gi, gd, ell_nnz)
    return HybMatrix(ell, CooMatrix(n, csr.n_cols, tr, tc, tv), tail_ptr)


def _ell_triplets(m: EllMatrix):
    dev = m.device
    total = int(m.row_nnz.sum().item()) if m.n_rows else 0
    r, c, v = _i32(total, dev), _i32(total, dev), _f64(total, dev)
    if m.n_rows:
        with torch.cuda.device(dev):
            check(
                LIB.spmvb_ell_to_coo(
                    m.n_rows, m.k, ptr(m.grid_indices), ptr(m.grid_data), ptr(m.row_nnz), ptr(r), ptr(c), ptr(v),
                    _lib.stream(dev),
                )
            )
    return r, c, v


def to_coo(m) -> CooMatrix:
    """Recover the canonical COO source of any format instance, bit-exactly.

    formats.py:406-453: triplets are extracted on the GPU and passed through
    ``canonicalize``, as the reference does."""
    if isinstance(m, CsrMatrix):
        dev = m.device
        rows = _i32(m.nnz, dev)
        with torch.cuda.device(dev):
            check(LIB.spmvb_csr_expand_rows(ptr(m.ptr), m.n_rows, ptr(rows), _lib.stream(dev)))
        return canonicalize(rows, m.indices, m.data, m.n_rows, m.n_cols, device=dev)
    if isinstance(m, Csr5Matrix):
        dev = m.device
        rows, col, val = _i32(m.nnz, dev), _i32(m.nnz, dev), _f64(m.nnz, dev)
        with torch.cuda.device(dev):
            s = _lib.stream(dev)
            check(LIB.spmvb_csr5_unstore(m.nnz, m.omega, m.sigma, ptr(m.indices), ptr(m.data), ptr(col), ptr(val), s))
            check(LIB.spmvb_csr_expand_rows(ptr(m.ptr), m.n_rows, ptr(rows), s))
        return canonicalize(rows, col, val, m.n_rows, m.n_cols, device=dev)
    if isinstance(m, EllMatrix):
        r, c, v = _ell_triplets(m)
        return canonicalize(r, c, v, m.n_rows, m.n_cols, device=m.device)
    if isinstance(m, SellMatrix):
        dev = m.device
        total = m.nnz
        r, c, v = _i32(total, dev), _i32(total, dev), _f64(total, dev)
        if m.n_rows:
            with torch.cuda.device(dev):
                check(
                    LIB.spmvb_sell_to_coo(
                        m.n_rows, m.c, ptr(m.perm), ptr(m.slice_off), ptr(m.row_nnz_perm), ptr(m.flat_indices),
                        ptr(m.flat_data), ptr(r), ptr(c), ptr(v), _lib.stream(dev),
                    )
                )
        return canonicalize(r, c, v, m.n_rows, m.n_cols, device=dev)
    if isinstance(m, HybMatrix):
        # ELL part and tail merged per row on the device: already canonical
        dev = m.device
        t = m.coo_tail
        total = m.nnz
        r, c, v = _i32(total, dev), _i32(total, dev), _f64(total, dev)
        if m.n_rows:
            with torch.cuda.device(dev):
                check(
                    LIB.spmvb_hyb_to_coo(
                        m.n_rows, m.k, ptr(m.ell.grid_indices), ptr(m.ell.grid_data), ptr(m.ell.row_nnz), t.nnz,
                        ptr(t.row), ptr(t.col), ptr(t.data), ptr(m.tail_ptr), ptr(r), ptr(c), ptr(v),
                        _lib.stream(dev),
                    )
                )
        return canonicalize(r, c, v, m.n_rows, m.n_cols, device=dev)
    raise TypeError(f"not a format matrix: {type(m).__name__}")


def convert(
    tag: FormatTag,
    a,
    *,
    omega: int = 4,
    sigma: int = 16,
    sell_c: int = 4,
    sell_sigma: int = 0,
    max_cells: int = DEFAULT_MAX_GRID_CELLS,
) -> FormatMatrix:
    """Convert canonical COO to the tagged format (formats.py:456-476)."""
    tag = FormatTag(tag)
    if tag is FormatTag.CSR:
        return a if isinstance(a, CsrMatrix) else to_csr(a)
    if tag is FormatTag.CSR5:
        return to_csr5(a, omega, sigma)
    if tag is FormatTag.ELL:
        return to_ell(a, max_cells)
    if tag is FormatTag.SELL:
        return to_sell(a, sell_c, sell_sigma, max_cells)
    return to_hyb(a, max_cells)
