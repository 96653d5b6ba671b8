"""SpMV entry points, one per storage format, plus the tag dispatcher.

Mirrors spmvkit.kernels (/root/reference/pkg/src/spmvkit/kernels.py): the
same names, signatures (``workers`` is accepted for compatibility; the GPU
kernel fixes its own decomposition) and error behaviour
(``ValueError("x has length L, expected N")``, ``ValueError("... does not
match ...")``).  Every call launches hand-written sm_100a kernels through
libspmvb.so; there is no CPU fallback.

Containers: a float64 CUDA tensor ``x`` gives a CUDA tensor ``y`` (no host
traffic); a CPU tensor gives a CPU tensor (pinned in -> pinned out, copies
on the current stream); anything else (numpy, list) is coerced like the
reference (``np.asarray(x, float64).ravel()``) and returns a numpy array.
Keyword-only extensions: ``out=`` (device output buffer) and ``scale=`` (a
device scalar multiplying every row result; power iteration uses it) and
``exact=True``: the reference's own summation order, so y equals spmvkit's
result (``workers=1``) bit for bit -- CSR / CSR5 / HYB run the reference-order
kernels of csrc/spmv_exact.cu (numpy's reduceat / bincount orders), SELL keeps
every slice on its thread-per-row path, ELL is unchanged; a verification mode,
slower than the default kernels, whose results meet the 1e-12 (|A||x|)
tolerance in a different fixed order.
Repeated calls are bit-identical (no floating-point atomics).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import LIB, check, ptr
from .formats import Csr5Matrix, CsrMatrix, EllMatrix, FormatMatrix, FormatTag, HybMatrix, SellMatrix

__all__ = ["BoundCall", "SpmvOperator", "bind", "bind_range", "plan_row_blocks", "spmv", "spmv_csr", "spmv_csr5", "spmv_csr5_push",
           "spmv_csr5_tiles", "spmv_ell", "spmv_hyb", "spmv_many", "spmv_sell", "spmv_sell_range"]


def plan_row_blocks(n_rows: int, workers: int) -> list[tuple[int, int]]:
    """Host task plan of the reference CPU path (kernels.py:61-66); kept for
    API compatibility.  The GPU kernels decompose by nonzero chunks, CSR5
    tiles or rows instead."""
    if n_rows == 0:
        return []
    block = max(1, n_rows // (4 * max(workers, 1)))
    return [(lo, min(lo + block, n_rows)) for lo in range(0, n_rows, block)]


def _prepare_x(x, n_cols: int, device: torch.device):
    """Move/validate x; returns (device tensor, how to return y)."""
    if isinstance(x, torch.Tensor):
        xv = x.reshape(-1)
        if xv.shape[0] != n_cols:
            raise ValueError(f"x has length {xv.shape[0]}, expected {n_cols}")
        if xv.is_cuda:
            if xv.device != device:
                raise ValueError(f"x is on {xv.device}, matrix is on {device}")
            return xv.to(torch.float64).contiguous(), ("cuda",)
        pinned = xv.is_pinned()
        xd = xv.to(torch.float64).contiguous().to(device, non_blocking=pinned)
        return xd, ("cpu", pinned)
    arr = np.asarray(x, dtype=np.float64).ravel()
    if arr.shape[0] != n_cols:
        raise ValueError(f"x has length {arr.shape[0]}, expected {n_cols}")
    xd = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    return xd, ("numpy",)


def _finish_y(y: torch.Tensor, how):
    if how[0] == "cuda":
        return y
    if how[0] == "cpu":
        pinned = how[1]
        host = torch.empty(y.shape, dtype=y.dtype, pin_memory=pinned)
        host.copy_(y, non_blocking=pinned)
        if pinned:
            torch.cuda.current_stream(y.device).synchronize()
        return host
    return y.cpu().numpy()


def _out(m, out):
    if out is None:
        return torch.empty(m.n_rows, dtype=torch.float64, device=m.device)
    if out.dtype != torch.float64 or not out.is_cuda or out.numel() != m.n_rows or not out.is_contiguous():
        raise ValueError("out must be a contiguous float64 CUDA tensor with n_rows elements")
    return out


def _is_host(a) -> bool:
    return a is not None and not (isinstance(a, torch.Tensor) and a.is_cuda)


def _host_out(out, n_rows: int) -> torch.Tensor:
    """A host ``out=`` buffer (CPU float64 tensor or writeable numpy array of
    n_rows elements) as a CPU tensor sharing its memory."""
    t = out if isinstance(out, torch.Tensor) else None
    if t is None and isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.writeable:
        t = torch.from_numpy(out)
    if t is None or t.dtype != torch.float64 or t.numel() != n_rows or not t.is_contiguous():
        raise ValueError("out must be a contiguous float64 tensor/array with n_rows elements")
    return t.reshape(-1)


def _run(m, x, out, scale, launch):
    host = _is_host(out)
    out_h = _host_out(out, m.n_rows) if host else None
    xd, how = _prepare_x(x, m.n_cols, m.device)
    y = _out(m, None if host else out)
    if m.n_rows:
        with torch.cuda.device(m.device):
            launch(xd, y, ptr(scale) if scale is not None else None, _lib.stream(m.device))
    if host:
        pinned = out_h.is_pinned()
        out_h.copy_(y, non_blocking=pinned)
        if pinned:
            torch.cuda.current_stream(m.device).synchronize()
        return out
    return _finish_y(y, how)


def _args_csr(m: CsrMatrix, xd, y, sp, scratch):
    plan = m.chunk_plan()
    cr, cv = scratch
    return "spmvb_spmv_csr", (m.n_rows, m.nnz, ptr(m.ptr), ptr(m.indices), ptr(m.data), ptr(plan.nz_rows), plan.n_nz,
                              ptr(plan.chunk_row), ptr(cr), ptr(cv), ptr(xd), ptr(y), sp)


def _scratch_csr(m: CsrMatrix):
    return m.chunk_plan().scratch(m.device)


def spmv_csr(m: CsrMatrix, x, workers: int = 1, *, out=None, scale=None, exact: bool = False):
    """y = A x for CSR via the chunked kernel (kernels.py:76-95);
    ``exact=True``: y_r = p_first + pairwise(rest), numpy's reduceat order."""
    if exact:
        def launch_exact(xd, y, sp, s):
            check(LIB.spmvb_spmv_csr_exact(m.n_rows, m.nnz, ptr(m.ptr), ptr(m.indices), ptr(m.data), ptr(xd), ptr(y),
                                           sp, s))

        return _run(m, x, out, scale, launch_exact)
    m.chunk_plan()

    def launch(xd, y, sp, s):
        name, args = _args_csr(m, xd, y, sp, _scratch_csr(m))
        check(getattr(LIB, name)(*args, s))

    return _run(m, x, out, scale, launch)


# Packed flag bits pay when x does not fit L2 (its gathers then miss, and the
# 8x smaller flag stream frees L1TEX and DRAM slots: C5 -4..6 % time); with x
# L2-resident (C4) the byte flags are ~3 % faster.  Results are identical.
_PACKED_FLAGS_MIN_X_BYTES = 64 << 20


def _packed_flags(m: Csr5Matrix):
    return m.flag_bits if m.n_cols * 8 >= _PACKED_FLAGS_MIN_X_BYTES else None


def _args_csr5(m: Csr5Matrix, xd, y, sp, carry):
    return "spmvb_spmv_csr5", (m.n_rows, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.tile_ptr), ptr(m.bit_flag),
                               ptr(_packed_flags(m)), ptr(m.indices), ptr(m.data), ptr(m.tile_aux),
                               ptr(m.nonempty_rows), m.n_nonempty, ptr(carry), ptr(xd), ptr(y), sp)


def _scratch_csr5(m: Csr5Matrix):
    return torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=m.device)


def spmv_csr5(m: Csr5Matrix, x, workers: int = 1, *, out=None, scale=None, ranges: int = 16, exact: bool = False):
    """y = A x for CSR5: per-tile segmented sums + ordered carry fix-up (kernels.py:139-174).
    ``exact=True``: per-tile reduceat sums added in ascending tile order, as the reference.

    Host x with a host (or no) ``out`` runs the streamed host-buffer entry
    point: x is copied in once, then ``ranges`` tile ranges compute in order
    while each range's finished rows of y are copied back on a second stream.
    """
    if exact:
        def launch_exact(xd, y, sp, s):
            check(LIB.spmvb_spmv_csr5_exact(m.n_rows, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.indices),
                                            ptr(m.data), ptr(xd), ptr(y), sp, s))

        return _run(m, x, out, scale, launch_exact)
    if _is_host(x) and (out is None or _is_host(out)):
        return _spmv_csr5_host(m, x, out, scale, ranges)

    def launch(xd, y, sp, s):
        name, args = _args_csr5(m, xd, y, sp, _scratch_csr5(m))
        check(getattr(LIB, name)(*args, s))

    return _run(m, x, out, scale, launch)


def spmv_csr5_tiles(m: Csr5Matrix, x: torch.Tensor, out: torch.Tensor, t_begin: int, t_end: int, row_begin: int,
                    row_end: int, *, scale=None, carry: torch.Tensor | None = None) -> torch.Tensor:
    """One range of a CSR5 SpMV on device buffers (spmvb_spmv_csr5_tiles):
    zero the empty rows of [row_begin, row_end) and run tiles [t_begin,
    t_end) with their fix-up.  Over the ranges of ``m.range_plan(k)``, in
    any order, this equals ``spmv_csr5(m, x, out=out)`` bit for bit; the
    multi-GPU power iteration sends each range's rows while the next one
    computes.  ``carry``: num_tiles doubles of scratch (allocated if None)."""
    xd = x.reshape(-1)
    if not xd.is_cuda or xd.dtype != torch.float64 or xd.numel() != m.n_cols:
        raise ValueError(f"x must be a float64 CUDA tensor of length {m.n_cols}")
    y = _out(m, out)
    if carry is None:
        carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=m.device)
    with torch.cuda.device(m.device):
        check(
            LIB.spmvb_spmv_csr5_tiles(
                m.n_rows, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.tile_ptr), ptr(m.bit_flag),
                ptr(_packed_flags(m)), ptr(m.indices),
                ptr(m.data), ptr(m.tile_aux), ptr(m.nonempty_rows), m.n_nonempty, ptr(carry), ptr(xd.contiguous()),
                ptr(y), ptr(scale) if scale is not None else None, int(t_begin), int(t_end), int(row_begin),
                int(row_end), _lib.stream(m.device),
            )
        )
    return y


def spmv_csr5_push(m: Csr5Matrix, x: torch.Tensor, out: torch.Tensor, peers: torch.Tensor, push_off: int, *,
                   scale=None, carry: torch.Tensor | None = None) -> torch.Tensor:
    """CSR5 SpMV fused with the multi-GPU exchange (spmvb_spmv_csr5_push):
    ``out = scale * A x`` and every row r is also stored at
    ``peers[p][push_off + r]`` (``peers``: int64 CUDA tensor of peer buffer
    addresses, e.g. symmetric-memory buffers of the other ranks).  Each block
    stores its rows right after computing them; the carry fix-up re-stores the
    rows it completes.  omega = 32, sigma = 16 or 8."""
    xd = x.reshape(-1)
    if not xd.is_cuda or xd.dtype != torch.float64 or xd.numel() != m.n_cols:
        raise ValueError(f"x must be a float64 CUDA tensor of length {m.n_cols}")
    if peers.dtype != torch.int64 or not peers.is_cuda:
        raise ValueError("peers must be an int64 CUDA tensor of buffer addresses")
    y = _out(m, out)
    if carry is None:
        carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=m.device)
    with torch.cuda.device(m.device):
        check(
            LIB.spmvb_spmv_csr5_push(
                m.n_rows, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.tile_ptr), ptr(m.bit_flag),
                ptr(_packed_flags(m)), ptr(m.indices), ptr(m.data), ptr(m.tile_aux), ptr(m.nonempty_rows),
                m.n_nonempty, ptr(carry), ptr(xd.contiguous()), ptr(y), ptr(scale) if scale is not None else None,
                ptr(peers), int(peers.numel()), int(push_off), _lib.stream(m.device),
            )
        )
    return y


def _spmv_csr5_host(m: Csr5Matrix, x, out, scale, ranges: int):
    if isinstance(x, torch.Tensor):
        xh = x.reshape(-1)
        kind = "tensor"
    else:
        xh = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel()))
        kind = "numpy"
    if xh.shape[0] != m.n_cols:
        raise ValueError(f"x has length {xh.shape[0]}, expected {m.n_cols}")
    xh = xh.to(torch.float64).contiguous()
    if out is not None:
        yh = _host_out(out, m.n_rows)
    else:
        yh = torch.empty(m.n_rows, dtype=torch.float64, pin_memory=kind == "tensor" and xh.is_pinned())
    dev = m.device
    tb, rb = m.range_plan(ranges)
    xd = torch.empty(max(m.n_cols, 1), dtype=torch.float64, device=dev)
    yd = torch.empty(max(m.n_rows, 1), dtype=torch.float64, device=dev)
    carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(
            LIB.spmvb_spmv_csr5_host(
                m.n_rows, m.n_cols, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.tile_ptr), ptr(m.bit_flag),
                ptr(_packed_flags(m)),
                ptr(m.indices), ptr(m.data), ptr(m.tile_aux), ptr(m.nonempty_rows), m.n_nonempty, ptr(carry),
                ptr(xh), ptr(xd), ptr(yd), ptr(yh), ptr(scale) if scale is not None else None, len(tb) - 1,
                tb.ctypes.data, rb.ctypes.data, _lib.stream(dev),
            )
        )
    if out is not None:
        return out
    return yh if kind == "tensor" else yh.numpy()


def _args_ell(m: EllMatrix, xd, y, sp, scratch):
    return "spmvb_spmv_ell", (m.n_rows, m.n_cols, m.k, ptr(m.grid_indices), ptr(m.grid_data), ptr(xd), ptr(y), sp)


def spmv_ell(m: EllMatrix, x, workers: int = 1, *, out=None, scale=None, exact: bool = False):
    """y = A x for ELL, sequential over the k slots (kernels.py:98-116): the
    reference recurrence, so ``exact`` changes nothing."""

    def launch(xd, y, sp, s):
        name, args = _args_ell(m, xd, y, sp, None)
        check(getattr(LIB, name)(*args, s))

    return _run(m, x, out, scale, launch)


def _args_sell(m: SellMatrix, xd, y, sp, scratch):
    wide, n_wide, max_narrow, first_piece, n_pieces, wide_cols, tail_from, hub, n_hub = m.wide_plan()
    perm = m.perm if m.sigma > 0 else None
    return "spmvb_spmv_sell", (m.n_rows, m.c, ptr(m.widths), ptr(m.slice_off), ptr(perm), ptr(m.flat_indices),
                               ptr(m.flat_data), ptr(wide), n_wide, ptr(first_piece), n_pieces, ptr(hub), n_hub,
                               wide_cols, tail_from, max_narrow, ptr(xd), ptr(y), sp)


def spmv_sell(m: SellMatrix, x, workers: int = 1, *, out=None, scale=None, exact: bool = False):
    """y = A x for SELL / SELL-C-sigma, scattered through perm (kernels.py:119-136).
    ``exact=True``: slices wider than the wide threshold also run a thread per
    row (the reference recurrence) instead of being summed in pieces."""
    if exact:
        def launch_exact(xd, y, sp, s):
            perm = m.perm if m.sigma > 0 else None
            check(LIB.spmvb_spmv_sell(m.n_rows, m.c, ptr(m.widths), ptr(m.slice_off), ptr(perm), ptr(m.flat_indices),
                                      ptr(m.flat_data), None, 0, None, 0, None, 0, 1 << 62, m.n_rows, -1, ptr(xd),
                                      ptr(y), sp, s))

        return _run(m, x, out, scale, launch_exact)
    m.wide_plan()

    def launch(xd, y, sp, s):
        name, args = _args_sell(m, xd, y, sp, None)
        check(getattr(LIB, name)(*args, s))

    return _run(m, x, out, scale, launch)


def spmv_sell_range(m: SellMatrix, x: torch.Tensor, out: torch.Tensor, r, *, scale=None) -> torch.Tensor:
    """One slice range of a SELL SpMV on device buffers (spmvb_spmv_sell_range);
    ``r`` is an entry of ``m.range_plan(k)``.  Over all of a plan's ranges, in
    any order, this equals ``spmv_sell(m, x, out=out)`` bit for bit; the
    multi-GPU power iteration sends each range's rows (r[6]:r[7] of y) while
    the next one computes."""
    xd = x.reshape(-1)
    if not xd.is_cuda or xd.dtype != torch.float64 or xd.numel() != m.n_cols:
        raise ValueError(f"x must be a float64 CUDA tensor of length {m.n_cols}")
    y = _out(m, out)
    wide, n_wide, max_narrow, first_piece, n_pieces, wide_cols, tail_from, hub, n_hub = m.wide_plan()
    perm = m.perm if m.sigma > 0 else None
    s0, s1, i0, i1, pc0, pc1 = (int(v) for v in r[:6])
    h0, h1 = int(r[8]), int(r[9])
    with torch.cuda.device(m.device):
        check(LIB.spmvb_spmv_sell_range(
            m.n_rows, m.c, ptr(m.widths), ptr(m.slice_off), ptr(perm), ptr(m.flat_indices), ptr(m.flat_data),
            ptr(wide), n_wide, ptr(first_piece), n_pieces, ptr(hub), n_hub, wide_cols, tail_from, max_narrow,
            ptr(xd.contiguous()), ptr(y), ptr(scale) if scale is not None else None, s0, s1, i0, i1, pc0, pc1, h0, h1,
            _lib.stream(m.device)))
    return y


def _args_hyb(m: HybMatrix, xd, y, sp, scratch):
    t = m.coo_tail
    plan = m.chunk_plan()
    cr, cv = scratch
    return "spmvb_spmv_hyb", (m.n_rows, m.k, ptr(m.ell.grid_indices), ptr(m.ell.grid_data), t.nnz, ptr(m.tail_ptr),
                              ptr(t.col), ptr(t.data), ptr(plan.nz_rows), plan.n_nz, ptr(plan.chunk_row), ptr(cr),
                              ptr(cv), ptr(xd), ptr(y), sp)


def _scratch_hyb(m: HybMatrix):
    return m.chunk_plan().scratch(m.device)


def spmv_hyb(m: HybMatrix, x, workers: int = 1, *, out=None, scale=None, exact: bool = False):
    """y = ELL part + COO tail (kernels.py:177-199), one fused kernel.
    ``exact=True``: ell_r + (the row's tail entries summed sequentially from
    0.0), the reference's spmv_ell + bincount order."""
    if exact:
        def launch_exact(xd, y, sp, s):
            t = m.coo_tail
            check(LIB.spmvb_spmv_hyb_exact(m.n_rows, m.k, ptr(m.ell.grid_indices), ptr(m.ell.grid_data), t.nnz,
                                           ptr(m.tail_ptr), ptr(t.col), ptr(t.data), ptr(xd), ptr(y), sp, s))

        return _run(m, x, out, scale, launch_exact)
    m.chunk_plan()

    def launch(xd, y, sp, s):
        name, args = _args_hyb(m, xd, y, sp, _scratch_hyb(m))
        check(getattr(LIB, name)(*args, s))

    return _run(m, x, out, scale, launch)


_KERNELS = {
    FormatTag.CSR: (CsrMatrix, spmv_csr),
    FormatTag.CSR5: (Csr5Matrix, spmv_csr5),
    FormatTag.ELL: (EllMatrix, spmv_ell),
    FormatTag.SELL: (SellMatrix, spmv_sell),
    FormatTag.HYB: (HybMatrix, spmv_hyb),
}


_BINDERS = {
    FormatTag.CSR: (_args_csr, _scratch_csr),
    FormatTag.CSR5: (_args_csr5, _scratch_csr5),
    FormatTag.ELL: (_args_ell, lambda m: None),
    FormatTag.SELL: (_args_sell, lambda m: None),
    FormatTag.HYB: (_args_hyb, _scratch_hyb),
}


class BoundCall:
    """One library launch with every argument resolved in advance: calling it
    is one ctypes call (no tensor checks, no allocation, no device context).
    The buffers it was bound to must stay alive and in place; the stream is
    the one current when it was bound."""

    __slots__ = ("_fn", "_args", "_keep", "stream")

    def __init__(self, name: str, args: tuple, stream: int, keep=()):
        self._fn = getattr(_lib.load(), name)
        self._args = tuple(args) + (stream,)
        self._keep = keep
        self.stream = stream

    def __call__(self) -> None:
        st = self._fn(*self._args)
        if st:
            check(st)


def bind(tag: FormatTag, m: FormatMatrix, x: torch.Tensor, out: torch.Tensor, scale: torch.Tensor | None = None
         ) -> BoundCall:
    """A prepared ``spmv(tag, m, x, out=out, scale=scale)`` on device buffers
    (the same kernels and results, bit for bit) for repeated calls on the same
    buffers, e.g. every step of a power iteration: the per-call host work of
    the generic entry point (argument checks, scratch allocation, device
    context, stream lookup) is done once here.  ``x``/``out``: contiguous
    float64 CUDA tensors of n_cols / n_rows elements on the matrix's device;
    ``scale``: a device scalar or None."""
    tag = FormatTag(tag)
    cls, _ = _KERNELS[tag]
    if not isinstance(m, cls):
        raise ValueError(f"format tag {tag.value!r} does not match {type(m).__name__}")
    for t, n, what in ((x, m.n_cols, "x"), (out, m.n_rows, "out")):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == n and t.device == m.device):
            raise ValueError(f"{what} must be a contiguous float64 CUDA tensor of {n} elements on {m.device}")
    if scale is not None and not (scale.is_cuda and scale.dtype == torch.float64 and scale.numel() >= 1):
        raise ValueError("scale must be a float64 CUDA scalar")
    args_fn, scratch_fn = _BINDERS[tag]
    scratch = scratch_fn(m)
    name, args = args_fn(m, x, out, ptr(scale) if scale is not None else None, scratch)
    return BoundCall(name, args, _lib.stream(m.device), keep=(m, x, out, scale, scratch))


def bind_range(tag: FormatTag, m: FormatMatrix, x: torch.Tensor, out: torch.Tensor, r, scale=None,
               carry: torch.Tensor | None = None) -> BoundCall:
    """A prepared row range of a CSR5 or SELL SpMV (``spmv_csr5_tiles`` /
    ``spmv_sell_range``): ``r`` is (row_begin, row_end, t_begin, t_end) for
    CSR5 (from ``m.range_plan``) or an entry of ``SellMatrix.range_plan``.
    ``out`` is the whole output vector of ``m`` (n_rows)."""
    tag = FormatTag(tag)
    for t, n, what in ((x, m.n_cols, "x"), (out, m.n_rows, "out")):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == n and t.device == m.device):
            raise ValueError(f"{what} must be a contiguous float64 CUDA tensor of {n} elements on {m.device}")
    sp = ptr(scale) if scale is not None else None
    st = _lib.stream(m.device)
    if tag is FormatTag.CSR5 and isinstance(m, Csr5Matrix):
        a, b, t0, t1 = (int(v) for v in r)
        if carry is None:
            carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=m.device)
        args = (m.n_rows, m.nnz, ptr(m.ptr), m.omega, m.sigma, ptr(m.tile_ptr), ptr(m.bit_flag),
                ptr(_packed_flags(m)), ptr(m.indices), ptr(m.data), ptr(m.tile_aux), ptr(m.nonempty_rows),
                m.n_nonempty, ptr(carry), ptr(x), ptr(out), sp, t0, t1, a, b)
        return BoundCall("spmvb_spmv_csr5_tiles", args, st, keep=(m, x, out, scale, carry))
    if tag is FormatTag.SELL and isinstance(m, SellMatrix):
        wide, n_wide, max_narrow, first_piece, n_pieces, wide_cols, tail_from, hub, n_hub = m.wide_plan()
        perm = m.perm if m.sigma > 0 else None
        s0, s1, i0, i1, pc0, pc1 = (int(v) for v in r[:6])
        args = (m.n_rows, m.c, ptr(m.widths), ptr(m.slice_off), ptr(perm), ptr(m.flat_indices), ptr(m.flat_data),
                ptr(wide), n_wide, ptr(first_piece), n_pieces, ptr(hub), n_hub, wide_cols, tail_from, max_narrow,
                ptr(x), ptr(out), sp, s0, s1, i0, i1, pc0, pc1, int(r[8]), int(r[9]))
        return BoundCall("spmvb_spmv_sell_range", args, st, keep=(m, x, out, scale))
    raise ValueError(f"row ranges exist for csr5 and sell matrices, not {tag.value!r} / {type(m).__name__}")


class SpmvOperator:
    """``op(x, out, scale)`` = ``spmv(tag, m, x, out=out, scale=scale)``, a
    ``local_spmv`` for ``dist.PowerIteration`` whose ``bind`` lets the
    iteration prepare its launches once per buffer pair (``kernels.bind``)."""

    def __init__(self, tag: FormatTag, m: FormatMatrix):
        self.tag = FormatTag(tag)
        cls, _ = _KERNELS[self.tag]
        if not isinstance(m, cls):
            raise ValueError(f"format tag {self.tag.value!r} does not match {type(m).__name__}")
        self.m = m

    def __call__(self, x, out, scale=None):
        return spmv(self.tag, self.m, x, out=out, scale=scale)

    def bind(self, x, out, scale=None) -> BoundCall:
        return bind(self.tag, self.m, x, out, scale)


def spmv(tag: FormatTag, m: FormatMatrix, x, workers: int = 1, **kw):
    """Dispatch to the kernel matching ``tag``; the instance type must agree."""
    cls, kernel = _KERNELS[FormatTag(tag)]
    if not isinstance(m, cls):
        raise ValueError(f"format tag {FormatTag(tag).value!r} does not match {type(m).__name__}")
    return kernel(m, x, workers, **kw)


def spmv_many(tag: FormatTag, m: FormatMatrix, xs, outs, *, scale=None, ranges: int = 16) -> list:
    """y_k = A x_k for a sequence of host vectors, transfers pipelined across
    vectors.  ``xs``: pinned float64 CPU tensors of length n_cols; ``outs``:
    pinned float64 CPU tensors of length n_rows (written in place, returned).

    The same results as ``spmv(tag, m, x_k, out=y_k)`` one after the other,
    bit for bit; but x_{k+1}'s host->device copy runs while y_k is computed
    and copied back (the PCIe link carries both directions at once), on two
    device buffer pairs.  CSR5 streams each of ``ranges`` row-aligned tile
    ranges back as soon as it is finished (as the single-vector host path);
    the other formats copy y_k back after its SpMV.  Returns ``outs``."""
    tag = FormatTag(tag)
    cls, _ = _KERNELS[tag]
    if not isinstance(m, cls):
        raise ValueError(f"format tag {tag.value!r} does not match {type(m).__name__}")
    xs, outs = list(xs), list(outs)
    if len(xs) != len(outs):
        raise ValueError(f"{len(xs)} inputs but {len(outs)} outputs")
    for xh in xs:
        if not (isinstance(xh, torch.Tensor) and not xh.is_cuda and xh.dtype == torch.float64
                and (xh.is_pinned() or xh.numel() == 0)):  # an empty tensor cannot be pinned
            raise ValueError("spmv_many needs pinned float64 CPU tensors (torch.empty(..., pin_memory=True))")
        if xh.numel() != m.n_cols:
            raise ValueError(f"x has length {xh.numel()}, expected {m.n_cols}")
    for yh in outs:
        if not (isinstance(yh, torch.Tensor) and not yh.is_cuda and yh.dtype == torch.float64
                and (yh.is_pinned() or yh.numel() == 0)):
            raise ValueError("spmv_many needs pinned float64 CPU output tensors")
        if yh.numel() != m.n_rows or not yh.is_contiguous():
            raise ValueError(f"out must be a contiguous tensor of length {m.n_rows}")
    if not xs:
        return outs
    dev = m.device
    with torch.cuda.device(dev):
        comp = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        s_in.wait_stream(comp)
        s_out.wait_stream(comp)
        xd = [torch.empty(max(m.n_cols, 1), dtype=torch.float64, device=dev) for _ in range(2)]
        yd = [torch.empty(max(m.n_rows, 1), dtype=torch.float64, device=dev) for _ in range(2)]
        x_free = [None, None]  # compute of the vector that last used xd[b] done
        y_free = [None, None]  # copy-back of the vector that last used yd[b] done
        plan = None
        if tag is FormatTag.CSR5 and m.nnz > 0 and m.n_rows > 0:
            tb, rb = m.range_plan(ranges)
            k_all = len(tb) - 1
            plan = [(int(rb[k]), int(rb[k + 1]) if k + 1 < k_all else m.n_rows, int(tb[k]), int(tb[k + 1]))
                    for k in range(k_all)][::-1]  # light rows (last ranges) first
            carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=dev)
        for k, (xh, yh) in enumerate(zip(xs, outs)):
            b = k % 2
            with torch.cuda.stream(s_in):
                if x_free[b] is not None:
                    s_in.wait_event(x_free[b])
                xd[b][: m.n_cols].copy_(xh.reshape(-1), non_blocking=True)
                x_in = torch.cuda.Event()
                x_in.record(s_in)
            comp.wait_event(x_in)
            if y_free[b] is not None:
                comp.wait_event(y_free[b])
            xv, yv = xd[b][: m.n_cols], yd[b][: m.n_rows]
            yflat = yh.reshape(-1)
            if plan is not None:
                for a, e, t0, t1 in plan:
                    spmv_csr5_tiles(m, xv, yv, t0, t1, a, e, scale=scale, carry=carry)
                    if e > a:
                        done = torch.cuda.Event()
                        done.record(comp)
                        s_out.wait_event(done)
                        with torch.cuda.stream(s_out):
                            yflat[a:e].copy_(yv[a:e], non_blocking=True)
            else:
                spmv(tag, m, xv, out=yv, scale=scale)
                done = torch.cuda.Event()
                done.record(comp)
                s_out.wait_event(done)
                with torch.cuda.stream(s_out):
                    yflat.copy_(yv, non_blocking=True)
            x_free[b] = torch.cuda.Event()
            x_free[b].record(comp)
            y_free[b] = torch.cuda.Event()
            y_free[b].record(s_out)
            # the host buffers stay referenced by the caller; the device ones
            # are released only after the streams below are joined
        comp.wait_stream(s_in)
        comp.wait_stream(s_out)
        comp.synchronize()
    return outs
