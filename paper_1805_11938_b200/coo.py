"""Canonical COO matrices on the GPU (mirrors spmvkit.coo).

Reference: /root/reference/pkg/src/spmvkit/coo.py.  A :class:`CooMatrix`
holds int32 ``row``/``col`` and float64 ``data`` CUDA tensors, sorted by
(row, col), duplicate-free, without stored zeros (coo.py:45-62).  The
reference stores int64 indices under a 32-bit contract (coo.py:37-38); values
compare equal element by element.

``canonicalize`` runs entirely on the device (LSD radix sort of the
(row, col) key, numpy-order duplicate sums, zero drop); see
csrc/coo.cu.  Matrix Market entries are tokenized on the host by a native
multithreaded parser (csrc/mmio.cpp) and handed to the GPU ``canonicalize``.
"""

from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._lib import LIB, check, ptr

__all__ = [
    "INDEX_LIMIT",
    "CooMatrix",
    "MatrixMarketError",
    "canonicalize",
    "coo_equal",
    "dense_spmv_oracle",
    "read_matrix_market",
    "row_nnz_histogram",
    "write_matrix_market",
]

INDEX_LIMIT = 2**32 - 1  # coo.py:38


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; the message names the offending line."""


@dataclass(eq=False)
class CooMatrix:
    """Canonical triplets on the GPU (int32 row/col, float64 data)."""

    n_rows: int
    n_cols: int
    row: torch.Tensor
    col: torch.Tensor
    data: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.data.shape[0])

    @property
    def device(self) -> torch.device:
        return self.data.device

    def to_host(self):
        """(row, col, data) as int64/int64/float64 numpy arrays."""
        return (
            self.row.cpu().numpy().astype(np.int64),
            self.col.cpu().numpy().astype(np.int64),
            self.data.cpu().numpy(),
        )


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    return _lib.require_cuda()


def _as_index_tensor(v, device: torch.device) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        t = v.reshape(-1)
        if t.dtype not in (torch.int32, torch.int64):
            t = t.to(torch.int64)
        return t.to(device).contiguous()
    arr = np.asarray(v, dtype=np.int64).ravel()
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


def _as_value_tensor(v, device: torch.device) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        return v.reshape(-1).to(device=device, dtype=torch.float64).contiguous()
    arr = np.asarray(v, dtype=np.float64).ravel()
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


def _check_shape(n_rows: int, n_cols: int) -> None:
    # coo.py:77-83
    if n_rows < 0 or n_cols < 0:
        raise ValueError(f"negative matrix shape {n_rows}x{n_cols}")
    if n_rows > INDEX_LIMIT or n_cols > INDEX_LIMIT:
        raise ValueError(f"matrix shape {n_rows}x{n_cols} exceeds the 32-bit index range")


def _empty(n_rows: int, n_cols: int, device: torch.device) -> CooMatrix:
    return CooMatrix(
        n_rows,
        n_cols,
        torch.empty(0, dtype=torch.int32, device=device),
        torch.empty(0, dtype=torch.int32, device=device),
        torch.empty(0, dtype=torch.float64, device=device),
    )


def canonicalize(row, col, data, n_rows: int, n_cols: int, *, device=None) -> CooMatrix:
    """Sort by (row, col), sum duplicates (stable order), drop zero sums.

    Same contract and error messages as coo.py:86-125; runs on the GPU.
    """
    n_rows, n_cols = int(n_rows), int(n_cols)
    _check_shape(n_rows, n_cols)
    dev = _device(device)
    r = _as_index_tensor(row, dev)
    c = _as_index_tensor(col, dev)
    v = _as_value_tensor(data, dev)
    if not (r.shape == c.shape == v.shape):
        raise ValueError(
            f"triplet arrays disagree in length: {r.shape[0]}, {c.shape[0]}, {v.shape[0]}"
        )
    nnz = int(r.shape[0])
    if nnz > INDEX_LIMIT:
        raise ValueError(f"nnz {nnz} exceeds the 32-bit index range")
    if nnz == 0:
        return _empty(n_rows, n_cols, dev)
    if r.dtype != c.dtype:
        r, c = r.to(torch.int64), c.to(torch.int64)
    width = 4 if r.dtype == torch.int32 else 8
    with torch.cuda.device(dev):
        s = _lib.stream(dev)
        plan = ctypes.c_void_p()
        nnz_out = ctypes.c_int64()
        bad = (ctypes.c_int64 * 3)()
        check(
            LIB.spmvb_canonicalize_begin(
                ptr(r), ptr(c), width, ptr(v), nnz, n_rows, n_cols, ctypes.byref(plan), ctypes.byref(nnz_out),
                bad, s,
            )
        )
        m = int(nnz_out.value)
        out = CooMatrix(
            n_rows,
            n_cols,
            torch.empty(m, dtype=torch.int32, device=dev),
            torch.empty(m, dtype=torch.int32, device=dev),
            torch.empty(m, dtype=torch.float64, device=dev),
        )
        check(LIB.spmvb_canonicalize_finish(plan, ptr(out.row), ptr(out.col), ptr(out.data), s))
    return out


def _host_arrays(a):
    """(n_rows, n_cols, row, col, data) as numpy for either package's CooMatrix."""
    if isinstance(a, CooMatrix):
        r, c, d = a.to_host()
        return a.n_rows, a.n_cols, r, c, d
    return (
        int(a.n_rows),
        int(a.n_cols),
        np.asarray(a.row, dtype=np.int64),
        np.asarray(a.col, dtype=np.int64),
        np.asarray(a.data, dtype=np.float64),
    )


def coo_equal(a, b) -> bool:
    """Exact equality (coo.py:65-74); either side may be a reference CooMatrix."""
    if isinstance(a, CooMatrix) and isinstance(b, CooMatrix) and a.device == b.device:
        return (
            a.n_rows == b.n_rows
            and a.n_cols == b.n_cols
            and a.nnz == b.nnz
            and bool(torch.equal(a.row, b.row))
            and bool(torch.equal(a.col, b.col))
            and bool(torch.equal(a.data.view(torch.int64), b.data.view(torch.int64)))
        )
    ar, ac, arow, acol, adata = _host_arrays(a)
    br, bc, brow, bcol, bdata = _host_arrays(b)
    return (
        ar == br
        and ac == bc
        and adata.shape == bdata.shape
        and np.array_equal(arow, brow)
        and np.array_equal(acol, bcol)
        and adata.tobytes() == bdata.tobytes()
    )


def row_nnz_histogram(a: CooMatrix) -> torch.Tensor:
    """Stored nonzeros per row (int64 CUDA tensor), coo.py:144-146."""
    out = torch.zeros(a.n_rows, dtype=torch.int64, device=a.device)
    if a.n_rows:
        with torch.cuda.device(a.device):
            check(LIB.spmvb_row_nnz_histogram(ptr(a.row), a.nnz, a.n_rows, ptr(out), _lib.stream(a.device)))
    return out


def _row_ptr(a: CooMatrix) -> torch.Tensor:
    ptr_t = torch.empty(a.n_rows + 1, dtype=torch.int32, device=a.device)
    col = torch.empty(a.nnz, dtype=torch.int32, device=a.device)
    val = torch.empty(a.nnz, dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        check(
            LIB.spmvb_coo_to_csr(
                ptr(a.row), ptr(a.col), ptr(a.data), a.nnz, a.n_rows, ptr(ptr_t), ptr(col), ptr(val),
                _lib.stream(a.device),
            )
        )
    return ptr_t


def dense_spmv_oracle(a: CooMatrix, x):
    """y = A x accumulated entry by entry in ascending (row, col) order.

    The reference's correctness contract (coo.py:128-141), evaluated on the
    GPU with separately rounded products: bit-identical to the reference.
    Returns the same container kind as ``x`` (CUDA tensor in, CUDA tensor
    out; host array in, numpy array out).
    """
    from .kernels import _prepare_x, _finish_y  # local import: kernels imports formats

    xd, ret = _prepare_x(x, a.n_cols, a.device)
    y = torch.empty(a.n_rows, dtype=torch.float64, device=a.device)
    if a.n_rows:
        p = _row_ptr(a)
        with torch.cuda.device(a.device):
            check(
                LIB.spmvb_spmv_sequential(
                    a.n_rows, ptr(p), ptr(a.col), ptr(a.data), ptr(xd), ptr(y), _lib.stream(a.device)
                )
            )
    return _finish_y(y, ret)


# ---------------------------------------------------------------------------
# Matrix Market I/O (host side; semantics of coo.py:149-278)
# ---------------------------------------------------------------------------
def _parse_header(lines: list[str]) -> tuple[bool, bool]:
    if not lines:
        raise MatrixMarketError("empty input (line 1)")
    head = lines[0].split()
    if len(head) != 5 or head[0].lower() != "%%matrixmarket":
        raise MatrixMarketError(f"malformed header {lines[0]!r} (line 1)")
    obj, layout, field, symmetry = (t.lower() for t in head[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r} (line 1)")
    if layout != "coordinate":
        raise MatrixMarketError(f"unsupported format {layout!r}, only coordinate is supported (line 1)")
    if field == "complex":
        raise MatrixMarketError("complex matrices are not supported (line 1)")
    if field not in ("real", "integer", "pattern"):
        raise MatrixMarketError(f"unsupported field {field!r} (line 1)")
    if symmetry not in ("general", "symmetric"):
        raise MatrixMarketError(f"unsupported symmetry {symmetry!r} (line 1)")
    return field == "pattern", symmetry == "symmetric"


# bytes on which str.splitlines()/strip() would differ from splitting on "\n"
_UNUSUAL = re.compile(rb"\r(?!\n)|[\x0b\x0c\x1c-\x1e\x80-\xff]")


def _read_bytes(source) -> bytes:
    if hasattr(source, "read"):
        raw = source.read()
        return raw if isinstance(raw, bytes) else raw.encode("utf-8")
    if isinstance(source, bytes):
        return source
    return Path(source).read_bytes()


def _fast_triplets(raw: bytes):
    """Header in Python, entries in the native multithreaded tokenizer
    (csrc/mmio.cpp).  Returns None whenever the reference-semantics parser
    must decide (errors, unusual text), so results and messages are the
    reference's in every case."""
    nl = raw.find(b"\n")
    if nl < 0:
        return None
    banner = raw[:nl - 1] if raw[:nl].endswith(b"\r") else raw[:nl]
    if b"\r" in banner:
        return None
    try:
        pattern, symmetric = _parse_header([banner.decode("ascii")])
    except (MatrixMarketError, UnicodeDecodeError):
        return None
    pos = nl + 1
    size_text = None
    while pos < len(raw):
        end = raw.find(b"\n", pos)
        end = len(raw) if end < 0 else end
        line = raw[pos:end]
        pos = end + 1
        try:
            cand = line.decode("ascii").strip()
        except UnicodeDecodeError:
            return None
        if cand and not cand.startswith("%"):
            size_text = cand
            break
    if size_text is None or _UNUSUAL.search(raw, 0, pos):
        return None
    fields = size_text.split()
    try:
        if len(fields) != 3:
            return None
        n_rows, n_cols, declared = (int(f) for f in fields)
    except ValueError:
        return None
    if min(n_rows, n_cols, declared) < 0 or max(n_rows, n_cols, declared) > INDEX_LIMIT:
        return None
    # the entries start at raw[pos]: hand the tokenizer the address (no copy
    # of the text); an entry line is at least 4 bytes ("1 1\n"), which bounds
    # the output without counting lines
    n_tail = max(len(raw) - pos, 0)
    base = ctypes.cast(ctypes.c_char_p(raw), ctypes.c_void_p).value or 0
    per = 2 if symmetric else 1
    cap = per * min(declared, n_tail // 4 + 1)
    rows = np.empty(cap, dtype=np.int64)
    cols = np.empty(cap, dtype=np.int64)
    vals = np.empty(cap, dtype=np.float64)
    n_out = ctypes.c_int64()
    err_line = ctypes.c_int64()
    err_ij = (ctypes.c_int64 * 2)()
    status = LIB.spmvb_mm_parse(
        base + min(pos, len(raw)), n_tail, int(pattern), int(symmetric), n_rows, n_cols, declared, cap, rows.ctypes.data,
        cols.ctypes.data, vals.ctypes.data, ctypes.byref(n_out), ctypes.byref(err_line), err_ij, os.cpu_count() or 1,
    )
    if status != 0:
        return None
    n = int(n_out.value)
    return rows[:n], cols[:n], vals[:n], n_rows, n_cols


def read_matrix_market(source, *, device=None) -> CooMatrix:
    """Parse coordinate Matrix Market text and canonicalize it on the GPU.

    1-based -> 0-based, symmetric storage mirrored, pattern entries = 1.0,
    errors name the line (MatrixMarketError), as coo.py:158-263.  Entries are
    tokenized by the native multithreaded parser; any error or unusual text
    is re-parsed by the reference-semantics parser below for the exact
    message.
    """
    raw = _read_bytes(source)
    fast = _fast_triplets(raw)
    if fast is not None:
        rows, cols, vals, n_rows, n_cols = fast
        return canonicalize(rows, cols, vals, n_rows, n_cols, device=device)
    rows, cols, vals, n_rows, n_cols = _parse_text_triplets(raw.decode("utf-8"))
    return canonicalize(rows, cols, vals, n_rows, n_cols, device=device)


def _parse_text_triplets(text: str):
    """Reference-semantics parser (coo.py:166-262): expanded triplets, or
    MatrixMarketError naming the offending line."""
    lines = text.splitlines()
    pattern, symmetric = _parse_header(lines)
    k = 1
    size_text = None
    while k < len(lines):
        cand = lines[k].strip()
        k += 1
        if cand and not cand.startswith("%"):
            size_text = cand
            break
    if size_text is None:
        raise MatrixMarketError(f"missing size line (line {len(lines)})")
    size_line_no = k
    fields = size_text.split()
    try:
        if len(fields) != 3:
            raise ValueError
        n_rows, n_cols, declared = (int(f) for f in fields)
        if min(n_rows, n_cols, declared) < 0:
            raise ValueError
    except ValueError:
        raise MatrixMarketError(f"malformed size line {size_text!r} (line {size_line_no})") from None
    if max(n_rows, n_cols, declared) > INDEX_LIMIT:
        raise MatrixMarketError(f"matrix exceeds the 32-bit index range (line {size_line_no})")

    need = 2 if pattern else 3
    rows: list[int] = []
    cols: list[int] = []
    vals: list[float] = []
    seen = 0
    for line_no in range(k + 1, len(lines) + 1):
        text = lines[line_no - 1].strip()
        if not text or text.startswith("%"):
            continue
        if seen == declared:
            raise MatrixMarketError(
                f"entry count mismatch: declared {declared}, found more (line {line_no})"
            )
        parts = text.split()
        if len(parts) != need:
            raise MatrixMarketError(f"malformed entry {text!r}, expected {need} fields (line {line_no})")
        try:
            i, j = int(parts[0]), int(parts[1])
            v = 1.0 if pattern else float(parts[2])
        except ValueError:
            raise MatrixMarketError(f"malformed entry {text!r} (line {line_no})") from None
        if not (1 <= i <= n_rows and 1 <= j <= n_cols):
            raise MatrixMarketError(
                f"index ({i}, {j}) out of declared bounds {n_rows}x{n_cols} (line {line_no})"
            )
        rows.append(i - 1)
        cols.append(j - 1)
        vals.append(v)
        if symmetric and i != j:
            rows.append(j - 1)
            cols.append(i - 1)
            vals.append(v)
        seen += 1
    if seen != declared:
        raise MatrixMarketError(
            f"entry count mismatch: declared {declared}, found {seen} (line {len(lines)})"
        )
    return rows, cols, vals, n_rows, n_cols


def write_matrix_market(a, dest) -> None:
    """``coordinate real general`` text, 1-based, 17 significant digits."""
    n_rows, n_cols, r, c, d = _host_arrays(a)
    head = f"%%MatrixMarket matrix coordinate real general\n{n_rows} {n_cols} {len(d)}\n"
    body = _format_entries(r, c, d)
    if hasattr(dest, "write"):
        try:
            dest.write(head + body.decode("ascii"))
        except TypeError:  # a binary stream
            dest.write(head.encode("ascii") + body)
    else:
        with open(dest, "wb") as fh:
            fh.write(head.encode("ascii"))
            fh.write(body)


def _format_entries(r, c, d) -> bytearray:
    """The entry lines ``"<i+1> <j+1> <v:.17g>\\n"`` of write_matrix_market,
    formatted by the native multithreaded formatter (csrc/mmio.cpp); byte
    for byte what the reference's Python expression produces."""
    r = np.ascontiguousarray(r, dtype=np.int64)
    c = np.ascontiguousarray(c, dtype=np.int64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    plan = ctypes.c_void_p()
    n = ctypes.c_int64()
    st = LIB.spmvb_mm_format_begin(r.ctypes.data, c.ctypes.data, d.ctypes.data, int(d.size), os.cpu_count() or 1,
                                   ctypes.byref(plan), ctypes.byref(n))
    if st != 0:
        raise MemoryError("Matrix Market formatter failed") if st == 5 else ValueError("bad triplet arrays")
    out = bytearray(int(n.value))
    buf = (ctypes.c_char * len(out)).from_buffer(out) if out else None
    LIB.spmvb_mm_format_finish(plan, ctypes.addressof(buf) if buf is not None else None)
    del buf
    return out
