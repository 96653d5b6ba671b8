"""ctypes binding of libspmvb.so (the C ABI declared in include/spmvb.h).

The library is mandatory: there is no CPU fallback.  Importing the package
on a machine without the built library raises immediately; calling a compute
entry point without a CUDA device raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

# SPMVB_LIB_PATH: another build of the same ABI (A/B experiments between builds only)
_LIB_PATH = Path(os.environ.get("SPMVB_LIB_PATH") or Path(__file__).resolve().with_name("libspmvb.so"))

SPMVB_OK = 0
SPMVB_INVALID_ARG = 1
SPMVB_GRID_TOO_LARGE = 2
SPMVB_OUT_OF_RANGE = 3
SPMVB_CUDA_ERROR = 4
SPMVB_OUT_OF_MEMORY = 5
SPMVB_INTERNAL = 6


class ConversionError(RuntimeError):
    """A format conversion could not be carried out (grid too large).

    Mirrors ``spmvkit.formats.ConversionError`` (formats.py:61-62)."""


c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
vp = ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_dbl = ctypes.POINTER(ctypes.c_double)
P_vp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); every symbol declared in include/spmvb.h.
SIGNATURES: dict[str, tuple] = {
    "spmvb_last_error": (ctypes.c_char_p, []),
    "spmvb_abi_version": (c_int, []),
    "spmvb_launch_count": (ctypes.c_ulonglong, []),
    "spmvb_canonicalize_begin": (c_int, [vp, vp, c_int, vp, c_i64, c_i64, c_i64, P_vp, P_i64, P_i64, vp]),
    "spmvb_canonicalize_finish": (c_int, [vp, vp, vp, vp, vp]),
    "spmvb_canonicalize_free": (None, [vp]),
    "spmvb_mm_format_begin": (c_int, [vp, vp, vp, c_i64, c_int, P_vp, P_i64]),
    "spmvb_mm_format_finish": (c_int, [vp, vp]),
    "spmvb_mm_parse": (
        c_int,
        [vp, c_i64, c_int, c_int, c_i64, c_i64, c_i64, c_i64, vp, vp, vp, P_i64, P_i64, P_i64, c_int],
    ),
    "spmvb_row_nnz_histogram": (c_int, [vp, c_i64, c_i64, vp, vp]),
    "spmvb_spmv_sequential": (c_int, [c_i64, vp, vp, vp, vp, vp, vp]),
    "spmvb_coo_to_csr": (c_int, [vp, vp, vp, c_i64, c_i64, vp, vp, vp, vp]),
    "spmvb_csr_row_stats": (c_int, [vp, c_i64, P_i64, vp]),
    "spmvb_csr_to_csr5": (c_int, [c_i64, c_i64, vp, vp, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_csr_nonempty_rows": (c_int, [vp, c_i64, vp, vp]),
    "spmvb_csr_to_ell": (c_int, [c_i64, vp, vp, vp, c_i64, c_i64, vp, vp, vp, vp]),
    "spmvb_sell_plan": (c_int, [c_i64, vp, c_i64, c_i64, c_i64, vp, vp, vp, vp, P_i64, vp]),
    "spmvb_sell_fill": (c_int, [c_i64, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp]),
    "spmvb_hyb_typical_k": (c_int, [vp, c_i64, P_i64, vp]),
    "spmvb_typical_k_counts": (c_int, [vp, c_i64, P_i64, vp]),
    "spmvb_csr_expand_rows": (c_int, [vp, c_i64, vp, vp]),
    "spmvb_csr5_unstore": (c_int, [c_i64, c_int, c_int, vp, vp, vp, vp, vp]),
    "spmvb_ell_to_coo": (c_int, [c_i64, c_i64, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_sell_to_coo": (c_int, [c_i64, c_i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_hyb_to_coo": (c_int, [c_i64, c_i64, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_hyb_plan": (c_int, [c_i64, vp, c_i64, c_i64, vp, P_i64, vp]),
    "spmvb_hyb_fill": (c_int, [c_i64, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_csr_chunk_size": (c_i64, []),
    "spmvb_csr_chunks": (c_i64, [c_i64]),
    "spmvb_csr_chunk_plan": (c_int, [c_i64, c_i64, vp, vp, c_i64, vp, vp]),
    "spmvb_spmv_csr": (c_int, [c_i64, c_i64, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_spmv_hyb": (
        c_int,
        [c_i64, c_i64, vp, vp, c_i64, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp],
    ),
    "spmvb_spmv_csr_exact": (c_int, [c_i64, c_i64, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_spmv_csr5_exact": (c_int, [c_i64, c_i64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp]),
    "spmvb_spmv_hyb_exact": (c_int, [c_i64, c_i64, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_csr5_pack_flags": (c_int, [c_i64, vp, vp, vp]),
    "spmvb_spmv_csr5": (
        c_int,
        [c_i64, c_i64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, vp],
    ),
    "spmvb_spmv_csr5_push": (
        c_int,
        [c_i64, c_i64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, c_int, c_i64, vp],
    ),
    "spmvb_csr5_range_bounds": (c_int, [c_i64, c_int, c_int, vp, vp, c_int, vp, vp, vp]),
    "spmvb_spmv_csr5_tiles": (
        c_int,
        [c_i64, c_i64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, c_i64, c_i64, c_i64,
         c_i64, vp],
    ),
    "spmvb_spmv_csr5_host": (
        c_int,
        [c_i64, c_i64, c_i64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp, c_i64, vp, vp, vp, vp, vp, vp, c_int,
         vp, vp, vp],
    ),
    "spmvb_spmv_ell": (c_int, [c_i64, c_i64, c_i64, vp, vp, vp, vp, vp, vp]),
    "spmvb_sell_wide_plan": (c_int, [c_i64, c_i64, vp, c_i64, vp, P_i64, P_i64, vp, P_i64, vp]),
    "spmvb_spmv_sell": (c_int, [c_i64, c_i64, vp, vp, vp, vp, vp, vp, c_i64, vp, c_i64, vp, c_i64, c_i64, c_i64,
                                c_i64, vp, vp, vp, vp]),
    "spmvb_spmv_sell_range": (c_int, [c_i64, c_i64, vp, vp, vp, vp, vp, vp, c_i64, vp, c_i64, vp, c_i64, c_i64, c_i64,
                                      c_i64, vp, vp, vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, vp]),
    "spmvb_sumsq": (c_int, [vp, c_i64, vp, vp]),
    "spmvb_inv_sqrt": (c_int, [vp, vp, vp]),
    "spmvb_norm_ws_bytes": (c_i64, []),
    "spmvb_norm_scale": (c_int, [vp, c_i64, vp, vp, vp, vp]),
    "spmvb_column_set": (c_int, [vp, c_i64, c_i64, vp, P_i64, vp]),
    "spmvb_gather_f64": (c_int, [vp, c_i64, vp, c_i64, vp, vp]),
    "spmvb_scatter_f64": (c_int, [vp, vp, c_i64, vp, vp]),
    "spmvb_degree_order": (c_int, [c_i64, vp, vp, c_i64, c_int, vp, vp, P_i64, vp]),
    "spmvb_relabel_csr": (c_int, [c_i64, vp, vp, vp, c_i64, vp, vp, vp, vp, vp]),
    "spmvb_push_rows": (c_int, [vp, c_i64, vp, c_int, c_i64, vp]),
    "spmvb_dist_init": (c_int, [vp, c_int, c_int, vp, P_vp]),
    "spmvb_dist_step": (c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_dist_destroy": (c_int, [vp]),
    "spmvb_dist_nccl_version": (c_int, [ctypes.POINTER(c_int)]),
    "spmvb_dist_init_ranges": (c_int, [vp, c_int, c_int, vp, c_int, vp, P_vp]),
    "spmvb_dist_step_ranges": (c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvb_sum_inv_sqrt": (c_int, [vp, c_int, vp, vp, vp]),
    "spmvb_gather_probe_threads": (c_i64, []),
    "spmvb_gather_probe": (c_int, [vp, vp, c_i64, vp, vp]),
    "spmvb_dot_probe": (c_int, [vp, vp, vp, c_i64, vp, vp]),
    "spmvb_csr_features": (c_int, [c_i64, c_i64, c_i64, vp, P_dbl, vp]),
    "spmvb_csr_extra_features": (c_int, [c_i64, c_i64, vp, vp, P_dbl, vp]),
    "spmvb_rmat_begin": (c_int, [c_int, c_i64, c_dbl, c_dbl, c_dbl, c_u64, P_vp, P_i64, vp]),
    "spmvb_rmat_finish": (c_int, [vp, vp, vp, vp, vp]),
    "spmvb_rmat_free": (None, [vp]),
    "spmvb_fill_uniform": (c_int, [vp, c_i64, c_dbl, c_dbl, c_u64, vp]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def library_path() -> Path:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load libspmvb.so once; raise loudly if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ImportError(
                    f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                if os.environ.get("SPMVB_LIB_PATH") and not hasattr(lib, name):
                    continue  # an older build under A/B: entry points it lacks stay unbound
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


class _Lib:
    def __getattr__(self, name):
        return getattr(load(), name)


LIB = _Lib()


def last_error() -> str:
    msg = load().spmvb_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status == SPMVB_OK:
        return
    msg = last_error()
    if status in (SPMVB_INVALID_ARG, SPMVB_OUT_OF_RANGE):
        raise ValueError(msg)
    if status == SPMVB_GRID_TOO_LARGE:
        raise ConversionError(msg)
    if status == SPMVB_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1805_11938_b200 requires a CUDA device (B200); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None):
    """Device pointer of a tensor (None / empty -> NULL)."""
    if t is None or t.numel() == 0:
        return None
    return t.data_ptr()
