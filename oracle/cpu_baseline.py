"""CPU baseline for bench.py (BENCH INFRASTRUCTURE; see oracle/port.py).

Times the reference's CPU SpMV algorithm (restated in oracle/port.py:
per-row-block products + numpy add.reduceat on a thread pool, exactly the
structure of spmvkit.kernels.spmv_csr, kernels.py:76-95) on a bounded,
unbiased sample of the benchmark matrix:

* R-MAT configs: every row r with mix64(r ^ 0xA5A5A5A5) % keep_mod == 0
  (about 1/keep_mod of the rows, all their entries; x keeps its full length
  so the gather footprint is the real one).  Draws are regenerated on the
  host by oracle/rmat_sample.c with the GPU generator's hash, deduplicated
  keeping the first draw, canonicalized with oracle/port.canonicalize.
* The rate is reported as GFLOP/s = 2 * nnz_sample / t (per-SpMV mean).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from pathlib import Path

import numpy as np

from . import port, synth_ref

HERE = Path(__file__).resolve().parent
SO = HERE / "_build" / "librmat_sample.so"


def _lib():
    if not SO.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    lib = ctypes.CDLL(str(SO))
    lib.rmat_sample_ranges.restype = ctypes.c_int64
    lib.rmat_sample_ranges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                       ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.rmat_csr.restype = ctypes.c_int64
    lib.rmat_csr.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                             ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                             ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
    lib.rmat_csr_free.restype = None
    lib.rmat_csr_free.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return lib


def rmat_full_csr(scale: int, edge_factor: int, seed: int, threads: int | None = None):
    """The whole R-MAT matrix (first-draw dedup) as canonical host CSR
    (ptr, indices, data) with int64 indices like the reference's arrays
    (formats.py:183-188), built by oracle/rmat_sample.c:rmat_csr."""
    threads = threads or port.host_cores()
    lib = _lib()
    n = 1 << scale
    p, c, v = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    nnz = lib.rmat_csr(scale, edge_factor << scale, 0.57, 0.19, 0.19, seed, threads, ctypes.byref(p),
                       ctypes.byref(c), ctypes.byref(v))
    if nnz < 0:
        raise MemoryError("rmat_csr: host allocation failed")
    try:
        ptr = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_int64)), (n + 1,)).copy()
        ind = np.ctypeslib.as_array(ctypes.cast(c, ctypes.POINTER(ctypes.c_int32)), (max(nnz, 1),))[:nnz]
        ind = ind.astype(np.int64)
        dat = np.ctypeslib.as_array(ctypes.cast(v, ctypes.POINTER(ctypes.c_double)), (max(nnz, 1),))[:nnz].copy()
    finally:
        lib.rmat_csr_free(p, c, v)
    return ptr, ind, dat


def host_ram_available() -> int:
    """MemAvailable of this host in bytes (0 if unknown)."""
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except (OSError, ValueError, IndexError):
        pass
    return 0


def kept_rows(n: int, keep_mod: int) -> np.ndarray:
    r = np.arange(n, dtype=np.uint64)
    h = synth_ref.mix64(r ^ np.uint64(0xA5A5A5A5))
    return np.nonzero(h % np.uint64(keep_mod) == 0)[0].astype(np.int64)


def rmat_row_subset(scale: int, edge_factor: int, seed: int, keep_mod: int = 0, ranges=(),
                    threads: int | None = None):
    """Canonical rows of the R-MAT matrix (first-draw dedup, as the GPU
    generator) for the hashed 1/keep_mod row sample (keep_mod 0: none) plus
    every row in the half-open ``ranges``: returns (rows, ptr, ind, dat),
    ``rows`` the ascending global row ids, CSR over them (compressed), all
    columns global."""
    threads = threads or port.host_cores()
    lib = _lib()
    n = 1 << scale
    draws = edge_factor << scale
    rng = np.ascontiguousarray(np.asarray(ranges, dtype=np.int32).reshape(-1, 2))
    span = int((rng[:, 1] - rng[:, 0]).clip(0).sum()) if rng.size else 0
    cap = (int(draws / keep_mod * 1.3) if keep_mod else 0) + (1 << 20)
    while True:
        e = np.empty(cap, np.int64)
        r = np.empty(cap, np.int32)
        c = np.empty(cap, np.int32)
        v = np.empty(cap, np.float64)
        total = lib.rmat_sample_ranges(scale, draws, 0.57, 0.19, 0.19, seed, keep_mod,
                                       rng.ctypes.data if rng.size else None, int(rng.shape[0]), cap,
                                       e.ctypes.data, r.ctypes.data, c.ctypes.data, v.ctypes.data, threads)
        if total <= cap:
            break
        cap = int(total) + 1
    r, c, v = r[:total].astype(np.int64), c[:total].astype(np.int64), v[:total]
    key = (r << scale) | c
    _, first = np.unique(key, return_index=True)  # draws ascend: index = first draw
    r, c, v = r[first], c[first], v[first]
    parts = [kept_rows(n, keep_mod)] if keep_mod else []
    parts += [np.arange(lo, hi, dtype=np.int64) for lo, hi in rng]
    rows = np.unique(np.concatenate(parts)) if parts else np.empty(0, np.int64)
    local = np.searchsorted(rows, r)
    lr, lc, lv = port.canonicalize(local, c, v, rows.size, n)
    ptr, ind, dat = port.to_csr(lr, lc, lv, rows.size)
    return rows, ptr, ind, dat


def rmat_row_sample(scale: int, edge_factor: int, seed: int, keep_mod: int, threads: int | None = None):
    """CSR (ptr, indices, data) of the sampled rows (compressed), n_cols = 2^scale."""
    rows, ptr, ind, dat = rmat_row_subset(scale, edge_factor, seed, keep_mod, (), threads)
    return ptr, ind, dat, rows.size, 1 << scale


def time_csr(ptr, ind, dat, n_rows, x, workers: int, min_seconds: float = 8.0, min_reps: int = 3,
             max_reps: int = 200):
    """Mean seconds per SpMV of the reference CPU algorithm."""
    port.spmv_csr(ptr, ind, dat, n_rows, x, workers)  # warm-up (pool start, page-in)
    times = []
    t_end = time.perf_counter() + min_seconds
    while len(times) < min_reps or (time.perf_counter() < t_end and len(times) < max_reps):
        t0 = time.perf_counter()
        port.spmv_csr(ptr, ind, dat, n_rows, x, workers)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), len(times)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return os.uname().machine
