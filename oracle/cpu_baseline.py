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
    lib.rmat_sample.restype = ctypes.c_int64
    lib.rmat_sample.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    return lib


def kept_rows(n: int, keep_mod: int) -> np.ndarray:
    r = np.arange(n, dtype=np.uint64)
    h = synth_ref.mix64(r ^ np.uint64(0xA5A5A5A5))
    return np.nonzero(h % np.uint64(keep_mod) == 0)[0].astype(np.int64)


def rmat_row_sample(scale: int, edge_factor: int, seed: int, keep_mod: int, threads: int | None = None):
    """CSR (ptr, indices, data) of the sampled rows (compressed), n_cols = 2^scale."""
    threads = threads or port.host_cores()
    lib = _lib()
    draws = edge_factor << scale
    cap = int(draws / keep_mod * 1.3) + (1 << 20)
    while True:
        e = np.empty(cap, np.int64)
        r = np.empty(cap, np.int32)
        c = np.empty(cap, np.int32)
        v = np.empty(cap, np.float64)
        total = lib.rmat_sample(scale, draws, 0.57, 0.19, 0.19, seed, keep_mod, cap, e.ctypes.data, r.ctypes.data,
                                c.ctypes.data, v.ctypes.data, threads)
        if total <= cap:
            break
        cap = int(total) + 1
    r, c, v = r[:total].astype(np.int64), c[:total].astype(np.int64), v[:total]
    key = (r << scale) | c
    _, first = np.unique(key, return_index=True)  # draws ascend: index = first draw
    r, c, v = r[first], c[first], v[first]
    rows = kept_rows(1 << scale, keep_mod)
    local = np.searchsorted(rows, r)
    n_s = rows.size
    lr, lc, lv = port.canonicalize(local, c, v, n_s, 1 << scale)
    ptr, ind, dat = port.to_csr(lr, lc, lv, n_s)
    return ptr, ind, dat, n_s, 1 << scale


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
