"""Matrix Market text I/O throughput on this host: the native
multithreaded formatter (write_matrix_market) and tokenizer
(read_matrix_market's entry parser) against the reference's pure-Python
expressions, on a C4-sized triplet list.  No GPU work is timed.

    python scripts/mm_io_bench.py [--nnz 20000000]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1805_11938_b200 import coo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", type=int, default=20_000_000)
    ap.add_argument("--py-sample", type=int, default=1_000_000)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    n = 1 << 21
    r = np.sort(rng.integers(0, n, args.nnz))
    c = rng.integers(0, n, args.nnz)
    v = rng.uniform(0.0, 1.0, args.nnz)
    best_w = best_r = 1e9
    for _ in range(3):
        t = time.perf_counter()
        body = coo._format_entries(r, c, v)
        best_w = min(best_w, time.perf_counter() - t)
    raw = f"%%MatrixMarket matrix coordinate real general\n{n} {n} {args.nnz}\n".encode() + bytes(body)
    for _ in range(3):
        t = time.perf_counter()
        out = coo._fast_triplets(raw)
        best_r = min(best_r, time.perf_counter() - t)
    assert np.array_equal(out[0], r) and np.array_equal(out[1], c) and out[2].tobytes() == v.tobytes()
    k = args.py_sample
    t = time.perf_counter()
    text = "".join(f"{i + 1} {j + 1} {x:.17g}\n" for i, j, x in zip(r[:k].tolist(), c[:k].tolist(), v[:k].tolist()))
    t_pw = time.perf_counter() - t
    head = f"%%MatrixMarket matrix coordinate real general\n{n} {n} {k}\n"
    t = time.perf_counter()
    coo._parse_text_triplets(head + text)
    t_pr = time.perf_counter() - t
    mb = len(raw) / 1e6
    print(f"host threads {os.cpu_count()}, {args.nnz} entries, {mb:.0f} MB of text")
    print(f"native write : {best_w:.3f} s  {args.nnz / best_w / 1e6:7.1f} M entries/s  {mb / best_w:7.0f} MB/s")
    print(f"native read  : {best_r:.3f} s  {args.nnz / best_r / 1e6:7.1f} M entries/s  {mb / best_r:7.0f} MB/s")
    print(f"python write : {k / t_pw / 1e6:7.2f} M entries/s (the reference's expression, {k} entries)"
          f"  -> native x{(args.nnz / best_w) / (k / t_pw):.0f}")
    print(f"python read  : {k / t_pr / 1e6:7.2f} M entries/s (the reference-semantics parser, {k} entries)"
          f"  -> native x{(args.nnz / best_r) / (k / t_pr):.0f}")


if __name__ == "__main__":
    main()
