"""Hot SpMV time per (workload, format) in one process, one line each.

    SPMVB_LIB_PATH=build_ab/libspmvb_HEAD.so python scripts/time_formats.py --workloads C4,C5 --formats csr,csr5

Used for same-box A/B runs between library builds (scripts/ab_lib.sh).
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from scripts.profile_kernel import PARAMS, build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C4")
    ap.add_argument("--formats", default="csr5")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    tag = Path(os.environ.get("SPMVB_LIB_PATH", "working-tree")).name
    for w in a.workloads.split(","):
        coo = build(w)
        csr = sp.to_csr(coo)
        del coo
        x = synth.uniform_vector(csr.n_cols, 7, device=dev)
        y = torch.empty(csr.n_rows, dtype=torch.float64, device=dev)
        for f in a.formats.split(","):
            try:
                m = sp.convert(f, csr, **PARAMS[f])
            except sp.ConversionError:
                continue
            for _ in range(3):
                sp.spmv(f, m, x, out=y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                sp.spmv(f, m, x, out=y)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / a.reps * 1e3
            print(f"{tag:24s} {w} {f:5s} {us:9.1f} us  {2 * m.nnz / us / 1e3:7.1f} GFLOP/s  "
                  f"ysum={float(y.sum()):.17g}", flush=True)
            del m
        del csr, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
