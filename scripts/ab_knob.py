"""Interleaved A/B of a per-launch environment knob on one format's SpMV.

    python scripts/ab_knob.py --var SPMVB_CSR5_PF --values 0,2368,4736 --workloads C4,C5 [--format csr5]

The matrix is built once per workload; the knob is read by the library at
every launch, so the values are timed alternately in one process (same box,
same matrix): rounds x values, 30 back-to-back SpMVs each, CUDA events.
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
    ap.add_argument("--var", required=True)
    ap.add_argument("--values", required=True)
    ap.add_argument("--workloads", default="C4,C5")
    ap.add_argument("--format", default="csr5")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--cold", action="store_true", help="read a 512 MB buffer before every rep (L2 flush); median")
    a = ap.parse_args()
    flush = torch.empty(1 << 26, dtype=torch.float64, device="cuda") if a.cold else None
    dev = torch.device("cuda", 0)
    for w in a.workloads.split(","):
        coo = build(w)
        m = sp.convert(a.format, sp.to_csr(coo), **PARAMS[a.format])
        del coo
        x = synth.uniform_vector(m.n_cols, 7, device=dev)
        y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
        ref = None
        res = {v: [] for v in a.values.split(",")}
        for _ in range(a.rounds):
            for v in res:
                os.environ[a.var] = v
                for _ in range(3):
                    sp.spmv(a.format, m, x, out=y)
                torch.cuda.synchronize()
                if flush is not None:
                    evs = []
                    for _ in range(a.reps):
                        flush.sum()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        sp.spmv(a.format, m, x, out=y)
                        e1.record()
                        evs.append((e0, e1))
                    torch.cuda.synchronize()
                    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
                    res[v].append(ts[len(ts) // 2])
                else:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.reps):
                        sp.spmv(a.format, m, x, out=y)
                    e1.record()
                    torch.cuda.synchronize()
                    res[v].append(e0.elapsed_time(e1) / a.reps * 1e3)
                if ref is None:
                    ref = y.clone()
                elif not torch.equal(ref, y):
                    print(f"  {w} {a.var}={v}: y differs from the first value's y", flush=True)
        nnz = m.nnz
        for v, ts in res.items():
            best = min(ts)
            print(f"{w} {a.format}{' cold' if a.cold else ''} {a.var}={v}: us/SpMV {' '.join(f'{t:.1f}' for t in ts)}  best {best:.1f}"
                  f"  {2 * nnz / best / 1e3:.1f} GFLOP/s", flush=True)
        del m, x, y, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
