"""Compute-side balance of the C5 row blocks on one GPU: every shard of a
P-way partition converted and timed alone (full-length x, CUDA events, hot,
20 reps), for the degree-ordered matrix cut into nnz-balanced blocks and
for the dealt order (DegreeOrder(parts=P): degree-sorted rows dealt
round-robin to the blocks).  efficiency = T(whole) / (P * slowest shard):
the best a P-GPU step can do before any exchange.

    python scripts/shard_balance.py [sell|csr5] > profiles/r02_shard_balance.txt
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402

FMT = sys.argv[1] if len(sys.argv) > 1 else "sell"
KW = dict(sell_c=32, sell_sigma=0, max_cells=1 << 34) if FMT == "sell" else dict(omega=32, sigma=8)


def hot(m, x, reps=20):
    y = torch.empty(m.n_rows, dtype=torch.float64, device=x.device)
    for _ in range(3):
        sp.spmv(FMT, m, x, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sp.spmv(FMT, m, x, out=y)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    w = bench.WORKLOADS["C5"]
    csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
    x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
    order = DegreeOrder(csr)
    whole = order.matrix(csr)
    t1 = hot(sp.convert(FMT, whole, **KW), order.to_new(x))
    print(f"C5 {FMT} {KW}: whole degree-ordered matrix {t1:.3f} ms", flush=True)
    torch.cuda.empty_cache()
    for P in (2, 4, 8):
        for scheme in ("nnz-balanced blocks", "dealt"):
            if scheme == "dealt":
                o = DegreeOrder(csr, parts=P)
                mat, xs, bounds = o.matrix(csr), o.to_new(x), o.part_bounds
            else:
                mat, xs = whole, order.to_new(x)
                bounds = [int(b) for b in spdist.nnz_balanced_bounds(mat.ptr, P)]
            times, nnzs = [], []
            for p in range(P):
                shard = spdist.row_block(mat, bounds[p], bounds[p + 1])
                times.append(hot(sp.convert(FMT, shard, **KW), xs))
                nnzs.append(shard.nnz)
                del shard
                torch.cuda.empty_cache()
            eff = t1 / (P * max(times))
            print(f"P={P} {scheme:20s} shard ms {' '.join(f'{t:.3f}' for t in times)}  max {max(times):.3f}  "
                  f"efficiency {eff:.3f}  nnz max/mean {max(nnzs) / (sum(nnzs) / P):.4f}", flush=True)
            if scheme == "dealt":
                del mat, xs, o
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
