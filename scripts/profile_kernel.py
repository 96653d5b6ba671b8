"""Run one format's SpMV a few times on a benchmark config (for ncu).

    python scripts/profile_kernel.py --workload C4 --format csr5 --reps 5
    python scripts/profile_kernel.py --workload C4 --format sell --relabel --shard 0/8

--relabel runs the bench's shadow layout (degree order; SELL-32 sigma 0,
CSR5 sigma 8); --shard p/P takes rank p's dealt row block of P.

Builds the matrix exactly as bench.py does, converts it with the bench's
tuned parameters, runs 2 warm-up SpMVs and `--reps` timed ones; under ncu
select the kernel with -k regex:... and skip the warm-ups with -s.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

PARAMS = {
    "csr": {},
    "csr5": dict(omega=32, sigma=16),
    "hyb": dict(max_cells=1 << 34),
    "sell": dict(sell_c=32, sell_sigma=32 * 256, max_cells=1 << 34),
    "ell": dict(max_cells=1 << 34),
}


def build(workload: str):
    if workload in ("C1", "C2", "C3"):
        return sp.synth.host_coo(workload)
    cfg = synth.CONFIGS[workload]
    return synth.rmat_coo(cfg["scale"], cfg["edge_factor"], cfg["seed"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--format", default="csr")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--relabel", action="store_true")
    ap.add_argument("--shard", default="0/1")
    args = ap.parse_args()
    a = build(args.workload)
    x = synth.uniform_vector(a.n_cols, 7)
    params = dict(PARAMS[args.format])
    if args.relabel:
        from paper_1805_11938_b200 import dist as spdist
        from paper_1805_11938_b200.relabel import DegreeOrder

        p, parts = (int(v) for v in args.shard.split("/"))
        csr = sp.to_csr(a)
        order = DegreeOrder(csr, parts=parts)
        a = order.matrix(csr)
        x = order.to_new(x)
        if parts > 1:
            a = spdist.row_block(a, order.part_bounds[p], order.part_bounds[p + 1])
        del csr
        params.update({"sell": dict(sell_c=32, sell_sigma=0, max_cells=1 << 34),
                       "csr5": dict(omega=32, sigma=8)}.get(args.format, {}))
    m = sp.convert(args.format, a, **params)
    y = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    for _ in range(2 + args.reps):
        sp.spmv(args.format, m, x, out=y)
    torch.cuda.synchronize()
    print(f"{args.workload} {args.format} nnz={a.nnz} bytes_model={sp.spmv_bytes(args.format, m)}")


if __name__ == "__main__":
    main()
