"""Run one format's SpMV a few times on a benchmark config (for ncu).

    python scripts/profile_kernel.py --workload C4 --format csr5 --reps 5

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
    args = ap.parse_args()
    a = build(args.workload)
    m = sp.convert(args.format, a, **PARAMS[args.format])
    x = synth.uniform_vector(a.n_cols, 7)
    y = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    for _ in range(2 + args.reps):
        sp.spmv(args.format, m, x, out=y)
    torch.cuda.synchronize()
    print(f"{args.workload} {args.format} nnz={a.nnz} bytes_model={sp.spmv_bytes(args.format, m)}")


if __name__ == "__main__":
    main()
