"""How concentrated the x gathers are on the degree-ordered layout: the
share of stored entries whose column id is below H (the hottest H columns of
x' after DegreeOrder), for C4 and C5, against the ~200 KB (25K doubles) of
L1 each SM has.

    python scripts/hot_columns_probe.py > profiles/r02_hot_columns_probe.txt
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402

HS = [1 << k for k in range(10, 24, 1)]


def main():
    dev = torch.device("cuda", 0)
    for wl in ("C4", "C5"):
        w = bench.WORKLOADS[wl]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        m = DegreeOrder(csr).matrix(csr)
        del csr
        cnt = torch.bincount(m.indices.long(), minlength=m.n_cols)
        cum = torch.cumsum(cnt, 0)
        nnz = int(m.nnz)
        print(f"{wl}: n {m.n_cols} nnz {nnz}")
        for h in HS:
            if h <= m.n_cols:
                print(f"  columns < {h:8d} ({h * 8 / 1024:8.0f} KB of x): {int(cum[h - 1]) / nnz:6.3f} of the entries",
                      flush=True)
        del m, cnt, cum
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
