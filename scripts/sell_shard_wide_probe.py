"""SELL-32 on one dealt C5 shard (DegreeOrder(parts=P), shard 0) with the
wide-slice threshold forced to 256..4096: which threshold a 1/P-size shard
wants (the size heuristic picks 512 at P = 8).

    python scripts/sell_shard_wide_probe.py > profiles/r02_sell_shard_wide_probe.txt
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
from paper_1805_11938_b200.formats import SellMatrix  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    w = bench.WORKLOADS["C5"]
    csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
    x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
    auto = SellMatrix.wide_cols
    for P in (2, 4, 8):
        o = DegreeOrder(csr, parts=P)
        mat, xs = o.matrix(csr), o.to_new(x)
        shard = spdist.row_block(mat, o.part_bounds[0], o.part_bounds[1])
        for wc in (None, 256, 512, 1024, 2048, 4096):
            SellMatrix.wide_cols = auto if wc is None else (lambda self, wc=wc: wc)
            m = sp.to_sell(shard, 32, 0, max_cells=1 << 34)
            y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
            for _ in range(3):
                sp.spmv("sell", m, xs, out=y)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                sp.spmv("sell", m, xs, out=y)
            b.record()
            b.synchronize()
            print(f"P={P} shard 0 ({shard.nnz} nnz): wide_cols {m.wide_plan()[5]:5d}{' (auto)' if wc is None else ''}: "
                  f"{a.elapsed_time(b) / 20 * 1e3:8.1f} us", flush=True)
            del m, y
        SellMatrix.wide_cols = auto
        del o, mat, xs, shard
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
