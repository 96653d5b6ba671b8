"""SELL SpMV timing for same-box A/B of library builds (SPMVB_LIB_PATH):
SELL-32 sigma 0 on the degree-ordered C5 (the power-iteration format
there), its dealt 8-way shard 0 and C4, and SELL-32 sigma 1024 on C3.  Prints time and a hash of y
(variants must agree bit for bit).

    for v in ab_libs/*.so; do SPMVB_LIB_PATH=$v python scripts/sell_ab.py; done
"""

from __future__ import annotations

import hashlib
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    lib = Path(os.environ.get("SPMVB_LIB_PATH", "default")).stem
    for cfg, relabel, kw in (("C5", True, dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),
                             ("C5/8", True, dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),
                             ("C4", True, dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),
                             ("C3", False, dict(sell_c=32, sell_sigma=1024, max_cells=1 << 34))):
        w = bench.WORKLOADS[cfg.split("/")[0]]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        if relabel:
            parts = int(cfg.split("/")[1]) if "/" in cfg else 1
            order = DegreeOrder(csr, key="row", parts=parts)
            csr, x = order.matrix(csr), order.to_new(x)
            if parts > 1:
                from paper_1805_11938_b200 import dist as spdist

                csr = spdist.row_block(csr, 0, order.part_bounds[1])
        m = sp.convert("sell", csr, **kw)
        y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
        fn = lambda: sp.spmv("sell", m, x, out=y)  # noqa: E731
        for _ in range(3):
            fn()
        times = []
        for _ in range(3):  # three rounds of 20 back-to-back (hot) or 10 flushed reps
            if cfg.startswith("C5"):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    fn()
                b.record()
                b.synchronize()
                times.append(a.elapsed_time(b) / 20 * 1e3)
            else:
                evs = []
                for _ in range(10):
                    flush.sum()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    b.record()
                    evs.append((a, b))
                torch.cuda.synchronize()
                times.append(statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3)
        h = hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"{lib:8s} {cfg} sell {kw['sell_c']}/{kw['sell_sigma']}{' relabelled' if relabel else ''}: "
              f"{min(times):8.1f} us (rounds {', '.join(f'{t:.1f}' for t in times)})  "
              f"{2 * csr.nnz / min(times) / 1e3:6.1f} GFLOP/s  y#{h}", flush=True)
        del m, y, csr, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
