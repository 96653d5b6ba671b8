"""CSR5 SpMV timing for same-box A/B of library builds (SPMVB_LIB_PATH):
omega 32 with sigma 8 and 16 on the degree-ordered C4 (L2-flushed, as the
configs block) and C5 (hot).  Prints time and a hash of y.

    for v in ab_libs/*.so; do SPMVB_LIB_PATH=$v python scripts/csr5_ab.py; done
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
    for cfg in ("C4", "C5"):
        w = bench.WORKLOADS[cfg]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        order = DegreeOrder(csr)
        csr, x = order.matrix(csr), order.to_new(x)
        for sigma in tuple(int(v) for v in os.environ.get("CSR5_AB_SIGMAS", "8,16").split(",")):
            m = sp.to_csr5(csr, 32, sigma)
            y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
            fn = lambda: sp.spmv("csr5", m, x, out=y)  # noqa: E731
            for _ in range(3):
                fn()
            times = []
            for _ in range(3):
                if cfg == "C5":
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
            hsh = hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:12]
            print(f"{lib:8s} {cfg} csr5 w32 s{sigma} relabelled: {min(times):8.1f} us "
                  f"(rounds {', '.join(f'{t:.1f}' for t in times)})  {2 * csr.nnz / min(times) / 1e3:6.1f} GFLOP/s "
                  f"y#{hsh}", flush=True)
            del m, y
        del csr, x, order
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
