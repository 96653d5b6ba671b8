"""Every format on the degree-ordered shadow layout (relabel.py) of C4 and C5:
SpMV time (CUDA events, hot, 20 reps; C4 also L2-flushed), GFLOP/s, the
byte-model fraction of the measured HBM peak, against the reference layout.

    python scripts/relabel_formats.py > profiles/r02_relabel_formats.txt
"""

from __future__ import annotations

import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from paper_1805_11938_b200.harness import spmv_bytes  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402

VARIANTS = [
    ("csr5", dict(omega=32, sigma=16)),
    ("csr5", dict(omega=32, sigma=8)),
    ("sell", dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),
    ("sell", dict(sell_c=32, sell_sigma=32 * 256, max_cells=1 << 34)),
    ("sell", dict(sell_c=16, sell_sigma=0, max_cells=1 << 34)),
]


def hot(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def flushed(fn, flush, reps=10):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs) / 1e3


def main():
    dev = torch.device("cuda", 0)
    peak, _ = bench.measured_peak()
    flush = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    for cfg in ("C4", "C5"):
        w = bench.WORKLOADS[cfg]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        layouts = []
        for key in ("sum", "row"):
            order = DegreeOrder(csr, key=key)
            layouts.append((f"relabel-{key}", order.matrix(csr), order.to_new(x)))
            del order
        for layout, mat, xv in layouts:
            for tag, kw in VARIANTS:
                label = bench.variant_label(tag, kw)
                try:
                    m = sp.convert(tag, mat, **kw)
                except sp.ConversionError as exc:
                    print(f"{cfg} {layout:10s} {label:14s} ConversionError {str(exc)[:60]}", flush=True)
                    continue
                y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
                fn = lambda: sp.spmv(tag, m, xv, out=y)  # noqa: E731
                t = hot(fn)
                b = spmv_bytes(tag, m)
                line = (f"{cfg} {layout:10s} {label:14s} hot {t * 1e6:9.1f} us  {2 * csr.nnz / t / 1e9:7.1f} GFLOP/s  "
                        f"bytes {b / 1e6:9.1f} MB  frac {b / t / 1e9 / peak:5.3f}")
                if cfg == "C4":
                    tf = flushed(fn, flush)
                    line += f"  | flushed {tf * 1e6:8.1f} us {2 * csr.nnz / tf / 1e9:7.1f} GFLOP/s frac {b / tf / 1e9 / peak:5.3f}"
                print(line, flush=True)
                del m, y
                torch.cuda.empty_cache()
        del csr, x, layouts, mat, xv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
