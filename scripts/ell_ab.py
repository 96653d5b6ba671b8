"""ELL SpMV timing (C1-C3, L2-flushed medians, and hot) for same-box A/B
builds (SPMVB_LIB_PATH).  Prints time and a hash of y."""

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


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    lib = Path(os.environ.get("SPMVB_LIB_PATH", "default")).stem
    for cfg in ("C1", "C2", "C3"):
        w = bench.WORKLOADS[cfg]
        a = bench.build_workload(sp, synth, w, dev)
        m = sp.to_ell(a)
        x = synth.uniform_vector(a.n_cols, w["x_seed"], device=dev)
        y = torch.empty(a.n_rows, dtype=torch.float64, device=dev)
        fn = lambda: sp.spmv("ell", m, x, out=y)  # noqa: E731
        for _ in range(3):
            fn()
        fl = []
        for _ in range(3):
            evs = []
            for _ in range(15):
                flush.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            fl.append(statistics.median(e0.elapsed_time(e1) for e0, e1 in evs) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        e1.synchronize()
        hot = e0.elapsed_time(e1) / 50 * 1e3
        h = hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"{lib:8s} {cfg} ell k={m.k}: flushed {min(fl):7.2f} us (rounds {', '.join(f'{t:.2f}' for t in fl)})  "
              f"hot {hot:7.2f} us  y#{h}", flush=True)
        del a, m, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
