"""What a one-wave, L2-flushed launch costs on this GPU, timed exactly as
bench.py times C1 (512 MB flush, then CUDA events around one launch): a
2 MB fill, a 20 MB torch sum (C1's bytes in one stream), a 2 MB copy, and
the C1 ELL SpMV (20 MB model bytes), so C1's roofline fraction can be read
against the launch + DRAM-latency floor rather than the streaming peak.

    python scripts/c1_floor_probe.py > profiles/r02_c1_floor_probe.txt
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


def flushed(fn, flush, reps=30):
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
    return statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    w = bench.WORKLOADS["C1"]
    csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
    x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
    m = sp.to_ell(csr)
    y = torch.empty(csr.n_rows, dtype=torch.float64, device=dev)
    buf = torch.rand(int(sp.spmv_bytes("ell", m)) // 8, dtype=torch.float64, device=dev)
    res = {
        "fill y (2 MB write)": flushed(lambda: y.fill_(1.0), flush),
        "copy x -> y (2 MB + 2 MB)": flushed(lambda: y.copy_(x), flush),
        f"torch sum over {buf.numel() * 8 / 1e6:.1f} MB": flushed(lambda: buf.sum(), flush),
        f"ELL SpMV C1 ({sp.spmv_bytes('ell', m) / 1e6:.1f} MB model)": flushed(lambda: sp.spmv("ell", m, x, out=y),
                                                                              flush),
    }
    for k, v in res.items():
        print(f"{k:40s} {v:7.2f} us (median of 30, L2 flushed)", flush=True)


if __name__ == "__main__":
    main()
