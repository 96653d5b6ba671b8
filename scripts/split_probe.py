"""Head/tail split of the degree-ordered matrix: the R_T rows in SELL
slices wider than T (the long rows, a prefix of the degree order) as CSR5
omega 32 sigma 8, whose lanes walk consecutive entries of a row (sorted
columns: neighbouring lanes share x lines), and the remaining rows as
SELL-32 sigma 0 (lane per row).  Times each part alone and both back to back
(CUDA events, hot, 20 reps) against SELL and CSR5 on the whole matrix, for
C4, C5 and C5's dealt 8-way shard 0.

    python scripts/split_probe.py > profiles/r02_split_probe.txt
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

SELL = dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)


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
    return a.elapsed_time(b) / reps * 1e3


def probe(name, csr, x):
    n = csr.n_rows
    y = torch.empty(n, dtype=torch.float64, device=x.device)
    whole_sell = sp.convert("sell", csr, **SELL)
    t_sell = hot(lambda: sp.spmv("sell", whole_sell, x, out=y))
    ref = y.clone()
    deg = torch.diff(csr.ptr)
    del whole_sell
    whole_c5 = sp.to_csr5(csr, 32, 8)
    t_c5 = hot(lambda: sp.spmv("csr5", whole_c5, x, out=y))
    del whole_c5
    torch.cuda.empty_cache()
    print(f"{name}: SELL-32 s0 whole {t_sell:8.1f} us   CSR5 w32 s8 whole {t_c5:8.1f} us", flush=True)
    for T in (64, 128, 256, 1024, 4096):
        # rows in slices wider than T: the slice width is its first row's degree (sorted)
        first = deg[::32]
        n_wide_sl = int((first > T).sum().item())
        r_w = min(n_wide_sl * 32, n)
        if r_w == 0 or r_w == n:
            continue
        head = sp.to_csr5(spdist.row_block(csr, 0, r_w), 32, 8)
        tail = sp.convert("sell", spdist.row_block(csr, r_w, n), **SELL)
        yh, yt = y[:r_w], y[r_w:]
        t_h = hot(lambda: sp.spmv("csr5", head, x, out=yh))
        t_t = hot(lambda: sp.spmv("sell", tail, x, out=yt))

        def both():
            sp.spmv("csr5", head, x, out=yh)
            sp.spmv("sell", tail, x, out=yt)

        t_b = hot(both)
        err = float(((y - ref).abs().max() / ref.abs().max()).item())
        print(f"  T {T:5d}: head rows {r_w:9d} nnz {head.nnz:10d} CSR5 {t_h:8.1f} us | tail nnz {tail.nnz:10d} "
              f"SELL {t_t:8.1f} us | both {t_b:8.1f} us  (max rel diff vs SELL {err:.1e})", flush=True)
        del head, tail
        torch.cuda.empty_cache()


def main():
    dev = torch.device("cuda", 0)
    for wl in ("C4", "C5"):
        w = bench.WORKLOADS[wl]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        order = DegreeOrder(csr)
        probe(f"{wl} whole", order.matrix(csr), order.to_new(x))
        del order
        torch.cuda.empty_cache()
        if wl == "C5":
            o = DegreeOrder(csr, parts=8)
            mat = o.matrix(csr)
            shard = spdist.row_block(mat, 0, o.part_bounds[1])
            del mat
            probe(f"{wl} dealt shard 0/8", shard, o.to_new(x))
            del shard, o
        del csr, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
