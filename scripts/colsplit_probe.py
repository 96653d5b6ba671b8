"""Column-band split of the degree-ordered matrix: A = A_hot + A_cold with
A_hot the entries in columns [0, H) (the head of the degree order: x[0, H)
is 8 H bytes, an L1-sized window) and A_cold the rest, each its own matrix in
the same row order.  An SM that runs only A_hot keeps x[0, H) resident in L1
(no cold misses evicting it); A_cold's gathers then miss either way.  Times
each part alone (L2-flushed, CUDA events) in CSR5 omega 32 sigma 8 and SELL-32
sigma 0 against the whole matrix in the same format.

    python scripts/colsplit_probe.py [C4 C5] > profiles/r02_colsplit_probe.txt
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
from paper_1805_11938_b200.formats import CsrMatrix  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402

SELL = dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)


def flushed(fn, flush, reps=10):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(reps):
        if flush is not None:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3


def band(csr, keep):
    """The entries of csr selected by the boolean mask, as a CSR of the same shape."""
    cnt = torch.zeros(csr.nnz + 1, dtype=torch.int64, device=csr.device)
    torch.cumsum(keep, 0, out=cnt[1:])
    ptr = cnt[csr.ptr.long()].to(torch.int32)
    return CsrMatrix(csr.n_rows, csr.n_cols, ptr, csr.indices[keep].contiguous(), csr.data[keep].contiguous())


def main():
    dev = torch.device("cuda", 0)
    for wl in (sys.argv[1:] or ["C4", "C5"]):
        w = bench.WORKLOADS[wl]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        order = DegreeOrder(csr)
        csr, x = order.matrix(csr), order.to_new(x)
        del order
        flush = torch.empty(1 << 26, dtype=torch.float64, device=dev) if wl != "C5" else None
        y = torch.empty(csr.n_rows, dtype=torch.float64, device=dev)
        y2 = torch.empty_like(y)

        def fmt(name, m_csr):
            if name == "csr5":
                m = sp.to_csr5(m_csr, 32, 8)
            else:
                m = sp.convert("sell", m_csr, **SELL)
            return m

        for name in ("csr5", "sell"):
            m = fmt(name, csr)
            t_whole = flushed(lambda: sp.spmv(name, m, x, out=y), flush)
            ref = y.clone()
            del m
            torch.cuda.empty_cache()
            print(f"{wl} {name}: whole {t_whole:8.1f} us ({csr.nnz / t_whole / 1e3:6.1f} G entries/s)", flush=True)
            for H in (4096, 8192, 16384, 32768, 65536):
                keep = csr.indices < H
                hot_csr, cold_csr = band(csr, keep), band(csr, ~keep)
                del keep
                mh, mc = fmt(name, hot_csr), fmt(name, cold_csr)
                t_h = flushed(lambda: sp.spmv(name, mh, x, out=y), flush)
                t_c = flushed(lambda: sp.spmv(name, mc, x, out=y2), flush)
                err = float(((y + y2 - ref).abs().max() / ref.abs().max()).item())
                print(f"  H {H:6d}: hot nnz {hot_csr.nnz:10d} ({hot_csr.nnz / csr.nnz:.3f}) {t_h:8.1f} us "
                      f"({hot_csr.nnz / t_h / 1e3:6.1f} G/s) | cold nnz {cold_csr.nnz:10d} {t_c:8.1f} us "
                      f"({cold_csr.nnz / t_c / 1e3:6.1f} G/s) | sum {t_h + t_c:8.1f} us vs whole {t_whole:8.1f} "
                      f"(rel diff {err:.1e})", flush=True)
                del mh, mc, hot_csr, cold_csr
                torch.cuda.empty_cache()
        del csr, x, y, y2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
