"""Per-shard view of the C5 row-block partition on ONE GPU: for P in
(1, 2, 4, 8) every nnz-balanced shard is converted and its local SpMV timed
(CUDA events, one shard at a time), and the x exchange volume of the
all-gatherv and of the sparse exchange is counted.  The multi-GPU step is
bounded below by max over shards of (local SpMV + exchange); this measures
the compute side and the bytes the exchange must move.  JSON lines on stdout."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402
from paper_1805_11938_b200.dist import GpuOps  # noqa: E402


def event_ms(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    scale, ef = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (25, 16)
    dev = torch.device("cuda", 0)
    r, c, v = synth.rmat_triplets(scale, ef, 105, dev)
    n = 1 << scale
    a = sp.canonicalize(r, c, v, n, n)
    del r, c, v
    csr = sp.to_csr(a)
    del a
    x = synth.uniform_vector(n, 7, device=dev)
    balance = sys.argv[3] if len(sys.argv) > 3 else "nnz"
    for P in (1, 2, 4, 8):
        bounds = (spdist.cost_balanced_bounds(csr.ptr, P) if balance == "cost"
                  else spdist.nnz_balanced_bounds(csr.ptr, P))
        for p in range(P):
            lo, hi = int(bounds[p]), int(bounds[p + 1])
            shard = spdist.row_block(csr, lo, hi) if P > 1 else csr
            rec = {"P": P, "shard": p, "balance": balance, "rows": hi - lo, "nnz": shard.nnz}
            best = None
            for tag, kw in (("csr5", dict(omega=32, sigma=16)),):
                m = sp.convert(tag, shard, **kw)
                y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
                ms = event_ms(lambda: sp.spmv(tag, m, x, out=y))
                rec[f"{tag}_ms"] = ms
                if best is None or ms < best[1]:
                    best = (tag, ms)
                del m, y
            rec["best"], rec["best_ms"] = best
            rec["gflops"] = 2.0 * shard.nnz / best[1] / 1e6
            cols = GpuOps.column_set(shard.indices, n)
            remote = int(cols.numel()) - int(((cols >= lo) & (cols < hi)).sum().item())
            rec["distinct_cols"] = int(cols.numel())
            rec["sparse_recv_entries"] = remote
            rec["allgatherv_recv_entries"] = n - (hi - lo)
            print(json.dumps(rec), flush=True)
            del shard, cols
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
