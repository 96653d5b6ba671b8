"""What a symmetric degree-ordered relabelling P A P^T buys the CSR5 / CSR
SpMV on R-MAT (C4 / C5).  Orderings compared: the original ids; ids sorted
by descending column degree (hot columns contiguous); the same with every
empty row moved last (then the non-empty rows are a prefix and the CSR5
row lookup needs no indirection).  Timed back to back on one box, x larger
or smaller than L2 as the config makes it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
scale, ef, seed = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (25, 16, 105)))
n = 1 << scale
r, c, v = synth.rmat_triplets(scale, ef, seed, dev)
a = sp.canonicalize(r, c, v, n, n)
del r, c, v
degc = torch.bincount(a.col.long(), minlength=n)
degr = torch.bincount(a.row.long(), minlength=n)
x = synth.uniform_vector(n, 7, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
flush = torch.empty(1 << 26, dtype=torch.float64, device=dev) if scale < 24 else None


def t_spmv(tag, m, xv, reps=30):
    for _ in range(3):
        sp.spmv(tag, m, xv, out=y)
    torch.cuda.synchronize()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            sp.spmv(tag, m, xv, out=y)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    ts = []
    for _ in range(reps):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sp.spmv(tag, m, xv, out=y)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ts)
    return ts[len(ts) // 2]


def relabel(key):
    order = torch.argsort(key, stable=True)  # new id -> old id
    new_id = torch.empty_like(order)
    new_id[order] = torch.arange(n, device=dev)
    b = sp.canonicalize(new_id[a.row.long()].int(), new_id[a.col.long()].int(), a.data, n, n)
    return sp.to_csr(b)


variants = {"original": sp.to_csr(a)}
variants["coldeg"] = relabel(-degc)
variants["empty-last+coldeg"] = relabel((degr == 0).long() * (1 << 40) - degc)
variants["empty-last+rowdeg"] = relabel((degr == 0).long() * (1 << 40) - degr)
variants["empty-last+sumdeg"] = relabel((degr == 0).long() * (1 << 40) - degr - degc)
del a
mats = {}
for name, csr in variants.items():
    mats[name] = {"csr5": sp.to_csr5(csr, 32, 16), "csr": csr}
    csr.chunk_plan()
for rnd in range(3):
    for name, ms in mats.items():
        for tag, m in ms.items():
            print(f"scale {scale} round {rnd} {name:20s} {tag:5s} SpMV {t_spmv(tag, m, x):.4f} ms"
                  f"  (n_nonempty {getattr(ms['csr5'], 'n_nonempty', -1)})", flush=True)
