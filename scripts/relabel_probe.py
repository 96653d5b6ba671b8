"""What a degree-ordered relabelling of C5 would buy (an experiment, not a
product path: it changes the stored arrays).  Columns (and, symmetrically,
rows) renumbered by descending column degree; CSR5 SpMV of the original and
the relabelled matrices timed back to back on the same box."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 25
r, c, v = synth.rmat_triplets(25, 16, 105, dev)
a = sp.canonicalize(r, c, v, n, n)
del r, c, v
deg = torch.bincount(a.col.long(), minlength=n)
order = torch.argsort(-deg, stable=True)          # new id -> old id
new_id = torch.empty_like(order)
new_id[order] = torch.arange(n, device=dev)       # old id -> new id
x = synth.uniform_vector(n, 7, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)


def t_spmv(m, xv, reps=30):
    for _ in range(3):
        sp.spmv("csr5", m, xv, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sp.spmv("csr5", m, xv, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


variants = {}
variants["original"] = sp.to_csr5(sp.to_csr(a), 32, 16)
cols = new_id[a.col.long()].int()
b = sp.canonicalize(a.row, cols, a.data, n, n)          # columns relabelled
variants["cols relabelled"] = sp.to_csr5(sp.to_csr(b), 32, 16)
del b
rows = new_id[a.row.long()].int()
b = sp.canonicalize(rows, cols, a.data, n, n)           # symmetric P A P^T
variants["rows+cols relabelled"] = sp.to_csr5(sp.to_csr(b), 32, 16)
del b, a
for rnd in range(3):
    for name, m in variants.items():
        print(f"round {rnd} {name:22s} CSR5 SpMV {t_spmv(m, x):.3f} ms", flush=True)
