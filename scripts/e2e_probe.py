"""Break the host-buffer SpMV call (bench.py's e2e leg) into its parts on one GPU."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

scale, ef = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (25, 16)
dev = torch.device("cuda", 0)
r, c, v = synth.rmat_triplets(scale, ef, 105, dev)
n = 1 << scale
a = sp.canonicalize(r, c, v, n, n)
del r, c, v
m = sp.to_csr5(sp.to_csr(a), omega=32, sigma=16)
del a
x = synth.uniform_vector(n, 7, device=dev)
xh = x.cpu().pin_memory()
y = torch.empty(n, dtype=torch.float64, device=dev)
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()


def timed(label, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms", flush=True)


timed("h2d pinned 8n", lambda: x.copy_(xh, non_blocking=True))
timed("d2h pinned 8n", lambda: yh.copy_(y, non_blocking=True))
timed("kernel (device x, out=)", lambda: sp.spmv("csr5", m, x, out=y))
timed("alloc pinned 8n", lambda: torch.empty(n, dtype=torch.float64, pin_memory=True))
timed("alloc pageable 8n", lambda: torch.empty(n, dtype=torch.float64))
timed("spmv(host pinned x)", lambda: sp.spmv("csr5", m, xh))
hold = []
timed("spmv(host pinned x) kept", lambda: hold.append(sp.spmv("csr5", m, xh)) or (len(hold) > 2 and hold.pop(0)))
timed("spmv(host x, out=host y) ranges=8", lambda: sp.spmv("csr5", m, xh, out=yh))
for k in (1, 2, 4, 16, 32):
    timed(f"spmv_csr5(host x, out=host y) ranges={k}", lambda: sp.spmv_csr5(m, xh, out=yh, ranges=k))
