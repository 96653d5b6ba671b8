"""Cost of the fused SpMV + peer push on one GPU: CSR5 SpMV of a workload
plain vs spmv_csr5_push into P local stand-in "peer" buffers (the stores go
to local HBM here, over NVLink in a multi-GPU run).
    python scripts/time_push.py [--workload C5] [--peers 1,3,7]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from scripts.profile_kernel import build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C5")
ap.add_argument("--peers", default="1,3,7")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
m = sp.to_csr5(sp.to_csr(build(a.workload)), 32, 16)
x = synth.uniform_vector(m.n_cols, 7, device=torch.device("cuda"))
y = torch.empty(m.n_rows, dtype=torch.float64, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


base = timed(lambda: sp.spmv("csr5", m, x, out=y))
print(f"{a.workload} plain CSR5 SpMV: {base * 1e3:.1f} us", flush=True)
for p in [int(v) for v in a.peers.split(",")]:
    bufs = [torch.empty(m.n_rows + 1, dtype=torch.float64, device="cuda") for _ in range(p)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    t = timed(lambda: sp.spmv_csr5_push(m, x, y, ptrs, 1))
    print(f"{a.workload} fused SpMV + push to {p} local buffers ({p * m.n_rows * 8 / 1e6:.0f} MB): "
          f"{t * 1e3:.1f} us (+{(t - base) * 1e3:.1f})", flush=True)
    del bufs
