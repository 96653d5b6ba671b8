"""Where a C5 power-iteration step's time goes, measured the way bench.py
measures it (sustained load, CUDA events): blocks of K back-to-back SpMVs
(with the device scale), of K sumsq+inv_sqrt, and of K full steps,
interleaved after a warm-up so all see the same (power-capped) clocks."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402
from scripts.profile_kernel import build  # noqa: E402

K = 50
m = sp.to_csr5(sp.to_csr(build("C5")), 32, 16)
n = m.n_rows
dev = torch.device("cuda", 0)
x0 = synth.uniform_vector(n, 205, device=dev)


def local(xv, out, scale):
    sp.spmv("csr5", m, xv, out=out, scale=scale)


pi = spdist.PowerIteration(local, [0, n], 0, 1, dev, x0)
y = torch.empty(n, dtype=torch.float64, device=dev)


def block(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


t_end = time.time() + 2.0
while time.time() < t_end:
    pi.step()
res = {"spmv": [], "norm": [], "step": [], "spmv_noscale": []}
for _ in range(4):
    res["spmv"].append(block(lambda: sp.spmv("csr5", m, pi.x, out=y, scale=pi.scale)))
    res["spmv_noscale"].append(block(lambda: sp.spmv("csr5", m, pi.x, out=y)))
    res["norm"].append(block(lambda: (pi.ops.sumsq(y, pi.sumsq), pi.ops.inv_sqrt(pi.sumsq, pi.scale))))
    res["step"].append(block(pi.step))
for k, v in res.items():
    print(f"{k:13s} ms per call: {' '.join(f'{t:.3f}' for t in v)}", flush=True)
