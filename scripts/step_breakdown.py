"""Where a C5 power-iteration step's time goes, measured the way bench.py
measures it (sustained load, CUDA events): blocks of K back-to-back SpMVs
on the same x -> y, of K ping-pong SpMVs (x -> y -> x ...), of K fused
norms, and of K full steps (PowerIteration fast path), interleaved after a
2 s warm-up so all see the same (power-capped) clocks.  Layout and format
as the headline: degree-ordered C5, SELL-32 sigma 0 (or argv[1] = csr5).

    python scripts/step_breakdown.py [sell|csr5] > profiles/r02_step_breakdown.txt
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402

K = 40
fmt = sys.argv[1] if len(sys.argv) > 1 else "sell"
kw = dict(sell_c=32, sell_sigma=0, max_cells=1 << 34) if fmt == "sell" else dict(omega=32, sigma=16)
dev = torch.device("cuda", 0)
w = bench.WORKLOADS["C5"]
csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
order = DegreeOrder(csr)
shadow = order.matrix(csr)
x0 = order.to_new(synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev))
del csr
m = sp.convert(fmt, shadow, **kw)
del shadow
torch.cuda.empty_cache()
n = m.n_rows
op = sp.SpmvOperator(fmt, m)
pi = spdist.PowerIteration(op, [0, n], 0, 1, dev, x0)
y = torch.empty(n, dtype=torch.float64, device=dev)
xa, xb = x0.clone(), torch.empty_like(x0)
s = torch.ones(1, dtype=torch.float64, device=dev)
ss = torch.empty(1, dtype=torch.float64, device=dev)
same = sp.bind(fmt, m, xa, y, s)
ping, pong = sp.bind(fmt, m, xa, xb, s), sp.bind(fmt, m, xb, xa, s)
norm = spdist.GpuOps.bind_norm_scale(y, ss, s)


def block(fn, k=K):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def pingpong():
    ping()
    pong()


t_end = time.time() + 2.0
while time.time() < t_end:
    pi.step()
res = {"spmv x->y": [], "spmv ping-pong": [], "norm (fused)": [], "step": []}
for _ in range(4):
    res["spmv x->y"].append(block(same))
    res["spmv ping-pong"].append(block(pingpong, K // 2) / 2)
    res["norm (fused)"].append(block(norm))
    res["step"].append(block(pi.step))
print(f"C5 degree-ordered, {fmt} {kw}")
for k, v in res.items():
    print(f"{k:15s} ms per call: {' '.join(f'{t:.3f}' for t in v)}", flush=True)
