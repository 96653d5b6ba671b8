"""Power-iteration step time eager vs CUDA graph (one GPU) on the small
configs, where host launch cost is comparable to the SpMV."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402

dev = torch.device("cuda", 0)
for name, tag, kw in [("C1", "ell", {}), ("C2", "ell", {}), ("C3", "ell", {}), ("C3", "csr5", dict(omega=32, sigma=16)),
                      ("C4", "csr5", dict(omega=32, sigma=16))]:
    if name in ("C1", "C2", "C3"):
        a = synth.host_coo(name, dev)
    else:
        cfg = synth.CONFIGS[name]
        a = synth.rmat_coo(cfg["scale"], cfg["edge_factor"], cfg["seed"], dev)
    m = sp.convert(tag, a, **kw)
    x0 = synth.uniform_vector(a.n_cols, 7, device=dev)
    res = {}
    for graph in (False, True):
        pi = spdist.PowerIteration(lambda xv, out, s: sp.spmv(tag, m, xv, out=out, scale=s), [0, a.n_rows], 0, 1,
                                   dev, x0)
        pi.run(10, graph=graph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pi.run(100, graph=graph)
        e1.record()
        torch.cuda.synchronize()
        res[graph] = (e0.elapsed_time(e1) / 100, pi.x.clone())
    same = torch.equal(res[False][1], res[True][1])
    # the default (graph=None): measured choice on the first long run
    pi = spdist.PowerIteration(lambda xv, out, s: sp.spmv(tag, m, xv, out=out, scale=s), [0, a.n_rows], 0, 1,
                               dev, x0)
    pi.run(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pi.run(100)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {tag}: eager {res[False][0] * 1e3:.1f} us/step, graph {res[True][0] * 1e3:.1f} us/step, "
          f"default {e0.elapsed_time(e1) * 10:.1f} us/step (graph chosen: {pi._graph_auto}), "
          f"identical iterates {same}", flush=True)
