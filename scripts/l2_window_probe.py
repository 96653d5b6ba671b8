"""L2 persisting window over the hot head of x on the degree-ordered C5
(the round-1 probe was on the reference layout, where the hot columns are
scattered): SELL-32 sigma 0 SpMV time with a persisting access-policy window
of W MB at the start of x' (the highest-degree columns), W = 0 / 16 / 32 /
48 / 64, set on the launching stream through cuda-python.

    python scripts/l2_window_probe.py > profiles/r02_l2_window_probe.txt
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402


def set_window(stream, base, nbytes):
    err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, nbytes)
    attr = rt.cudaStreamAttrValue()
    w = attr.accessPolicyWindow
    w.base_ptr = base
    w.num_bytes = nbytes
    w.hitRatio = 1.0 if nbytes else 0.0
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting if nbytes else rt.cudaAccessProperty.cudaAccessPropertyNormal
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    err2, = rt.cudaStreamSetAttribute(stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr)
    rt.cudaCtxResetPersistingL2Cache()
    return err, err2


def main():
    dev = torch.device("cuda", 0)
    w = bench.WORKLOADS["C5"]
    csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
    order = DegreeOrder(csr)
    xp = order.to_new(synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev))
    m = sp.convert("sell", order.matrix(csr), sell_c=32, sell_sigma=0, max_cells=1 << 34)
    del csr
    y = torch.empty(m.n_rows, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for rnd in range(2):
        for mb in (0, 16, 32, 48, 64, 0):
            errs = set_window(stream, xp.data_ptr(), mb << 20)
            for _ in range(5):
                sp.spmv("sell", m, xp, out=y)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                sp.spmv("sell", m, xp, out=y)
            b.record()
            b.synchronize()
            print(f"round {rnd} window {mb:3d} MB: {a.elapsed_time(b) / 20 * 1e3:8.1f} us  (status {errs})", flush=True)
    set_window(stream, 0, 0)


if __name__ == "__main__":
    main()
