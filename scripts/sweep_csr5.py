"""Time CSR5 (omega, sigma) variants and CSR on C4/C5 (device time, CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

for name in sys.argv[1:] or ["C5"]:
    cfg = synth.CONFIGS[name]
    a = synth.rmat_coo(cfg["scale"], cfg["edge_factor"], cfg["seed"])
    m = sp.to_csr(a)
    del a
    x = synth.uniform_vector(m.n_cols, 5)
    y = torch.empty(m.n_rows, dtype=torch.float64, device="cuda")
    for tag, kw in [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("csr5", dict(omega=32, sigma=8)),
                    ("csr5", dict(omega=16, sigma=16)), ("csr5", dict(omega=8, sigma=16)), ("hyb", {})]:
        mm = sp.convert(tag, m, **kw)
        for _ in range(3):
            sp.spmv(tag, mm, x, out=y)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            sp.spmv(tag, mm, x, out=y)
        e.record()
        e.synchronize()
        t = s.elapsed_time(e) / 20 / 1e3
        print(name, tag, kw, f"{t*1e3:.3f} ms {2*m.nnz/t/1e9:.1f} GF {sp.spmv_bytes(tag, mm)/t/1e9:.0f} GB/s", flush=True)
        del mm
        torch.cuda.empty_cache()
