"""Device-synchronised wall time of the public converters on one workload,
for same-box A/B runs between library builds (SPMVB_LIB_PATH).

    python scripts/time_convert.py --workloads C4,C5 --formats csr5,hyb,sell
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from scripts.profile_kernel import PARAMS, build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="C4,C5")
ap.add_argument("--formats", default="csr5")  # csr5_default: omega=4, sigma=16
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
tag = Path(os.environ.get("SPMVB_LIB_PATH", "working-tree")).name
for w in a.workloads.split(","):
    csr = sp.to_csr(build(w))
    for f in a.formats.split(","):
        ts = []
        for _ in range(a.reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            name, kw = (f, PARAMS[f]) if f in PARAMS else ("csr5", dict(omega=4, sigma=16))
            m = sp.convert(name, csr, **kw)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            del m
        print(f"{tag:22s} {w} to_{f}: ms {' '.join(f'{t:.2f}' for t in ts[1:])}", flush=True)
    del csr
    torch.cuda.empty_cache()
