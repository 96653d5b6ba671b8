"""Device-synchronised wall time of the non-SpMV public calls on C4/C5:
feature extraction, row histogram, typical K, to_coo round trips,
dense_spmv_oracle.  python scripts/time_api.py [--workloads C4,C5]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402
from scripts.profile_kernel import PARAMS, build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="C4,C5")
a = ap.parse_args()


def t(name, w, fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{w} {name:28s} ms {min(ts):9.2f}", flush=True)


for w in a.workloads.split(","):
    coo = build(w)
    csr = sp.to_csr(coo)
    x = synth.uniform_vector(csr.n_cols, 7, device=torch.device("cuda"))
    t("extract_features(coo)", w, lambda: sp.extract_features(coo))
    t("extract_features(csr)", w, lambda: sp.extract_features(csr))
    t("extract_extra_features", w, lambda: sp.extract_extra_features(csr))
    t("row_nnz_histogram", w, lambda: sp.row_nnz_histogram(coo))
    t("dense_spmv_oracle", w, lambda: sp.dense_spmv_oracle(coo, x))
    for f in ("csr", "csr5", "hyb", "sell"):
        m = sp.convert(f, csr, **PARAMS[f])
        t(f"to_coo({f})", w, lambda: sp.to_coo(m), reps=2)
        del m
    del coo, csr, x
    torch.cuda.empty_cache()
