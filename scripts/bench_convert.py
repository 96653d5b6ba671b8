"""Conversion throughput on one B200 (device time, CUDA events).

    python scripts/bench_convert.py [--configs C1,C2,C3,C4,C5]

For each config: canonicalize (unsorted input), to_csr and every format
conversion from CSR, with the algorithmic bytes of SURVEY §8(d): one read of
the input and one write of the output (COO->CSR reads 16 B/entry and writes
12 B/nnz + 4(n+1); CSR->X reads 12 nnz + 4(n+1) and writes the X arrays of
the byte model without the x/y terms).
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    args = ap.parse_args()
    for name in args.configs.split(","):
        if name in ("C1", "C2", "C3"):
            cfg = dict(synth.CONFIGS[name])
            kind = cfg.pop("kind")
            r, c, v, n = {"laplace2d": synth.laplace2d, "banded": synth.banded, "stencil27": synth.stencil27}[kind](**cfg)
            perm = np.random.default_rng(0).permutation(r.size)
            r = torch.from_numpy(r[perm].astype(np.int32)).cuda()
            c = torch.from_numpy(c[perm].astype(np.int32)).cuda()
            v = torch.from_numpy(v[perm]).cuda()
        else:
            cfg = synth.CONFIGS[name]
            r, c, v = synth.rmat_triplets(cfg["scale"], cfg["edge_factor"], cfg["seed"])
            n = 1 << cfg["scale"]
        nin = int(r.numel())
        t, a = timed(lambda: sp.canonicalize(r, c, v, n, n))
        rec = {"config": name, "n": n, "nnz_in": nin, "nnz": a.nnz}
        rec["canonicalize"] = {"ms": t * 1e3, "Mentries_per_s": nin / t / 1e6,
                               "GBs_min_bytes": (16 * nin + 16 * a.nnz) / t / 1e9}
        del r, c, v
        t, m = timed(lambda: sp.to_csr(a))
        csr_bytes = 12 * a.nnz + 4 * (n + 1)
        rec["to_csr"] = {"ms": t * 1e3, "GBs_min_bytes": (16 * a.nnz + csr_bytes) / t / 1e9}
        for tag, kw in [("csr5", dict(omega=32, sigma=16)), ("csr5", dict(omega=4, sigma=16)), ("ell", {}),
                        ("sell", dict(sell_c=32, sell_sigma=1024, max_cells=1 << 34)), ("sell", dict(sell_c=4)),
                        ("hyb", {})]:
            key = tag + "".join(f"_{v}" for k, v in kw.items() if k != "max_cells")
            try:
                t, mm = timed(lambda: sp.convert(tag, m, **kw), reps=2)
            except sp.ConversionError as exc:
                rec[key] = {"error": str(exc)[:60]}
                continue
            out_bytes = sp.spmv_bytes(tag, mm) - 8 * (mm.n_rows + mm.n_cols)
            rec[key] = {"ms": t * 1e3, "GBs_min_bytes": (csr_bytes + out_bytes) / t / 1e9}
            del mm
            torch.cuda.empty_cache()
        print(json.dumps(rec), flush=True)
        del a, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
