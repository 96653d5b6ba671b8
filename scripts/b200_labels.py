"""B200 best-format labels for a synthetic corpus.

Generates ~250 matrices on the GPU across the structure families that
separate the five formats (regular stencils and bands, block-diagonal,
uniform random, log-normal row lengths, R-MAT power law, bands with a few
dense rows, rectangular shapes), benchmarks every format on each with
``harness.bench_corpus`` (the reference's CI stopping rule, CUDA-event
clock) and writes, in the REFERENCE's own file formats,

    <out>/b200_records.txt    one BenchRecord line per (matrix, format)
    <out>/b200_features.txt   one feature line per matrix (GPU features)
    <out>/b200_corpus.jsonl   family / parameters / n / nnz per matrix

spmvkit's unchanged CPU code (train_tree, cross_validate, save_model) then
trains the B200 selector from them: scripts/train_b200_model.py.

    python scripts/b200_labels.py [--out gpurun_out] [--quick]

Hot-cache protocol, as the reference's run_bench: repetitions run back to
back, so matrices under ~100 MB are served from the 126 MB L2.  A timed
sample is 20 back-to-back prepared launches (BenchConfig.inner_reps): one
SpMV of the smaller matrices takes 3-10 us, below what one event pair
resolves.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import harness, synth  # noqa: E402

DEV = torch.device("cuda", 0)


def _vals(n, g):
    return torch.rand(n, generator=g, device=DEV, dtype=torch.float64) * 0.9 + 0.1


def _coo(r, c, g, n_rows, n_cols):
    return sp.canonicalize(r.to(torch.int32), c.to(torch.int32), _vals(r.numel(), g), n_rows, n_cols)


def gen_uniform(n_rows, n_cols, deg, g):
    nnz = int(n_rows * deg)
    r = torch.randint(0, n_rows, (nnz,), generator=g, device=DEV)
    c = torch.randint(0, n_cols, (nnz,), generator=g, device=DEV)
    return _coo(r, c, g, n_rows, n_cols)


def gen_banded(n, k, half, drop, g):
    r = torch.arange(n, device=DEV).repeat_interleave(k)
    c = (r + torch.randint(-half, half + 1, (r.numel(),), generator=g, device=DEV)).clamp_(0, n - 1)
    if drop > 0:
        keep = torch.rand(r.numel(), generator=g, device=DEV) >= drop
        r, c = r[keep], c[keep]
    return _coo(r, c, g, n, n)


def gen_blockdiag(n, b, g):
    r = torch.arange(n, device=DEV).repeat_interleave(b)
    c = (r // b) * b + torch.arange(b, device=DEV).repeat(n)
    c = c.clamp_(0, n - 1)
    return _coo(r, c, g, n, n)


def gen_lognormal(n_rows, n_cols, mean_len, sigma, g):
    """Row lengths ~ lognormal with the given mean and shape: the variation
    feature sweeps continuously from ELL-friendly to CSR5 territory."""
    mu = math.log(mean_len) - 0.5 * sigma * sigma
    z = torch.randn(n_rows, generator=g, device=DEV, dtype=torch.float64)
    lens = torch.exp(mu + sigma * z).round_().clamp_(0, n_cols // 2).to(torch.int64)
    r = torch.arange(n_rows, device=DEV).repeat_interleave(lens)
    c = torch.randint(0, n_cols, (r.numel(),), generator=g, device=DEV)
    return _coo(r, c, g, n_rows, n_cols)


def gen_rmat(scale, ef, seed, abc):
    r, c, v = synth.rmat_triplets(scale, ef, seed, DEV, abc=abc)
    n = 1 << scale
    return sp.canonicalize(r, c, v, n, n)


def gen_band_dense_rows(n, k, n_dense, dense_len, g):
    r = torch.arange(n, device=DEV).repeat_interleave(k)
    c = (r + torch.randint(-32, 33, (r.numel(),), generator=g, device=DEV)).clamp_(0, n - 1)
    dr = torch.randint(0, n, (n_dense,), generator=g, device=DEV).repeat_interleave(dense_len)
    dc = torch.randint(0, n, (dr.numel(),), generator=g, device=DEV)
    return _coo(torch.cat([r, dr]), torch.cat([c, dc]), g, n, n)


def gen_host(kind, **kw):
    hr, hc, hv, n = {"laplace2d": synth.laplace2d, "stencil27": synth.stencil27}[kind](**kw)
    return sp.canonicalize(torch.from_numpy(hr).to(DEV, torch.int32), torch.from_numpy(hc).to(DEV, torch.int32),
                           torch.from_numpy(hv).to(DEV), n, n)


def corpus(quick: bool):
    """(matrix_id, family, params, maker) in a fixed order; every maker is seeded."""
    out = []

    def add(family, params, fn):
        mid = family + "/" + "_".join(f"{k}{v}" for k, v in params.items())
        out.append((mid, family, params, fn))

    def gen(seed):
        g = torch.Generator(device=DEV)
        g.manual_seed(seed)
        return g

    seed = 1000
    for gsz in ([256, 512] if quick else [192, 256, 384, 512, 768, 1024, 1536, 2048]):
        add("laplace2d", dict(g=gsz), lambda gsz=gsz: gen_host("laplace2d", g=gsz))
    for gsz in ([32] if quick else [24, 32, 48, 64, 80, 96, 112]):
        add("stencil27", dict(g=gsz), lambda gsz=gsz: gen_host("stencil27", g=gsz))
    for logn in ([18] if quick else [17, 18, 19, 20, 21, 22]):
        for k in ([8] if quick else [3, 6, 12, 24, 48]):
            for drop in (0.0, 0.3):
                if (1 << logn) * k > 40_000_000:
                    continue
                seed += 1
                add("banded", dict(n=1 << logn, k=k, drop=drop),
                    lambda logn=logn, k=k, drop=drop, s=seed: gen_banded(1 << logn, k, 64, drop, gen(s)))
    for logn in ([18] if quick else [17, 19, 21]):
        for b in ([8] if quick else [4, 8, 16, 32]):
            seed += 1
            add("blockdiag", dict(n=1 << logn, b=b), lambda logn=logn, b=b, s=seed: gen_blockdiag(1 << logn, b, gen(s)))
    for logn in ([18] if quick else [16, 18, 20, 21]):
        for deg in ([8] if quick else [2, 5, 10, 20, 40]):
            if (1 << logn) * deg > 40_000_000:
                continue
            seed += 1
            add("uniform", dict(n=1 << logn, deg=deg),
                lambda logn=logn, deg=deg, s=seed: gen_uniform(1 << logn, 1 << logn, deg, gen(s)))
    for logn in ([18] if quick else [17, 19, 21]):
        for mean_len in ([8] if quick else [4, 12, 32]):
            for sigma in ([1.0] if quick else [0.25, 0.5, 1.0, 1.5, 2.0]):
                if (1 << logn) * mean_len > 40_000_000:
                    continue
                seed += 1
                add("lognormal", dict(n=1 << logn, len=mean_len, s=sigma),
                    lambda logn=logn, mean_len=mean_len, sigma=sigma, s=seed:
                    gen_lognormal(1 << logn, 1 << logn, mean_len, sigma, gen(s)))
    for scale in ([16] if quick else [16, 17, 18, 19, 20, 21, 22]):
        for ef in ([8] if quick else [4, 8, 16, 32]):
            for name, abc in (("g500", (0.57, 0.19, 0.19)), ("mild", (0.45, 0.22, 0.22)), ("flat", (0.30, 0.25, 0.25))):
                if (1 << scale) * ef > 40_000_000 or (quick and name != "g500"):
                    continue
                seed += 1
                add("rmat", dict(scale=scale, ef=ef, abc=name),
                    lambda scale=scale, ef=ef, abc=abc, s=seed: gen_rmat(scale, ef, s, abc))
    for logn in ([18] if quick else [18, 20]):
        for n_dense, dense_len in ([(4, 20000)] if quick else [(1, 5000), (4, 20000), (16, 50000), (64, 100000)]):
            seed += 1
            add("band_dense", dict(n=1 << logn, rows=n_dense, len=dense_len),
                lambda logn=logn, n_dense=n_dense, dense_len=dense_len, s=seed:
                gen_band_dense_rows(1 << logn, 8, n_dense, min(dense_len, (1 << logn) // 2), gen(s)))
    for (nr, nc) in ([] if quick else [(1 << 21, 1 << 15), (1 << 15, 1 << 21), (1 << 20, 1 << 18), (1 << 18, 1 << 20)]):
        for deg in (6, 30):
            if nr * deg > 40_000_000:
                continue
            seed += 1
            add("rect", dict(rows=nr, cols=nc, deg=deg), lambda nr=nr, nc=nc, deg=deg, s=seed: gen_uniform(nr, nc, deg, gen(s)))
    return out


def feature_line(mid: str, f) -> str:
    """spmvkit.features.features_to_line (features.py:105-110), token for token."""
    toks = [f"matrix_id:{mid}"]
    for name in sp.FEATURE_NAMES:
        v = getattr(f, name)
        toks.append(f"{name}:{v if isinstance(v, int) else repr(float(v))}")
    return " ".join(toks)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--quick", action="store_true", help="a dozen small matrices (smoke run)")
    args = ap.parse_args()
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    cfg = harness.BenchConfig(min_reps=5, max_reps=200, ci_gap=0.05, warmup_reps=3, csr5_omega=32, csr5_sigma=16,
                              sell_c=32, sell_sigma=1024, max_grid_cells=1 << 28, inner_reps=20)
    records, feats, meta = [], [], []
    t_start = time.perf_counter()
    items = corpus(args.quick)
    for i, (mid, family, params, make) in enumerate(items):
        a = make()
        if a.nnz == 0:
            continue
        f = sp.extract_features(a)
        recs, labels, _ = harness.bench_corpus([(mid, a)], cfg)
        records += recs
        feats.append(feature_line(mid, f))
        per = {r.format.value: r.mean_time_s for r in recs if r.converted_ok}
        meta.append(dict(matrix_id=mid, family=family, params=params, n_rows=a.n_rows, n_cols=a.n_cols, nnz=a.nnz,
                         best=labels[mid].value, us={k: round(v * 1e6, 2) for k, v in per.items()}))
        print(f"[{i + 1}/{len(items)}] {mid}: nnz {a.nnz} best {labels[mid].value} "
              + " ".join(f"{k} {v * 1e6:.1f}" for k, v in per.items()), flush=True)
        del a
        torch.cuda.empty_cache()
    harness.write_records(records, out / "b200_records.txt")
    (out / "b200_features.txt").write_text("".join(line + "\n" for line in feats))
    (out / "b200_corpus.jsonl").write_text("".join(json.dumps(m) + "\n" for m in meta))
    hist = {}
    for m in meta:
        hist[m["best"]] = hist.get(m["best"], 0) + 1
    print(f"{len(meta)} matrices, {len(records)} records in {time.perf_counter() - t_start:.0f} s; labels {hist}")


if __name__ == "__main__":
    main()
