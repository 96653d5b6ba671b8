"""Generate golden fixtures by running the REFERENCE package (spmvkit).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``spmvkit`` from /root/reference/pkg/src, builds every format at
several parameter sets for a fixed list of seeded inputs (the paper's 4x4
Table-1 matrix, random sparse matrices, dense-row / empty-band / empty /
rectangular edge cases, duplicate-and-cancellation triplets), runs every
reference kernel and feature extractor, and stores inputs and outputs in
``tests/golden/cases.npz``.  The GPU box has no /root/reference; tests there
compare against these committed fixtures and against oracle/port.py.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().with_name("cases.npz")

CSR5_PARAMS = [(2, 2), (4, 16), (32, 16), (3, 5), (4, 3), (1, 1), (8, 4), (16, 2)]
SELL_PARAMS = [(4, 0), (2, 4), (3, 0), (4, 8), (32, 64), (1, 0), (2, 2)]


def _cases(rng):
    """(name, n_rows, n_cols, row, col, val) raw (possibly unsorted) triplets."""
    demo = [(0, 1, 6.0), (0, 2, 1.0), (1, 0, 2.0), (1, 2, 8.0), (1, 3, 3.0), (2, 2, 4.0), (3, 1, 7.0), (3, 2, 5.0)]
    r, c, v = (np.array(t) for t in zip(*demo))
    yield "demo", 4, 4, r[::-1].copy(), c[::-1].copy(), v[::-1].astype(np.float64).copy()
    for i in range(14):
        nr = int(rng.integers(1, 65))
        nc = int(rng.integers(1, 65))
        dens = float(rng.uniform(0.005, 0.25))
        nnz = min(nr * nc, max(0, round(dens * nr * nc)))
        flat = rng.choice(nr * nc, size=nnz, replace=False)
        vals = rng.uniform(0.1, 3.0, size=nnz) * rng.choice([-1.0, 1.0], size=nnz)
        yield f"rand{i}", nr, nc, flat // nc, flat % nc, vals
    # 200x200 at 5% (the reference's kernel property-test size)
    flat = rng.choice(40000, size=2000, replace=False)
    yield "rand200", 200, 200, flat // 200, flat % 200, rng.normal(size=2000)
    # a dense row in a sparse matrix
    n = 64
    flat = rng.choice(n * n, size=80, replace=False)
    dr = 17
    yield ("dense_row", n, n, np.concatenate([flat // n, np.full(n, dr)]), np.concatenate([flat % n, np.arange(n)]),
           np.concatenate([rng.uniform(0.1, 3, 80), rng.uniform(0.1, 1.0, n)]))
    # empty band of rows and empty leading columns
    n = 80
    flat = rng.choice(n * n, size=320, replace=False)
    rr, cc = flat // n, flat % n
    keep = ((rr < n // 3) | (rr >= 2 * n // 3)) & (cc >= 4)
    yield "empty_band", n, n, rr[keep], cc[keep], rng.uniform(-2, 2, int(keep.sum()))
    # one row spanning several CSR5 tiles, plus rows that start mid-tile
    yield "long_row", 3, 150, np.concatenate([np.zeros(130, int), [1, 2, 2]]), \
        np.concatenate([np.arange(130), [5, 0, 149]]), np.linspace(0.5, 2.0, 133)
    # duplicates (summed in numpy reduceat order), cancellation, signed zeros
    yield ("dups", 5, 6, np.array([1, 0, 1, 4, 4, 4, 2, 2, 3, 3, 3, 3, 0, 0]),
           np.array([1, 0, 1, 5, 5, 5, 2, 2, 0, 0, 0, 0, 3, 3]),
           np.array([2.0, 1.0, 3.0, 0.1, 0.2, 0.3, 1.5, -1.5, 1e16, 1.0, -1e16, 1.0, -0.0, 0.0]))
    many = rng.integers(0, 4, size=300)
    yield "dup_run", 4, 2, many, np.zeros(300, int), rng.normal(size=300)
    yield "empty", 5, 7, np.empty(0, int), np.empty(0, int), np.empty(0)
    yield "one", 1, 1, np.array([0]), np.array([0]), np.array([3.0])
    yield "zero_rows", 0, 5, np.empty(0, int), np.empty(0, int), np.empty(0)
    yield "zero_cols", 5, 0, np.empty(0, int), np.empty(0, int), np.empty(0)
    for shape in [(1, 200), (200, 1), (3, 97)]:
        nr, nc = shape
        nnz = round(0.3 * nr * nc)
        flat = rng.choice(nr * nc, size=nnz, replace=False)
        yield f"rect{nr}x{nc}", nr, nc, flat // nc, flat % nc, rng.normal(size=nnz)


def main() -> None:
    sys.path.insert(0, str(REF))
    import spmvkit as sk  # the reference, unmodified
    from spmvkit.kernels import _csr5_tile_partials

    rng = np.random.default_rng(20240817)
    out: dict[str, np.ndarray] = {}
    names = []
    for name, nr, nc, r, c, v in _cases(rng):
        names.append(name)
        p = f"{name}/"
        out[p + "shape"] = np.array([nr, nc])
        out[p + "in_row"], out[p + "in_col"], out[p + "in_val"] = (np.asarray(r, np.int64), np.asarray(c, np.int64),
                                                                  np.asarray(v, np.float64))
        a = sk.canonicalize(r, c, v, nr, nc)
        out[p + "row"], out[p + "col"], out[p + "data"] = a.row, a.col, a.data
        out[p + "counts"] = sk.row_nnz_histogram(a)
        x = rng.normal(size=nc)
        out[p + "x"] = x
        out[p + "y_oracle"] = sk.dense_spmv_oracle(a, x)
        m = sk.to_csr(a)
        out[p + "csr/ptr"] = m.ptr
        out[p + "csr/y"] = sk.spmv("csr", m, x)
        for om, sg in CSR5_PARAMS:
            m5 = sk.to_csr5(a, om, sg)
            q = f"{p}csr5_{om}_{sg}/"
            for f in ("tile_ptr", "bit_flag", "y_off", "seg_off", "indices", "data"):
                out[q + f] = getattr(m5, f)
            out[q + "y"] = sk.spmv("csr5", m5, x)
            if m5.num_tiles:
                rows, sums = [], []
                for t in range(m5.num_tiles):
                    rr, ss = _csr5_tile_partials(m5, x, t)
                    rows.append(rr)
                    sums.append(ss)
                out[q + "partial_rows"] = np.concatenate(rows)
                out[q + "partial_sums"] = np.concatenate(sums)
        try:
            me = sk.to_ell(a)
            out[p + "ell/k"] = np.array(me.k)
            out[p + "ell/indices"], out[p + "ell/data"], out[p + "ell/row_nnz"] = me.indices, me.data, me.row_nnz
            out[p + "ell/y"] = sk.spmv("ell", me, x)
        except sk.ConversionError:
            out[p + "ell/k"] = np.array(-1)
        for cc, ss in SELL_PARAMS:
            ms = sk.to_sell(a, cc, ss)
            q = f"{p}sell_{cc}_{ss}/"
            out[q + "perm"], out[q + "widths"], out[q + "row_nnz_perm"] = ms.perm, ms.widths, ms.row_nnz_perm
            out[q + "flat_data"] = np.concatenate([d.ravel(order="F") for d in ms.data]) if ms.data else np.empty(0)
            out[q + "flat_indices"] = (np.concatenate([d.ravel(order="F") for d in ms.indices]) if ms.indices
                                       else np.empty(0, np.int64))
            out[q + "y"] = sk.spmv("sell", ms, x)
        mh = sk.to_hyb(a)
        out[p + "hyb/k"] = np.array(mh.k)
        out[p + "hyb/ell_indices"], out[p + "hyb/ell_data"] = mh.ell.indices, mh.ell.data
        out[p + "hyb/ell_row_nnz"] = mh.ell.row_nnz
        out[p + "hyb/tail_row"], out[p + "hyb/tail_col"] = mh.coo_tail.row, mh.coo_tail.col
        out[p + "hyb/tail_data"] = mh.coo_tail.data
        out[p + "hyb/y"] = sk.spmv("hyb", mh, x)
        if nr and nc:
            f = sk.extract_features(a)
            out[p + "features"] = f.as_array()
        if nr:
            out[p + "hyb_k"] = np.array(sk.hyb_typical_k(out[p + "counts"]))
        out[p + "bytes"] = np.array([
            sk.bandwidth_estimate("csr", m, 1.0),
            sk.bandwidth_estimate("csr5", sk.to_csr5(a, 4, 16), 1.0),
            sk.bandwidth_estimate("sell", sk.to_sell(a, 4, 0), 1.0),
            sk.bandwidth_estimate("hyb", mh, 1.0),
        ])
    # A format-selection model trained by the reference itself (train_tree on
    # its helpers' synthetic cost-model corpus), saved in its text format,
    # plus the tag its predict() assigns to every case above.
    import io

    sys.path.insert(0, str(REF.parent / "tests"))
    import helpers  # reference test helpers (cost-model corpus)

    corpus = helpers.make_cost_corpus(7, 60)
    samples = []
    for mid, a in corpus:
        f = sk.extract_features(a)
        best = min(sk.FormatTag, key=lambda t: (helpers.cost_model(f, t), list(sk.FormatTag).index(t)))
        samples.append(sk.LabeledSample(mid, f, best))
    model = sk.train_tree(samples, max_depth=6, min_samples_leaf=2)
    buf = io.StringIO()
    sk.save_model(model, buf)
    out["__model__"] = np.array(buf.getvalue())
    for name in names:
        nr, nc = (int(t) for t in out[name + "/shape"])
        if nr and nc:
            a = sk.canonicalize(out[name + "/row"], out[name + "/col"], out[name + "/data"], nr, nc)
            out[name + "/predicted"] = np.array(sk.predict(model, sk.extract_features(a)).value)
    out["__names__"] = np.array(names)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(names)} cases)")


if __name__ == "__main__":
    main()
