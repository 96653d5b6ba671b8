"""Pin the CPU oracle (oracle/port.py) before trusting it.

(1) The reference's own golden vectors: the paper's Table-1 arrays asserted
    by the reference tests (test_formats.py:23-27, 42-50, 126-132, 167-185,
    242-249; test_kernels.py:45-47, 82-90; test_features.py:22-31).
(2) Fixtures produced by running the reference itself
    (tests/golden/make_golden.py): every array must match bit for bit.
CPU only.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import demo_triplets
from oracle import port, synth_ref

CSR5_PARAMS = [(2, 2), (4, 16), (32, 16), (3, 5), (4, 3), (1, 1), (8, 4), (16, 2)]
SELL_PARAMS = [(4, 0), (2, 4), (3, 0), (4, 8), (32, 64), (1, 0), (2, 2)]


def _demo():
    r, c, v = demo_triplets()
    return port.canonicalize(r, c, v, 4, 4)


def test_table1_csr():
    r, c, v = _demo()
    ptr, ind, dat = port.to_csr(r, c, v, 4)
    assert ptr.tolist() == [0, 2, 5, 6, 8]
    assert ind.tolist() == [1, 2, 0, 2, 3, 2, 1, 2]
    assert dat.tolist() == [6, 1, 2, 8, 3, 4, 7, 5]


def test_table1_csr5():
    r, c, v = _demo()
    ptr, ind, dat = port.to_csr(r, c, v, 4)
    m = port.to_csr5(ptr, ind, dat, 4, 2, 2)
    assert m.num_tiles == 2
    assert m.tile_ptr.tolist() == [0, 1, 4]
    assert m.bit_flag.tolist() == [True, True, False, False, True, True, True, False]
    assert m.y_off.tolist() == [[0, 1], [0, 2]]
    assert m.seg_off.tolist() == [[0, 0], [0, 0]]
    assert m.indices.tolist() == [1, 0, 2, 2, 3, 1, 2, 2]
    assert m.data.tolist() == [6, 2, 1, 8, 3, 7, 4, 5]
    x = np.ones(4)
    r0, s0 = port.csr5_tile_partials(m, x, 0)
    r1, s1 = port.csr5_tile_partials(m, x, 1)
    assert r0.tolist() == [0, 1] and s0.tolist() == [7.0, 10.0]
    assert r1.tolist() == [1, 2, 3] and s1.tolist() == [3.0, 4.0, 12.0]


def test_table1_ell_sell_hyb():
    r, c, v = _demo()
    ptr, ind, dat = port.to_csr(r, c, v, 4)
    k, gi, gd, cnt = port.to_ell(ptr, ind, dat, 4)
    assert k == 3
    assert gd.tolist() == [[6, 1, 0], [2, 8, 3], [4, 0, 0], [7, 5, 0]]
    assert gi.tolist() == [[1, 2, 2], [0, 2, 3], [2, 2, 2], [1, 2, 2]]
    s = port.to_sell(ptr, ind, dat, 4, 2, 0)
    assert s.widths.tolist() == [3, 2]
    assert s.data[0].tolist() == [[6, 1, 0], [2, 8, 3]] and s.data[1].tolist() == [[4, 0], [7, 5]]
    assert s.indices[1].tolist() == [[2, 2], [1, 2]]
    s = port.to_sell(ptr, ind, dat, 4, 2, 4)
    assert s.perm.tolist() == [1, 0, 3, 2]
    assert s.data[0].tolist() == [[2, 8, 3], [6, 1, 0]]
    K, hi, hd, hn, tail = port.to_hyb(r, c, v, 4)
    assert K == 2
    assert hd.tolist() == [[6, 1], [2, 8], [4, 0], [7, 5]]
    assert hi.tolist() == [[1, 2], [0, 2], [2, 2], [1, 2]]
    assert [t.tolist() for t in tail] == [[1], [3], [3.0]]
    assert port.hyb_typical_k([2, 3, 1, 2]) == 2
    assert port.hyb_typical_k([1, 1, 1, 100]) == 1
    assert port.hyb_typical_k([10, 0, 0]) == 1


def test_table1_kernels_and_features():
    r, c, v = _demo()
    ptr, ind, dat = port.to_csr(r, c, v, 4)
    x = np.ones(4)
    want = [7.0, 13.0, 4.0, 12.0]
    assert port.spmv_csr(ptr, ind, dat, 4, x).tolist() == want
    assert port.spmv_csr5(port.to_csr5(ptr, ind, dat, 4, 2, 2), 4, x).tolist() == want
    k, gi, gd, _ = port.to_ell(ptr, ind, dat, 4)
    assert port.spmv_ell(k, gi, gd, x).tolist() == want
    assert port.spmv_sell(port.to_sell(ptr, ind, dat, 4, 2, 4), 4, x).tolist() == want
    K, hi, hd, _, tail = port.to_hyb(r, c, v, 4)
    assert port.spmv_hyb(K, hi, hd, tail, 4, x).tolist() == want
    f = port.extract_features(r, 4, 4)
    assert f == (4, 4, 0.5, 1, 3, 2.0, math.sqrt(0.5), math.sqrt(0.5) / 2.0)
    assert port.dense_spmv_oracle(r, c, v, 4, x).tolist() == want


def test_byte_model_golden():
    r, c, v = _demo()
    assert port.spmv_bytes("csr", 4, 4, nnz=8) == 180  # bench.py byte model, test_bench.py:121-125
    assert port.spmv_bytes("ell", 4, 4, k=3) == 144 + 64
    assert port.spmv_bytes("csr5", 4, 4, nnz=8, num_tiles=2, omega=2) == 12 * 8 + 20 + 12 + 8 + 32 + 64


def _cases(golden):
    return golden.names


def test_oracle_matches_reference_fixtures(golden):
    for name in golden.names:
        g = golden.case(name)
        nr, nc = (int(t) for t in g["shape"])
        r, c, v = port.canonicalize(g["in_row"], g["in_col"], g["in_val"], nr, nc)
        assert np.array_equal(r, g["row"]) and np.array_equal(c, g["col"]), name
        assert v.tobytes() == g["data"].tobytes(), name
        x = g["x"]
        assert port.dense_spmv_oracle(r, c, v, nr, x).tobytes() == g["y_oracle"].tobytes(), name
        ptr, ind, dat = port.to_csr(r, c, v, nr)
        assert np.array_equal(ptr, g["csr/ptr"]), name
        assert port.spmv_csr(ptr, ind, dat, nr, x).tobytes() == g["csr/y"].tobytes(), name
        for om, sg in CSR5_PARAMS:
            m = port.to_csr5(ptr, ind, dat, nr, om, sg)
            q = f"csr5_{om}_{sg}/"
            for f in ("tile_ptr", "bit_flag", "y_off", "seg_off", "indices"):
                assert np.array_equal(getattr(m, f), g[q + f]), (name, q, f)
            assert m.data.tobytes() == g[q + "data"].tobytes()
            assert port.spmv_csr5(m, nr, x).tobytes() == g[q + "y"].tobytes(), (name, q)
        if int(g["ell/k"]) >= 0:
            k, gi, gd, cnt = port.to_ell(ptr, ind, dat, nr)
            assert k == int(g["ell/k"]) and np.array_equal(gi, g["ell/indices"]), name
            assert gd.tobytes() == g["ell/data"].tobytes() and np.array_equal(cnt, g["ell/row_nnz"])
            assert port.spmv_ell(k, gi, gd, x).tobytes() == g["ell/y"].tobytes(), name
        for cc, ss in SELL_PARAMS:
            s = port.to_sell(ptr, ind, dat, nr, cc, ss)
            q = f"sell_{cc}_{ss}/"
            assert np.array_equal(s.perm, g[q + "perm"]) and np.array_equal(s.widths, g[q + "widths"]), (name, q)
            flat_d = np.concatenate([d.ravel(order="F") for d in s.data]) if s.data else np.empty(0)
            flat_i = np.concatenate([d.ravel(order="F") for d in s.indices]) if s.indices else np.empty(0, np.int64)
            assert flat_d.tobytes() == g[q + "flat_data"].tobytes() and np.array_equal(flat_i, g[q + "flat_indices"])
            assert port.spmv_sell(s, nr, x).tobytes() == g[q + "y"].tobytes(), (name, q)
        K, hi, hd, hn, tail = port.to_hyb(r, c, v, nr)
        assert K == int(g["hyb/k"]) and np.array_equal(hi, g["hyb/ell_indices"]), name
        assert np.array_equal(tail[0], g["hyb/tail_row"]) and np.array_equal(tail[1], g["hyb/tail_col"])
        assert port.spmv_hyb(K, hi, hd, tail, nr, x).tobytes() == g["hyb/y"].tobytes(), name
        if nr and nc:
            assert np.array(port.extract_features(r, nr, nc)).tobytes() == g["features"].tobytes(), name
        if nr:
            assert port.hyb_typical_k(g["counts"]) == int(g["hyb_k"])


def test_hyb_typical_k_brute_force(rng):
    # independent scan: largest K where strictly more than n/3 rows reach K (test_formats.py:229-238)
    for _ in range(200):
        counts = rng.integers(0, 20, size=int(rng.integers(1, 30)))
        best = 1
        for k in range(1, 21):
            if 3 * int((counts >= k).sum()) > counts.size:
                best = k
        assert port.hyb_typical_k(counts) == best


def test_synth_ref_rmat_is_deterministic_and_deduplicated():
    r, c, v = synth_ref.rmat(8, 4, seed=7)
    r2, c2, v2 = synth_ref.rmat(8, 4, seed=7)
    assert np.array_equal(r, r2) and v.tobytes() == v2.tobytes()
    key = (r << 8) | c
    assert np.unique(key).size == key.size
    assert (v > 0).all() and (v <= 1).all()
    # the quadrant skew (a=0.57) makes low row ids denser
    assert (r < 128).mean() > 0.6


def test_model_loading_and_prediction_match_reference(golden):
    """model.load_model parses the reference's model file; model.predict (host
    tree descent, model.py:216-223) reproduces the reference's predictions on
    the reference's own feature vectors."""
    import io

    from paper_1805_11938_b200.features import FeatureVector
    from paper_1805_11938_b200.model import load_model, predict

    model = load_model(io.StringIO(str(golden.d["__model__"])))
    checked = 0
    for name in golden.names:
        g = golden.case(name)
        if "predicted" not in g:
            continue
        f = g["features"]
        fv = FeatureVector(int(f[0]), int(f[1]), float(f[2]), int(f[3]), int(f[4]), float(f[5]), float(f[6]),
                           float(f[7]))
        assert predict(model, fv).value == str(g["predicted"]), name
        checked += 1
    assert checked >= 20


def test_full_rmat_csr_builder_matches_port():
    """oracle/rmat_sample.c:rmat_csr (the CPU reference arm's whole-matrix
    build) equals the port's canonicalize/to_csr of the host-regenerated
    draws, bit for bit."""
    from oracle import cpu_baseline, synth_ref

    for scale, ef, seed in [(11, 8, 3), (13, 16, 105), (9, 1, 7)]:
        p, i, d = cpu_baseline.rmat_full_csr(scale, ef, seed, threads=4)
        hr, hc, hv = synth_ref.rmat(scale, ef, seed)
        n = 1 << scale
        r, c, v = port.canonicalize(hr, hc, hv, n, n)
        p2, i2, d2 = port.to_csr(r, c, v, n)
        assert np.array_equal(p, p2) and np.array_equal(i, i2) and d.tobytes() == d2.tobytes()


def test_row_subset_matches_port():
    from oracle import cpu_baseline, synth_ref

    rows, ptr, ind, dat = cpu_baseline.rmat_row_subset(12, 8, 3, keep_mod=5, ranges=[(0, 3), (2000, 2100)], threads=3)
    hr, hc, hv = synth_ref.rmat(12, 8, 3)
    r, c, v = port.canonicalize(hr, hc, hv, 1 << 12, 1 << 12)
    P, I, D = port.to_csr(r, c, v, 1 << 12)
    assert {0, 1, 2, 2050} <= set(rows.tolist())
    for k, row in enumerate(rows):
        assert np.array_equal(I[P[row]:P[row + 1]], ind[ptr[k]:ptr[k + 1]])
        assert D[P[row]:P[row + 1]].tobytes() == dat[ptr[k]:ptr[k + 1]].tobytes()
