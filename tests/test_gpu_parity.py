"""GPU parity against the reference's fixtures (tests/golden/cases.npz) and
the CPU oracle.  Every call goes through the C ABI (libspmvb.so).

Bar: conversions and canonicalize bit-exact (indices by value, fp64 by
bits); ELL/SELL SpMV and dense_spmv_oracle bit-identical to the reference;
CSR/CSR5/HYB SpMV within |y - y_ref| <= 1e-12 * (|A| |x|) elementwise (the
north-star tolerance) and <= 1e-12 * (1 + |y_ref|) (the reference tests'
tolerance, test_kernels.py:25-30); repeated runs bit-identical.
"""

from __future__ import annotations

import io
import math

import numpy as np
import pytest
import torch

from conftest import demo_triplets, random_triplets
from oracle import port

pytestmark = pytest.mark.gpu

CSR5_PARAMS = [(2, 2), (4, 16), (32, 16), (3, 5), (4, 3), (1, 1), (8, 4), (16, 2)]
SELL_PARAMS = [(4, 0), (2, 4), (3, 0), (4, 8), (32, 64), (1, 0), (2, 2)]
TOL = 1e-12


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def same_bits(a, b) -> bool:
    a, b = np.asarray(np_(a), dtype=np.float64), np.asarray(np_(b), dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def assert_within(y, ref, absA_absx):
    y, ref = np_(y), np.asarray(ref)
    d = np.abs(y - ref)
    assert np.all(d <= TOL * absA_absx), float((d - TOL * absA_absx).max())
    assert np.all(d <= TOL * (1.0 + np.abs(ref)))


def abs_bound(g, nr):
    return port.dense_spmv_oracle(g["row"], g["col"], np.abs(g["data"]), nr, np.abs(g["x"]))


def test_every_case_matches_reference(sp, golden):
    for name in golden.names:
        g = golden.case(name)
        nr, nc = (int(t) for t in g["shape"])
        a = sp.canonicalize(g["in_row"], g["in_col"], g["in_val"], nr, nc)
        assert np.array_equal(np_(a.row), g["row"]) and np.array_equal(np_(a.col), g["col"]), name
        assert same_bits(a.data, g["data"]), name
        assert np.array_equal(np_(sp.row_nnz_histogram(a)), g["counts"]), name
        x = torch.from_numpy(g["x"]).cuda()
        bound = abs_bound(g, nr)
        assert same_bits(sp.dense_spmv_oracle(a, x), g["y_oracle"]), name
        m = sp.to_csr(a)
        assert np.array_equal(np_(m.ptr), g["csr/ptr"]), name
        y = sp.spmv("csr", m, x)
        assert_within(y, g["y_oracle"], bound)
        assert same_bits(sp.spmv("csr", m, x), y)
        for om, sg in CSR5_PARAMS:
            q = f"csr5_{om}_{sg}/"
            m5 = sp.to_csr5(a, om, sg)
            for f in ("tile_ptr", "bit_flag", "y_off", "seg_off", "indices"):
                assert np.array_equal(np_(getattr(m5, f)), g[q + f]), (name, q, f)
            assert same_bits(m5.data, g[q + "data"]), (name, q)
            y5 = sp.spmv("csr5", m5, x)
            assert_within(y5, g["y_oracle"], bound)
            assert same_bits(sp.spmv("csr5", m5, x), y5)
            assert sp.coo_equal(sp.to_coo(m5), a), (name, q)
        if int(g["ell/k"]) >= 0:
            me = sp.to_ell(a)
            assert me.k == int(g["ell/k"]), name
            assert np.array_equal(np_(me.indices), g["ell/indices"]), name
            assert same_bits(me.data.contiguous(), g["ell/data"]) and np.array_equal(np_(me.row_nnz), g["ell/row_nnz"])
            assert same_bits(sp.spmv("ell", me, x), g["ell/y"]), name
            assert sp.coo_equal(sp.to_coo(me), a), name
        for cc, ss in SELL_PARAMS:
            q = f"sell_{cc}_{ss}/"
            ms = sp.to_sell(a, cc, ss)
            assert np.array_equal(np_(ms.perm), g[q + "perm"]), (name, q)
            assert np.array_equal(np_(ms.widths), g[q + "widths"]), (name, q)
            assert np.array_equal(np_(ms.row_nnz_perm), g[q + "row_nnz_perm"]), (name, q)
            assert np.array_equal(np_(ms.flat_indices), g[q + "flat_indices"]), (name, q)
            assert same_bits(ms.flat_data, g[q + "flat_data"]), (name, q)
            assert same_bits(sp.spmv("sell", ms, x), g[q + "y"]), (name, q)
            assert sp.coo_equal(sp.to_coo(ms), a), (name, q)
        mh = sp.to_hyb(a)
        assert mh.k == int(g["hyb/k"]), name
        assert np.array_equal(np_(mh.ell.indices), g["hyb/ell_indices"]), name
        assert same_bits(mh.ell.data.contiguous(), g["hyb/ell_data"]), name
        assert np.array_equal(np_(mh.ell.row_nnz), g["hyb/ell_row_nnz"]), name
        assert np.array_equal(np_(mh.coo_tail.row), g["hyb/tail_row"]), name
        assert np.array_equal(np_(mh.coo_tail.col), g["hyb/tail_col"]), name
        assert same_bits(mh.coo_tail.data, g["hyb/tail_data"]), name
        yh = sp.spmv("hyb", mh, x)
        assert_within(yh, g["y_oracle"], bound)
        assert sp.coo_equal(sp.to_coo(mh), a), name
        assert sp.coo_equal(sp.to_coo(m), a), name
        if nr and nc:
            f = sp.extract_features(a)
            assert f.as_array().tobytes() == g["features"].tobytes(), name
        if nr:
            assert sp.hyb_typical_k(g["counts"]) == int(g["hyb_k"]), name
        got = [sp.bandwidth_estimate("csr", m, 1.0), sp.bandwidth_estimate("csr5", sp.to_csr5(a, 4, 16), 1.0),
               sp.bandwidth_estimate("sell", sp.to_sell(a, 4, 0), 1.0), sp.bandwidth_estimate("hyb", mh, 1.0)]
        assert got == g["bytes"].tolist(), name


def test_demo_hand_results(sp):
    r, c, v = demo_triplets()
    a = sp.canonicalize(r, c, v, 4, 4)
    for tag in sp.FormatTag:
        m = sp.convert(tag, a, omega=2, sigma=2, sell_c=2, sell_sigma=4)
        assert sp.spmv(tag, m, np.ones(4)).tolist() == [7.0, 13.0, 4.0, 12.0]
        assert sp.spmv(tag, m, np.zeros(4)).tolist() == [0.0] * 4
        with pytest.raises(ValueError, match="length"):
            sp.spmv(tag, m, np.ones(5))
    with pytest.raises(ValueError, match="does not match"):
        sp.spmv("hyb", sp.to_csr(a), np.ones(4))
    f = sp.extract_features(a)
    assert f.nnz_std == math.sqrt(0.5) and f.variation == math.sqrt(0.5) / 2.0 and f.nnz_frac == 0.5


def test_containers(sp):
    r, c, v = demo_triplets()
    m = sp.to_csr(sp.canonicalize(r, c, v, 4, 4))
    y = sp.spmv("csr", m, [1, 1, 1, 1])
    assert isinstance(y, np.ndarray) and y.tolist() == [7.0, 13.0, 4.0, 12.0]
    yc = sp.spmv("csr", m, torch.ones(4, dtype=torch.float64).pin_memory())
    assert isinstance(yc, torch.Tensor) and not yc.is_cuda and yc.tolist() == [7.0, 13.0, 4.0, 12.0]
    yd = sp.spmv("csr", m, torch.ones(4, dtype=torch.float64, device="cuda"))
    assert yd.is_cuda


def test_host_buffers(sp, rng):
    """Host x / host out= calls: bit-identical to the device call; the CSR5
    streamed entry point (spmvb_spmv_csr5_host) for every range count,
    including more ranges than tiles and chains of continuation tiles."""
    r, c, v = sp.synth.rmat_triplets(scale=13, edge_factor=12, seed=9)
    a = sp.canonicalize(r, c, v, 1 << 13, 1 << 13)
    x = rng.uniform(-1.0, 1.0, size=1 << 13)
    xd = torch.from_numpy(x).cuda()
    for tag, kw in [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("csr5", dict(omega=4, sigma=16)),
                    ("csr5", dict(omega=3, sigma=5)), ("hyb", {}), ("sell", dict(sell_c=32, sell_sigma=64))]:
        m = sp.convert(tag, a, **kw)
        yd = np_(sp.spmv(tag, m, xd))
        assert same_bits(sp.spmv(tag, m, x), yd), tag
        assert same_bits(sp.spmv(tag, m, torch.from_numpy(x).pin_memory()), yd), tag
        out = torch.empty(m.n_rows, dtype=torch.float64).pin_memory()
        assert sp.spmv(tag, m, torch.from_numpy(x).pin_memory(), out=out) is out and same_bits(out, yd), tag
        outn = np.empty(m.n_rows)
        assert sp.spmv(tag, m, x, out=outn) is outn and same_bits(outn, yd), tag
        if tag == "csr5":
            for k in (1, 2, 3, 8, 64, 10 ** 6):
                tb, rb = m.range_plan(k)
                assert tb[0] == 0 and tb[-1] == m.num_tiles and np.all(np.diff(tb) >= 0)
                assert rb[0] == 0 and rb[-1] == m.n_rows and np.all(np.diff(rb) >= 0)
                aux = np_(m.tile_aux).view(np.uint32)
                inner = tb[1:-1][tb[1:-1] < m.num_tiles]
                assert not np.any(aux[inner] >> 31), k  # ranges start at row-start tiles
                assert same_bits(sp.spmv_csr5(m, x, ranges=k), yd), (kw, k)
                # device ranges in shuffled order (the multi-GPU overlap path)
                yt = torch.full((m.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
                for j in rng.permutation(len(tb) - 1):
                    hi = int(rb[j + 1]) if j + 1 < len(tb) - 1 else m.n_rows
                    sp.spmv_csr5_tiles(m, xd, yt, int(tb[j]), int(tb[j + 1]), int(rb[j]), hi)
                assert same_bits(yt, yd), (kw, k)
    with pytest.raises(ValueError, match="out"):
        sp.spmv("csr", sp.to_csr(a), x, out=np.empty(3))
    # empty matrix / zero nnz through the host entry point
    e = sp.to_csr5(sp.canonicalize([], [], [], 5, 4), 4, 16)
    assert sp.spmv("csr5", e, np.ones(4)).tolist() == [0.0] * 5


def test_packed_flags_identical(sp, rng, monkeypatch):
    """The tile kernel's packed-flag path (one bit per entry, used when x
    exceeds L2) gives the same bits as the byte-flag path, for every
    specialised (omega, sigma), on the device, streamed-host and range paths."""
    from paper_1805_11938_b200 import kernels

    r, c, v = sp.synth.rmat_triplets(scale=13, edge_factor=12, seed=11)
    a = sp.canonicalize(r, c, v, 1 << 13, 1 << 13)
    x = rng.uniform(-1.0, 1.0, size=1 << 13)
    xd = torch.from_numpy(x).cuda()
    for om, sg in [(32, 16), (16, 16), (8, 16), (4, 16), (32, 8), (16, 8), (8, 8), (4, 8)]:
        m = sp.to_csr5(a, om, sg)
        assert m.flag_bits is not None
        monkeypatch.setattr(kernels, "_PACKED_FLAGS_MIN_X_BYTES", 1 << 62)
        yb = np_(sp.spmv("csr5", m, xd))
        monkeypatch.setattr(kernels, "_PACKED_FLAGS_MIN_X_BYTES", 0)
        assert same_bits(sp.spmv("csr5", m, xd), yb), (om, sg)
        assert same_bits(sp.spmv_csr5(m, x, ranges=5), yb), (om, sg)
        bits = np_(m.flag_bits).view(np.uint32)
        flags = np_(m.bit_flag).astype(np.uint32)
        padded = np.zeros(bits.size * 32, dtype=np.uint32)
        padded[: flags.size] = flags
        assert np.array_equal(bits, (padded.reshape(-1, 32) << np.arange(32, dtype=np.uint32)).sum(1)), (om, sg)


def test_select_format_measured(sp, rng):
    """The measured selector returns the fastest converted format and its
    matrix; ELL that cannot convert is skipped."""
    r, c, v = sp.synth.rmat_triplets(scale=12, edge_factor=8, seed=2)
    a = sp.canonicalize(r, c, v, 1 << 12, 1 << 12)
    tag, m, times = sp.select_format_measured(a, reps=3,
                                              params={sp.FormatTag.ELL: dict(max_cells=10)})
    assert sp.FormatTag.ELL not in times and tag in times
    assert times[tag] == min(times.values())
    x = torch.from_numpy(rng.uniform(-1, 1, size=1 << 12)).cuda()
    assert_within(sp.spmv(tag, m, x), sp.dense_spmv_oracle(a, x).cpu().numpy(),
                  sp.dense_spmv_oracle(sp.canonicalize(np_(a.row), np_(a.col), np.abs(np_(a.data)), 1 << 12,
                                                       1 << 12), torch.abs(x)).cpu().numpy())


def test_errors(sp):
    r, c, v = demo_triplets()
    a = sp.canonicalize(r, c, v, 4, 4)
    with pytest.raises(ValueError, match="omega"):
        sp.to_csr5(a, 0, 2)
    with pytest.raises(ValueError, match="sigma"):
        sp.to_csr5(a, 4, 0)
    with pytest.raises(ValueError, match="multiple"):
        sp.to_sell(a, 2, 3)
    big = sp.canonicalize([0] * 8 + [1], list(range(8)) + [0], [1.0] * 9, 64, 8)
    with pytest.raises(sp.ConversionError, match="cell"):
        sp.to_ell(big, max_cells=100)
    with pytest.raises(sp.ConversionError, match="cell"):
        sp.to_sell(big, 4, 0, max_cells=10)
    with pytest.raises(ValueError, match="outside"):
        sp.canonicalize([0, 2], [0, 0], [1.0, 1.0], 2, 2)
    with pytest.raises(ValueError, match="outside"):
        sp.canonicalize([0], [-1], [1.0], 2, 2)
    with pytest.raises(ValueError, match="32-bit"):
        sp.canonicalize([], [], [], 2**32, 1)
    with pytest.raises(ValueError, match="undefined"):
        sp.extract_features(sp.canonicalize([], [], [], 0, 5))
    with pytest.raises(ValueError, match="disagree"):
        sp.canonicalize([0, 1], [0], [1.0], 2, 2)
    assert sp.canonicalize([0, 0, 0], [0, 1, 1], [1.0, -1.0, 1.0], 1, 2).data.tolist() == [1.0]


def test_random_sweep_against_oracle(sp, rng):
    for trial in range(40):
        rr, cc, vv, nr, nc = random_triplets(rng, max_dim=300)
        # shuffle + duplicate some entries to exercise the radix sort and sums
        dup = rng.integers(0, max(len(rr), 1), size=len(rr) // 4) if len(rr) else np.empty(0, int)
        rr = np.concatenate([rr, rr[dup]]); cc = np.concatenate([cc, cc[dup]]); vv = np.concatenate([vv, vv[dup]])
        perm = rng.permutation(len(rr))
        rr, cc, vv = rr[perm], cc[perm], vv[perm]
        a = sp.canonicalize(torch.from_numpy(rr).int(), torch.from_numpy(cc).int(), vv, nr, nc)
        orow, ocol, oval = port.canonicalize(rr, cc, vv, nr, nc)
        assert np.array_equal(np_(a.row), orow) and np.array_equal(np_(a.col), ocol)
        assert same_bits(a.data, oval)
        x = rng.normal(size=nc)
        ref = port.dense_spmv_oracle(orow, ocol, oval, nr, x)
        bound = port.dense_spmv_oracle(orow, ocol, np.abs(oval), nr, np.abs(x))
        om = int(rng.choice([1, 2, 4, 8, 16, 32, 3, 5]))
        sg = int(rng.integers(1, 40))
        for tag, kw in [("csr", {}), ("csr5", dict(omega=om, sigma=sg)), ("ell", {}),
                        ("sell", dict(sell_c=int(rng.integers(1, 40)), sell_sigma=0)), ("hyb", {})]:
            m = sp.convert(tag, a, **kw)
            y = sp.spmv(tag, m, x)
            assert_within(y, ref, bound)
            assert sp.coo_equal(sp.to_coo(m), a), (trial, tag)


def test_matrix_market_round_trip(sp, rng):
    demo = ("%%MatrixMarket matrix coordinate real general\n% c\n4 4 8\n1 2 6\n1 3 1\n2 1 2\n2 3 8\n2 4 3\n"
            "3 3 4\n4 2 7\n4 3 5\n")
    a = sp.read_matrix_market(io.BytesIO(demo.encode()))
    assert np_(a.row).tolist() == [0, 0, 1, 1, 1, 2, 3, 3]
    sym = sp.read_matrix_market(b"%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 5\n3 3 7\n")
    assert np_(sym.col).tolist() == [1, 0, 2] and np_(sym.data).tolist() == [5, 5, 7]
    with pytest.raises(sp.MatrixMarketError, match="line 3"):
        sp.read_matrix_market(b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 9\n")
    rr, cc, vv, nr, nc = random_triplets(rng, max_dim=60)
    b = sp.canonicalize(rr, cc, vv, nr, nc)
    buf = io.StringIO()
    sp.write_matrix_market(b, buf)
    assert sp.coo_equal(sp.read_matrix_market(buf.getvalue().encode()), b)


def test_select_format_matches_reference(sp, golden):
    """select_format (model.py:305-319): GPU features -> host tree descent ->
    GPU convert, with a model trained and saved by the reference."""
    model = sp.load_model(io.StringIO(str(golden.d["__model__"])))
    for name in golden.names:
        g = golden.case(name)
        if "predicted" not in g:
            continue
        nr, nc = (int(t) for t in g["shape"])
        a = sp.canonicalize(g["row"], g["col"], g["data"], nr, nc)
        tag, m = sp.select_format(a, model)
        assert tag.value == str(g["predicted"]), name
        assert sp.coo_equal(sp.to_coo(m), a), name


def test_extra_features_against_oracle(sp, rng):
    for _ in range(10):
        rr, cc, vv, nr, nc = random_triplets(rng, max_dim=200)
        a = sp.canonicalize(rr, cc, vv, nr, nc)
        r, c, v = port.canonicalize(rr, cc, vv, nr, nc)
        assert sp.extract_extra_features(a) == port.extra_features(r, c, nr, nc)


@pytest.mark.parametrize("rts", ["0", "1"])
@pytest.mark.parametrize("shape", [(2000, 1500), (1 << 24, 3_000_017)])
def test_canonicalize_many_tiles(sp, rng, monkeypatch, rts, shape):
    """3M shuffled triplets (~730 radix tiles): dense duplicate runs with
    cancellations and signed zeros on a small grid, 6-7 radix passes on a
    large one; both sort schemes (single-pass look-back and, forced by
    SPMVB_RADIX_RTS=1, reduce-then-scan) bit-exact against the oracle."""
    monkeypatch.setenv("SPMVB_RADIX_RTS", rts)
    nr, nc = shape
    n = 3_000_000
    rr = rng.integers(0, nr, n, dtype=np.int64)
    cc = rng.integers(0, nc, n, dtype=np.int64)
    vv = rng.choice([-1.5, -0.5, 0.0, -0.0, 0.25, 0.5, 1.5], size=n) + rng.integers(0, 2, n) * rng.normal(size=n)
    a = sp.canonicalize(torch.from_numpy(rr).int().cuda(), torch.from_numpy(cc).int().cuda(),
                        torch.from_numpy(vv).cuda(), nr, nc)
    orow, ocol, oval = port.canonicalize(rr, cc, vv, nr, nc)
    assert np.array_equal(np_(a.row), orow) and np.array_equal(np_(a.col), ocol)
    assert same_bits(a.data, oval)


def test_wide_rows_sell_hyb(sp, rng):
    """Rows far wider than the SELL wide-slice threshold (256 columns) and
    the per-row copy limit (LONG_ROW = 512) next to short and empty rows:
    SELL grids (flat storage, several c/sigma) and the HYB ELL part and tail
    bit-exact against the oracle; SpMV within tolerance."""
    n, nc = 700, 6000
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(600, 3000)) if r % 97 == 5 else int(rng.integers(0, 12))
        cs = np.sort(rng.choice(nc, size=k, replace=False))
        rows.append(np.full(k, r)); cols.append(cs)
    rr, cc = np.concatenate(rows), np.concatenate(cols)
    vv = rng.normal(size=rr.size)
    a = sp.canonicalize(torch.from_numpy(rr).int(), torch.from_numpy(cc).int(), vv, n, nc)
    orow, ocol, oval = port.canonicalize(rr, cc, vv, n, nc)
    optr, oind, odat = port.to_csr(orow, ocol, oval, n)
    x = rng.normal(size=nc)
    ref = port.dense_spmv_oracle(orow, ocol, oval, n, x)
    bound = port.dense_spmv_oracle(orow, ocol, np.abs(oval), n, np.abs(x))
    for c_, s_ in [(4, 0), (32, 0), (32, 64), (100, 0), (7, 7 * 20)]:
        so = port.to_sell(optr, oind, odat, n, c_, s_, max_cells=1 << 30)
        ms = sp.to_sell(a, c_, s_, max_cells=1 << 30)
        assert np.array_equal(np_(ms.perm), so.perm) and np.array_equal(np_(ms.widths), so.widths)
        assert np.array_equal(np_(ms.flat_indices), so.flat_indices), (c_, s_)
        assert np_(ms.flat_data).tobytes() == so.flat_data.tobytes(), (c_, s_)
        assert_within(sp.spmv("sell", ms, x), ref, bound)
        assert sp.coo_equal(sp.to_coo(ms), a), (c_, s_)
    K, hi, hd, hn, tail = port.to_hyb(orow, ocol, oval, n)
    mh = sp.to_hyb(a)
    assert mh.k == K and np.array_equal(np_(mh.ell.indices), hi) and np_(mh.ell.data).tobytes() == hd.tobytes()
    assert np.array_equal(np_(mh.coo_tail.row), tail[0]) and np.array_equal(np_(mh.coo_tail.col), tail[1])
    assert np_(mh.coo_tail.data).tobytes() == tail[2].tobytes()
    assert_within(sp.spmv("hyb", mh, x), ref, bound)
    assert sp.coo_equal(sp.to_coo(mh), a)
    assert sp.coo_equal(sp.to_coo(sp.to_csr(a)), a) and sp.coo_equal(sp.to_coo(sp.to_csr5(a, 32, 16)), a)


@pytest.mark.parametrize("n_rows", [(1 << 24) + 5, (1 << 25) + 3, (1 << 26) + 11])
def test_features_many_rows(sp, rng, n_rows):
    """Row counts past 2^24 (the depth-13 pairwise combine needs 64 KB of
    shared memory): all 8 features bit-identical to numpy."""
    nnz = 2_000_000
    rr = np.sort(rng.integers(0, n_rows, nnz))
    cc = rng.integers(0, 1000, nnz)
    a = sp.canonicalize(torch.from_numpy(rr).int().cuda(), torch.from_numpy(cc).int().cuda(),
                        torch.ones(nnz, dtype=torch.float64, device="cuda"), n_rows, 1000)
    r, c, v = port.canonicalize(rr, cc, np.ones(nnz), n_rows, 1000)
    got = sp.extract_features(a).as_array()
    want = np.array(port.extract_features(r, n_rows, 1000), dtype=np.float64)
    assert got.tobytes() == want.tobytes(), (got, want)


@pytest.mark.parametrize("tag,kw", [("csr5", dict(omega=32, sigma=16)), ("csr", {}), ("hyb", {}), ("sell", dict(sell_c=32))])
def test_spmv_many_pipelined_matches_single_calls(sp, rng, tag, kw):
    """spmv_many (host vectors, transfers pipelined across vectors on two
    device buffer pairs) == spmv(..., out=) one call at a time, bit for bit."""
    rr, cc, vv, nr, nc = random_triplets(rng, max_dim=3000)
    a = sp.canonicalize(rr, cc, vv, nr, nc)
    m = sp.convert(tag, a, **kw)
    xs = [torch.from_numpy(rng.normal(size=nc)).pin_memory() for _ in range(5)]
    ys = [torch.full((nr,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(5)]
    out = sp.spmv_many(tag, m, xs, ys, ranges=4)
    assert len(out) == len(ys) and all(o is y for o, y in zip(out, ys))
    for xh, yh in zip(xs, ys):
        want = sp.spmv(tag, m, xh.cuda()).cpu()
        assert yh.numpy().tobytes() == want.numpy().tobytes()
    with pytest.raises(ValueError, match="pinned"):
        sp.spmv_many(tag, m, [xs[0].clone()], [ys[0]])


def test_new_entry_points_on_degenerate_shapes(sp):
    """Empty matrices / empty rows through to_coo, spmv_many and the fused
    push: zeros where the reference gives zeros, no out-of-bounds work."""
    for nr, nc in [(3, 3), (5, 0), (0, 4), (1, 1)]:
        rr = np.array([0]) if (nr, nc) == (1, 1) else np.empty(0, dtype=np.int64)
        a = sp.canonicalize(rr, rr.copy(), np.ones(rr.size), nr, nc)
        for tag, kw in [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("ell", {}), ("sell", dict(sell_c=4)),
                        ("hyb", {})]:
            m = sp.convert(tag, a, **kw)
            assert sp.coo_equal(sp.to_coo(m), a), (nr, nc, tag)
            xs = [torch.ones(nc, dtype=torch.float64).pin_memory() for _ in range(3)]
            ys = [torch.full((nr,), 7.0, dtype=torch.float64).pin_memory() for _ in range(3)]
            sp.spmv_many(tag, m, xs, ys)
            want = sp.spmv(tag, m, torch.ones(nc, dtype=torch.float64, device="cuda")).cpu()
            for y in ys:
                assert y.numpy().tobytes() == want.numpy().tobytes(), (nr, nc, tag)
        if nr > 0 and nc > 0:
            m5 = sp.to_csr5(a, 32, 16)
            peer = torch.full((nr + 2,), -1.0, dtype=torch.float64, device="cuda")
            ptrs = torch.tensor([peer.data_ptr()], dtype=torch.int64, device="cuda")
            y = sp.spmv_csr5_push(m5, torch.ones(nc, dtype=torch.float64, device="cuda"), None, ptrs, 1)
            torch.cuda.synchronize()
            assert peer[1:nr + 1].cpu().numpy().tobytes() == y.cpu().numpy().tobytes()
            assert float(peer[0]) == -1.0 and float(peer[nr + 1]) == -1.0
