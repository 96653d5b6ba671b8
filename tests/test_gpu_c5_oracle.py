"""C5 (the headline config, R-MAT scale 25, 5.29e8 nnz) pinned to the CPU oracle.

The full C5 matrix is too large for the numpy oracle, so the host
regenerates parts of it independently (oracle/rmat_sample.c re-runs the GPU
generator's counter hash; oracle/cpu_baseline.rmat_row_subset dedups and
canonicalizes with oracle/port.py) and the GPU result is compared there:

* a hashed 1/64 row sample (~5e5 rows, ~8e6 nnz): the canonical CSR rows
  bit-exact; y = A x at those rows for CSR, CSR5 (omega 32 and the
  reference default omega 4, sigma 16), HYB and SELL-32 within the north-star
  tolerance |y - y_ref| <= 1e-12 (|A| |x|) of port.dense_spmv_oracle
  (coo.py:128-141) with the full-length x; the HYB ELL rows (indices, data,
  row_nnz) and tail rows bit-exact (formats.py:361-397);
* three CSR5 tile windows (the first tiles, the middle, the trailing partial
  tile): every rows of the window regenerated on the host, rebased to a CSR
  that starts at the window's first entry, and port.to_csr5
  (formats.py:196-250) run on it; tile_ptr, bit_flag, y_off, seg_off,
  indices and data of the GPU conversion are bit-exact against it.  y_off
  and seg_off are not read by the SpMV kernel, so only this check covers
  them at C5 scale;
* the headline power-iteration path itself: the degree-ordered shadow layout
  in the format bench.py times (SELL-32 sigma 0 with the 4096-column
  wide-slice threshold and the empty-tail path; CSR5 omega 32 sigma 8),
  mapped back through the permutation, y at the sampled rows within the
  same tolerance.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import cpu_baseline, port, synth_ref

pytestmark = pytest.mark.gpu

TOL = 1e-12
KEEP_MOD = 64


def h(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def c5():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import synth

    cfg = synth.CONFIGS["C5"]
    scale, ef, seed = cfg["scale"], cfg["edge_factor"], cfg["seed"]
    n = 1 << scale
    r, c, v = synth.rmat_triplets(scale, ef, seed)
    a = sp.canonicalize(r, c, v, n, n)
    del r, c, v
    m = sp.to_csr(a)
    del a
    torch.cuda.empty_cache()
    x = synth.uniform_vector(n, 31)
    hx = synth_ref.uniform(n, 31)
    assert h(x).tobytes() == hx.tobytes()
    return dict(sp=sp, scale=scale, ef=ef, seed=seed, n=n, m=m, x=x, hx=hx)


def _windows(tile_ptr, T, n):
    """(t0, t1, r0, r1): first, middle and trailing tile windows with the
    rows [r0, r1) that hold their entries."""
    out = []
    for t0, t1 in [(0, min(3, T)), (max(T // 2 - 1, 0), min(T // 2 + 2, T)), (max(T - 3, 0), T)]:
        r0 = int(tile_ptr[t0])
        r1 = n if t1 == T else min(n, int(tile_ptr[t1]) + 1)
        out.append((t0, t1, r0, r1))
    return out


def _host(c5, ranges):
    return cpu_baseline.rmat_row_subset(c5["scale"], c5["ef"], c5["seed"], KEEP_MOD, ranges)


@pytest.fixture(scope="module")
def host(c5):
    sp, m = c5["sp"], c5["m"]
    m5 = sp.to_csr5(m, 32, 16)
    tp = h(m5.tile_ptr)
    wins = {32: _windows(tp, m5.num_tiles, c5["n"])}
    del m5
    torch.cuda.empty_cache()
    m4 = sp.to_csr5(m, 4, 16)
    wins[4] = _windows(h(m4.tile_ptr), m4.num_tiles, c5["n"])
    del m4
    m8 = sp.to_csr5(m, 32, 8)
    wins[(32, 8)] = _windows(h(m8.tile_ptr), m8.num_tiles, c5["n"])
    del m8
    torch.cuda.empty_cache()
    ranges = sorted({(r0, r1) for w in wins.values() for _, _, r0, r1 in w})
    rows, ptr, ind, dat = _host(c5, ranges)
    sampled = cpu_baseline.kept_rows(c5["n"], KEEP_MOD)
    return dict(rows=rows, ptr=ptr, ind=ind, dat=dat, sampled=sampled, wins=wins)


def _rows_of(host, want):
    """Host CSR (ptr, ind, dat) of the global rows ``want`` (ascending, all present)."""
    k = np.searchsorted(host["rows"], want)
    assert np.array_equal(host["rows"][k], want)
    cnt = host["ptr"][k + 1] - host["ptr"][k]
    ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    pos = np.repeat(host["ptr"][k] - ptr[:-1], cnt) + np.arange(int(ptr[-1]))
    return ptr, host["ind"][pos], host["dat"][pos]


def _device_rows(dptr, rows, cnt, *arrays):
    """Entries of the device CSR rows ``rows`` (whose lengths are ``cnt``)."""
    starts = torch.from_numpy(dptr[rows].astype(np.int64)).cuda()
    cd = torch.from_numpy(cnt).cuda()
    base = torch.repeat_interleave(starts - torch.cumsum(cd, 0) + cd, cd)
    pos = base + torch.arange(int(cnt.sum()), device="cuda")
    return [h(t[pos]) for t in arrays]


def test_c5_sampled_rows_bit_exact(c5, host):
    m = c5["m"]
    dptr = h(m.ptr).astype(np.int64)
    assert int(dptr[-1]) == m.nnz
    rows = host["sampled"]
    ptr, ind, dat = _rows_of(host, rows)
    cnt = np.diff(ptr)
    assert np.array_equal(dptr[rows + 1] - dptr[rows], cnt)
    gi, gd = _device_rows(dptr, rows, cnt, m.indices, m.data)
    assert np.array_equal(gi, ind)
    assert gd.tobytes() == dat.tobytes()
    # every row of the tile windows too
    for r0, r1 in sorted({(r0, r1) for w in host["wins"].values() for _, _, r0, r1 in w}):
        wr = np.arange(r0, r1)
        wp, wi, wd = _rows_of(host, wr)
        assert np.array_equal(dptr[r0 + 1:r1 + 1] - dptr[r0:r1], np.diff(wp))
        gi, gd = _device_rows(dptr, wr, np.diff(wp), m.indices, m.data)
        assert np.array_equal(gi, wi) and gd.tobytes() == wd.tobytes()


@pytest.mark.parametrize("omega,sigma", [(32, 16), (4, 16), (32, 8)])
def test_c5_csr5_tile_windows(c5, host, omega, sigma):
    sp, m = c5["sp"], c5["m"]
    tile = omega * sigma
    m5 = sp.to_csr5(m, omega, sigma)
    T = m5.num_tiles
    dptr = h(m.ptr).astype(np.int64)
    for t0, t1, r0, r1 in host["wins"][omega if sigma == 16 else (omega, sigma)]:
        wptr, wind, wdat = _rows_of(host, np.arange(r0, r1))
        p0, p1 = t0 * tile, min(t1 * tile, m.nnz)
        o = p0 - int(dptr[r0])
        assert 0 <= o < max(int(wptr[-1]), 1)
        W = p1 - p0
        sub_ptr = np.clip(wptr - o, 0, W)
        o5 = port.to_csr5(sub_ptr, wind[o:o + W], wdat[o:o + W], r1 - r0, omega, sigma)
        assert o5.num_tiles == t1 - t0
        got_tp = h(m5.tile_ptr[t0:t1]).astype(np.int64)
        assert np.array_equal(got_tp, o5.tile_ptr[:-1] + r0), (omega, t0)
        if t1 == T:
            assert int(m5.tile_ptr[T]) == c5["n"]
        assert np.array_equal(h(m5.bit_flag[p0:p1]).astype(bool), o5.bit_flag), (omega, t0)
        assert np.array_equal(h(m5.y_off[t0:t1]), o5.y_off), (omega, t0)
        assert np.array_equal(h(m5.seg_off[t0:t1]), o5.seg_off), (omega, t0)
        assert np.array_equal(h(m5.indices[p0:p1]), o5.indices), (omega, t0)
        assert h(m5.data[p0:p1]).tobytes() == o5.data.tobytes(), (omega, t0)


@pytest.fixture(scope="module")
def y_ref(c5, host):
    rows = host["sampled"]
    ptr, ind, dat = _rows_of(host, rows)
    lr = np.repeat(np.arange(rows.size), np.diff(ptr))
    ref = port.dense_spmv_oracle(lr, ind, dat, rows.size, c5["hx"])
    bound = port.dense_spmv_oracle(lr, ind, np.abs(dat), rows.size, np.abs(c5["hx"]))
    return rows, ref, bound


@pytest.mark.parametrize("tag,kw", [
    ("csr", {}),
    ("csr5", dict(omega=32, sigma=16)),
    ("csr5", dict(omega=4, sigma=16)),
    ("hyb", {}),
    ("sell", dict(sell_c=32, sell_sigma=32 * 256, max_cells=1 << 34)),
])
def test_c5_spmv_sampled_rows(c5, y_ref, tag, kw):
    sp = c5["sp"]
    rows, ref, bound = y_ref
    mm = sp.convert(tag, c5["m"], **kw)
    y = sp.spmv(tag, mm, c5["x"])
    got = h(y[torch.from_numpy(rows).cuda()])
    err = np.abs(got - ref)
    assert np.all(err <= TOL * bound), (tag, kw, float(np.max(err / np.maximum(bound, 1e-300))))
    del mm, y
    torch.cuda.empty_cache()


def test_c5_hyb_rows(c5, host):
    sp = c5["sp"]
    mh = sp.to_hyb(c5["m"])
    K = mh.k
    rows = host["sampled"]
    ptr, ind, dat = _rows_of(host, rows)
    cnt = np.diff(ptr)
    # K = hyb_typical_k of the full histogram (formats.py:347-358), recomputed
    # on the host from the device counts (themselves checked at the sampled rows)
    dcnt = np.diff(h(c5["m"].ptr).astype(np.int64))
    assert K == port.hyb_typical_k(dcnt)
    rd = torch.from_numpy(rows).cuda()
    gi = h(mh.ell.indices[rd])
    gd = h(mh.ell.data[rd])
    ec = np.minimum(cnt, K)
    assert np.array_equal(h(mh.ell.row_nnz[rd]), ec)
    eptr = np.concatenate([[0], np.cumsum(ec)])
    keep = (np.arange(ind.size) - np.repeat(ptr[:-1], cnt)) < K
    ei, ed = port._grids(rows.size, K, ec, eptr, ind[keep], dat[keep], 1 << 62)
    assert np.array_equal(gi, ei)
    assert gd.tobytes() == ed.tobytes()
    # tail rows: the remaining entries in canonical order
    tptr = h(mh.tail_ptr).astype(np.int64)
    tc = cnt - ec
    assert np.array_equal(tptr[rows + 1] - tptr[rows], tc)
    tr, tcol, tval = _device_rows(tptr, rows, tc, mh.coo_tail.row, mh.coo_tail.col, mh.coo_tail.data)
    assert np.array_equal(tr, np.repeat(rows, tc))
    assert np.array_equal(tcol, ind[~keep])
    assert tval.tobytes() == dat[~keep].tobytes()


@pytest.mark.parametrize("tag,kw", [
    ("sell", dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),  # the headline power-iteration format
    ("csr5", dict(omega=32, sigma=8)),
])
def test_c5_shadow_layout_spmv_sampled_rows(c5, y_ref, tag, kw):
    """The power-iteration path itself: the degree-ordered shadow layout
    (DegreeOrder, P A P^T, x' = P x) in the format bench.py times (SELL-32
    with the large wide-slice threshold and the empty-tail fast path), mapped
    back with P^T: y at the sampled rows within tolerance of the oracle."""
    sp = c5["sp"]
    rows, ref, bound = y_ref
    order = sp.DegreeOrder(c5["m"])
    rm = sp.convert(tag, order.matrix(c5["m"]), **kw)
    if tag == "sell":
        _, n_wide, _, _, _, wide_cols, tail_from = rm.wide_plan()[:7]
        assert wide_cols == 4096 and n_wide > 0 and tail_from == -(-order.n_nonempty // 32) * 32
    y = order.to_old(sp.spmv(tag, rm, order.to_new(c5["x"])))
    got = h(y[torch.from_numpy(rows).cuda()])
    err = np.abs(got - ref)
    assert np.all(err <= TOL * bound), (tag, float(np.max(err / np.maximum(bound, 1e-300))))
    del rm, y, order
    torch.cuda.empty_cache()


def test_c5_exact_mode_sampled_rows(c5, host):
    """exact=True at C5: y at the sampled rows bit-identical to the
    reference's summation orders evaluated on the host copies of those rows
    -- CSR (reduceat: first + pairwise(rest)), CSR5 omega 32 sigma 16 (the
    row's pieces inside each GLOBAL tile, reduceat each, added in tile order)
    and HYB (the sequential ELL part of the first K entries + the bincount
    sum of the rest)."""
    sp, m, hx = c5["sp"], c5["m"], c5["hx"]
    rows = host["sampled"]
    rd = torch.from_numpy(rows).cuda()
    ptr, ind, dat = _rows_of(host, rows)
    cnt = np.diff(ptr)
    live = np.nonzero(cnt)[0]
    prod = dat * hx[ind]
    # CSR
    want = np.zeros(rows.size)
    want[live] = np.add.reduceat(prod, ptr[:-1][live])
    got = h(sp.spmv("csr", m, c5["x"], exact=True)[rd])
    assert got.tobytes() == want.tobytes()
    # CSR5: cut every sampled row at the global tile boundaries
    tile = 32 * 16
    dptr = h(m.ptr).astype(np.int64)
    g0 = dptr[rows]                                     # global CSR position of each row's first entry
    gpos = np.repeat(g0 - ptr[:-1], cnt) + np.arange(prod.size)
    start = np.zeros(prod.size, dtype=bool)
    start[ptr[:-1][live]] = True
    start |= gpos % tile == 0
    starts = np.nonzero(start)[0]
    sums = np.add.reduceat(prod, starts)
    seg_row = np.searchsorted(ptr, starts, side="right") - 1
    want5 = np.zeros(rows.size)
    np.add.at(want5, seg_row, sums)                     # in order: ((0 + s_1) + s_2) + ...
    m5 = sp.to_csr5(m, 32, 16)
    got5 = h(sp.spmv("csr5", m5, c5["x"], exact=True)[rd])
    del m5
    torch.cuda.empty_cache()
    assert got5.tobytes() == want5.tobytes()
    assert (cnt > 3 * tile).any() and want5.tobytes() != want.tobytes()  # rows spanning tiles: the orders differ
    # HYB
    mh = sp.to_hyb(m)
    K = mh.k
    ec = np.minimum(cnt, K)
    keep = (np.arange(ind.size) - np.repeat(ptr[:-1], cnt)) < K
    ei, ed = port._grids(rows.size, K, ec, np.concatenate([[0], np.cumsum(ec)]), ind[keep], dat[keep], 1 << 62)
    wanth = port.spmv_ell(K, ei, ed, hx)
    local = np.repeat(np.arange(rows.size), cnt)
    wanth += np.bincount(local[~keep], weights=prod[~keep], minlength=rows.size)
    goth = h(sp.spmv("hyb", mh, c5["x"], exact=True)[rd])
    assert goth.tobytes() == wanth.tobytes()
