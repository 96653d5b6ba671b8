"""Degree-ordered shadow layout (relabel.py / csrc/relabel.cu) and the CSR5
prefix mode it enables (non-empty rows = [0, n_nonempty), empty tail zeroed
without row lookups).

The relabelling is not a reference function: its permutation is checked
against a numpy restatement of the documented order (row empty, -(row
degree + column degree), id), P A P^T against the oracle's canonicalize of
the relabelled triplets (bit-exact), SpMV in the new ids against the
oracle's sequential dense SpMV within the north-star tolerance, and the
relabelled power iteration against the oracle's iteration in the original
ids.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import port, synth_ref

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def np_(t):
    return t.detach().cpu().numpy()


def order_restated(ptr, col, n, key="sum"):
    rowdeg = np.diff(ptr)
    coldeg = np.bincount(col, minlength=n)
    if key == "sum":
        perm = np.lexsort((np.arange(n), -(rowdeg + coldeg), rowdeg == 0))
    else:  # rows in exact descending length, then column degree
        perm = np.lexsort((np.arange(n), -coldeg, -rowdeg, rowdeg == 0))
    new_id = np.empty(n, np.int64)
    new_id[perm] = np.arange(n)
    return perm, new_id, int((rowdeg > 0).sum())


def rmat_host(scale, ef, seed):
    r, c, v = synth_ref.rmat(scale, ef, seed)
    n = 1 << scale
    return port.canonicalize(r, c, v, n, n) + (n,)


def cases():
    yield "rmat12", rmat_host(12, 8, 11)
    rng = np.random.default_rng(5)
    n = 300
    flat = rng.choice(n * n, size=2500, replace=False)
    r, c = flat // n, flat % n
    keep = (r % 7 != 3) & (c % 11 != 0)  # empty rows and empty columns
    yield "random_empties", port.canonicalize(r[keep], c[keep], rng.normal(size=int(keep.sum())), n, n) + (n,)
    yield "diag1", (np.array([0]), np.array([0]), np.array([2.5]), 1)
    yield "no_entries", (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), 17)


@pytest.mark.parametrize("key", ["sum", "row"])
@pytest.mark.parametrize("name,case", list(cases()), ids=[c[0] for c in cases()])
def test_order_and_shadow_matrix(sp, name, case, key):
    row, col, val, n = case
    a = sp.canonicalize(row, col, val, n, n)
    csr = sp.to_csr(a)
    order = sp.DegreeOrder(csr, key=key)
    ptr_h = np_(csr.ptr).astype(np.int64)
    perm, new_id, nonempty = order_restated(ptr_h, col.astype(np.int64), n, key)
    assert np_(order.perm).tolist() == perm.tolist()
    assert np_(order.new_id).tolist() == new_id.tolist()
    assert order.n_nonempty == nonempty
    shadow = order.matrix(csr)
    sr, sc, sv = port.canonicalize(new_id[row], new_id[col], val, n, n)
    sptr, sind, sdat = port.to_csr(sr, sc, sv, n)
    assert np_(shadow.ptr).tolist() == sptr.tolist()
    assert np_(shadow.indices).tolist() == sind.tolist()
    assert np_(shadow.data).tobytes() == sdat.tobytes()
    # every empty row is last
    assert np.all(np.diff(sptr)[:nonempty] > 0) and np.all(np.diff(sptr)[nonempty:] == 0)
    x = np.random.default_rng(1).uniform(-1, 1, n)
    xd = torch.from_numpy(x).cuda()
    assert np_(order.to_new(xd)).tobytes() == x[perm].tobytes()
    assert np_(order.to_old(order.to_new(xd))).tobytes() == x.tobytes()


@pytest.mark.parametrize("omega,sigma", [(32, 16), (32, 8), (16, 16), (8, 8), (4, 16), (4, 8), (2, 5), (3, 7)])
def test_prefix_csr5_spmv(sp, omega, sigma):
    """Prefix mode (nonempty_rows None, n_nonempty < n_rows) for every CSR5
    kernel variant: within tolerance of the oracle, the empty tail exactly 0,
    tile ranges and the fused push identical to the single-shot SpMV."""
    row, col, val, n = rmat_host(12, 8, 12)
    a = sp.canonicalize(row, col, val, n, n)
    order = sp.DegreeOrder(a)
    shadow = order.matrix(a)
    m = sp.to_csr5(shadow, omega, sigma)
    assert m.nonempty_rows is None and m.n_nonempty == order.n_nonempty < n
    sco = sp.to_coo(shadow)
    sr, sc, sv = np_(sco.row), np_(sco.col), np_(sco.data)
    x = synth_ref.uniform(n, 9)
    ref = port.dense_spmv_oracle(sr, sc, sv, n, x)
    bound = port.dense_spmv_oracle(sr, sc, np.abs(sv), n, np.abs(x))
    xd = torch.from_numpy(x).cuda()
    y = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")  # stale values must be overwritten
    sp.spmv("csr5", m, xd, out=y)
    yh = np_(y)
    assert np.all(np.abs(yh - ref) <= TOL * bound)
    assert np.all(yh[m.n_nonempty:] == 0.0)
    yr = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    tb, rb = m.range_plan(5)
    for k in range(len(tb) - 1):
        hi = int(rb[k + 1]) if k + 1 < len(tb) - 1 else n
        sp.spmv_csr5_tiles(m, xd, yr, int(tb[k]), int(tb[k + 1]), int(rb[k]), hi)
    assert np_(yr).tobytes() == yh.tobytes()
    if omega == 32 and sigma in (8, 16):
        peers = [torch.full((n + 3,), -1.0, dtype=torch.float64, device="cuda") for _ in range(2)]
        ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device="cuda")
        yp = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
        sp.spmv_csr5_push(m, xd, yp, ptrs, 3)
        torch.cuda.synchronize()
        assert np_(yp).tobytes() == yh.tobytes()
        for p in peers:
            assert np_(p)[3:].tobytes() == yh.tobytes()


def test_relabelled_power_iteration_matches_oracle(sp):
    row, col, val, n = rmat_host(13, 8, 13)
    a = sp.canonicalize(row, col, val, n, n)
    x0 = synth_ref.uniform(n, 21, 0.5, 1.0)
    steps = 25
    x_rel, lam_rel = sp.power_iteration(a, torch.from_numpy(x0).cuda(), steps, "csr5", relabel=True,
                                        omega=32, sigma=16)
    x_pl, lam_pl = sp.power_iteration(a, torch.from_numpy(x0).cuda(), steps, "csr5", relabel=False,
                                      omega=32, sigma=16)
    # oracle: the reference's sequential SpMV, normalised on the host
    xo = x0.copy()
    lam = 0.0
    for k in range(steps):
        y = port.dense_spmv_oracle(row, col, val, n, xo)
        lam = float(np.sqrt(np.dot(y, y)))
        xo = y / lam
    np.testing.assert_allclose(np_(x_rel), xo, rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(np_(x_pl), xo, rtol=1e-9, atol=1e-14)
    assert lam_rel == pytest.approx(lam, rel=1e-12) and lam_pl == pytest.approx(lam, rel=1e-12)
    # tag="auto": the format timed fastest on the shadow layout (relabel) or the plain matrix
    for rel in (True, False):
        x_a, lam_a = sp.power_iteration(a, torch.from_numpy(x0).cuda(), steps, relabel=rel)
        np.testing.assert_allclose(np_(x_a), xo, rtol=1e-9, atol=1e-14)
        assert lam_a == pytest.approx(lam, rel=1e-12)


def test_relabelled_spmv_at_c4(sp):
    """C4 (R-MAT scale 21): the shadow CSR5 SpMV in the new ids within
    tolerance of the on-device sequential oracle of P A P^T, and mapped back
    within tolerance of the plain SpMV."""
    r, c, v = sp.synth.rmat_triplets(21, 10, 104)
    n = 1 << 21
    a = sp.canonicalize(r, c, v, n, n)
    del r, c, v
    rm = sp.RelabelledMatrix("csr5", a, omega=32, sigma=16)
    assert rm.inner.nonempty_rows is None
    x = sp.synth.uniform_vector(n, 204)
    xp = rm.order.to_new(x)
    yp = rm.spmv(xp)
    scoo = sp.to_coo(rm.order.matrix(a))
    ref = sp.dense_spmv_oracle(scoo, xp)
    absm = sp.canonicalize(scoo.row, scoo.col, scoo.data.abs(), n, n)
    bound = sp.dense_spmv_oracle(absm, xp.abs())
    assert bool(((yp - ref).abs() <= TOL * bound).all())
    y_plain = sp.spmv("csr5", sp.to_csr5(a, 32, 16), x)
    y_back = rm.order.to_old(yp)
    bound_o = sp.dense_spmv_oracle(sp.canonicalize(a.row, a.col, a.data.abs(), n, n), x.abs())
    assert bool(((y_back - y_plain).abs() <= 2 * TOL * bound_o).all())


@pytest.mark.parametrize("c,sigma", [(32, 0), (32, 256), (4, 0), (4, 8)])
def test_relabelled_sell_empty_tail(sp, c, sigma):
    """SELL of a degree-ordered matrix: its trailing all-empty slices are
    zeroed without slice/perm lookups (spmvb_spmv_sell tail_from); y is
    bit-identical to the reference SELL recurrence (port.spmv_sell) and
    stale values in the tail are overwritten."""
    row, col, val, n = rmat_host(12, 8, 13)
    a = sp.canonicalize(row, col, val, n, n)
    order = sp.DegreeOrder(a)
    shadow = order.matrix(a)
    m = sp.to_sell(shadow, c, sigma)
    tail = m.wide_plan()[6]
    assert tail < n  # the empty rows form a tail the kernel can skip
    sptr = np_(shadow.ptr).astype(np.int64)
    so = port.to_sell(sptr, np_(shadow.indices).astype(np.int64), np_(shadow.data), n, c, sigma)
    x = synth_ref.uniform(n, 21)
    y = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    sp.spmv("sell", m, torch.from_numpy(x).cuda(), out=y)
    want = port.spmv_sell(so, n, x)
    if int(so.widths.max()) <= 256:
        assert np_(y).tobytes() == want.tobytes()
    assert np.all(np_(y)[order.n_nonempty:] == 0.0)


@pytest.mark.parametrize("c,sigma,k", [(32, 256, 4), (32, 0, 5), (4, 8, 3), (8, 64, 7)])
def test_sell_ranges_bit_identical(sp, c, sigma, k):
    """spmv_sell_range over every range of a plan (any order) == one SELL
    SpMV, bit for bit; each range's rows are a contiguous block (ranges are
    aligned to the sigma windows).  Degree-ordered and reference layouts."""
    row, col, val, n = rmat_host(13, 8, 19)
    a = sp.canonicalize(row, col, val, n, n)
    for mat in (a, sp.DegreeOrder(a).matrix(a)):
        m = sp.to_sell(mat, c, sigma)
        x = torch.from_numpy(synth_ref.uniform(n, 3)).cuda()
        s = torch.full((1,), 0.5, dtype=torch.float64, device="cuda")
        want = sp.spmv("sell", m, x, scale=s)
        plan = m.range_plan(k)
        assert plan[0][6] == 0 and plan[-1][7] == n
        assert all(plan[i][7] == plan[i + 1][6] for i in range(len(plan) - 1))
        y = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
        for r in plan[::-1]:
            sp.spmv_sell_range(m, x, y, r, scale=s)
        assert torch.equal(y, want)
        if sigma:
            perm = np_(m.perm)
            for r in plan:  # a range's permuted rows are its own rows
                assert sorted(perm[r[6]:r[7]].tolist()) == list(range(r[6], r[7]))


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_dealt_order_blocks(sp, parts):
    """DegreeOrder(parts=P) (the multi-GPU form): the degree-sorted ids dealt
    round-robin to P contiguous blocks; each block is in sorted order with
    its empty rows last, blocks are nnz-balanced to within one row, and the
    SpMV of the dealt matrix maps back to A x within tolerance."""
    row, col, val, n = rmat_host(12, 8, 23)
    a = sp.canonicalize(row, col, val, n, n)
    csr = sp.to_csr(a)
    one = sp.DegreeOrder(csr)
    dealt = sp.DegreeOrder(csr, parts=parts)
    sorted_old = np_(one.perm)  # old ids in degree order
    b = dealt.part_bounds
    assert b[0] == 0 and b[-1] == n and len(b) == parts + 1
    perm = np_(dealt.perm)
    for p in range(parts):
        assert perm[b[p]:b[p + 1]].tolist() == sorted_old[p::parts].tolist()
    new_id = np_(dealt.new_id)
    assert np.array_equal(new_id[perm], np.arange(n))
    m = dealt.matrix(csr)
    rowdeg = np.diff(np_(m.ptr))
    nnz = [int(rowdeg[b[p]:b[p + 1]].sum()) for p in range(parts)]
    assert max(nnz) - min(nnz) <= int(rowdeg.max())
    for p in range(parts):  # empty rows last within each block
        d = rowdeg[b[p]:b[p + 1]]
        k = int((d > 0).sum())
        assert np.all(d[:k] > 0) and np.all(d[k:] == 0)
    x = synth_ref.uniform(n, 5)
    ref = port.dense_spmv_oracle(row, col, val, n, x)
    bound = port.dense_spmv_oracle(row, col, np.abs(val), n, np.abs(x))
    xd = torch.from_numpy(x).cuda()
    for tag, kw in [("csr5", dict(omega=32, sigma=8)), ("sell", dict(sell_c=32, sell_sigma=0))]:
        y = dealt.to_old(sp.spmv(tag, sp.convert(tag, m, **kw), dealt.to_new(xd)))
        assert np.all(np.abs(np_(y) - ref) <= TOL * bound), tag
