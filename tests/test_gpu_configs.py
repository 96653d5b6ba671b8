"""Parity at the BASELINE.json configuration sizes (GPU).

C1-C3 (host-generated) and C4 (R-MAT on the GPU, regenerated bit for bit on
the host by oracle/synth_ref.py): canonicalize and every conversion
bit-exact against oracle/port.py; SpMV per format within
|y - y_ref| <= 1e-12 (|A| |x|) of the sequential oracle; ELL/SELL
bit-identical.  C5 (5.3e8 nnz) is checked through size-independent
properties on the device: canonical order, cross-format agreement,
exact linearity under power-of-two scaling, repeat bit-identity and the
power-iteration normalisation.
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


def h(t):
    return t.detach().cpu().numpy()


def check_within(y, ref, bound):
    d = np.abs(h(y) - ref)
    assert np.all(d <= TOL * bound), float(np.max(d / np.maximum(bound, 1e-300)))


def host_triplets(name):
    from paper_1805_11938_b200 import synth

    cfg = dict(synth.CONFIGS[name])
    kind = cfg.pop("kind")
    fn = {"laplace2d": synth.laplace2d, "banded": synth.banded, "stencil27": synth.stencil27}[kind]
    return fn(**cfg)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_parity(sp, name):
    if name == "C4":
        from paper_1805_11938_b200 import synth

        cfg = synth.CONFIGS["C4"]
        r, c, v = synth.rmat_triplets(cfg["scale"], cfg["edge_factor"], cfg["seed"])
        hr, hc, hv = synth_ref.rmat(cfg["scale"], cfg["edge_factor"], cfg["seed"])
        assert np.array_equal(h(r), hr) and np.array_equal(h(c), hc) and h(v).tobytes() == hv.tobytes()
        n = 1 << cfg["scale"]
        a = sp.canonicalize(r, c, v, n, n)
        row, col, val = port.canonicalize(hr, hc, hv, n, n)
    else:
        rr, cc, vv, n = host_triplets(name)
        perm = np.random.default_rng(0).permutation(rr.size)  # unsorted input for the GPU sort
        a = sp.canonicalize(rr[perm], cc[perm], vv[perm], n, n)
        row, col, val = port.canonicalize(rr, cc, vv, n, n)
    assert np.array_equal(h(a.row), row) and np.array_equal(h(a.col), col)
    assert h(a.data).tobytes() == val.tobytes()
    ptr, ind, dat = port.to_csr(row, col, val, n)
    x = synth_ref.uniform(n, 17)
    xd = torch.from_numpy(x).cuda()
    ref = port.dense_spmv_oracle(row, col, val, n, x)
    bound = port.dense_spmv_oracle(row, col, np.abs(val), n, np.abs(x))
    assert h(sp.dense_spmv_oracle(a, xd)).tobytes() == ref.tobytes()

    m = sp.to_csr(a)
    assert np.array_equal(h(m.ptr), ptr)
    check_within(sp.spmv("csr", m, xd), ref, bound)
    # exact=True: the reference's own summation order, bit for bit (csrc/spmv_exact.cu)
    assert h(sp.spmv("csr", m, xd, exact=True)).tobytes() == port.spmv_csr(ptr, ind, dat, n, x).tobytes()

    for om, sg in [(4, 16), (32, 16), (32, 8)]:
        m5 = sp.to_csr5(m, om, sg)
        o5 = port.to_csr5(ptr, ind, dat, n, om, sg)
        for f in ("tile_ptr", "bit_flag", "y_off", "seg_off", "indices"):
            assert np.array_equal(h(getattr(m5, f)), getattr(o5, f)), f
        assert h(m5.data).tobytes() == o5.data.tobytes()
        y5 = sp.spmv("csr5", m5, xd)
        check_within(y5, ref, bound)
        assert h(sp.spmv("csr5", m5, xd)).tobytes() == h(y5).tobytes()
        if sg == 16:
            assert h(sp.spmv("csr5", m5, xd, exact=True)).tobytes() == port.spmv_csr5(o5, n, x).tobytes()

    try:
        k, gi, gd, cnt = port.to_ell(ptr, ind, dat, n)
        ell_ok = True
    except port.GridTooLarge:
        ell_ok = False
    if ell_ok:
        me = sp.to_ell(m)
        assert me.k == k and np.array_equal(h(me.indices), gi) and h(me.data.contiguous()).tobytes() == gd.tobytes()
        assert h(sp.spmv("ell", me, xd)).tobytes() == port.spmv_ell(k, gi, gd, x).tobytes()
    else:
        with pytest.raises(sp.ConversionError, match="cell"):
            sp.to_ell(m)

    for c_, s_ in [(4, 0), (32, 1024)]:
        try:
            so = port.to_sell(ptr, ind, dat, n, c_, s_)
        except port.GridTooLarge:
            with pytest.raises(sp.ConversionError, match="cell"):
                sp.to_sell(m, c_, s_)
            continue
        ms = sp.to_sell(m, c_, s_)
        assert np.array_equal(h(ms.perm), so.perm) and np.array_equal(h(ms.widths), so.widths)
        flat = np.concatenate([d.ravel(order="F") for d in so.data])
        assert h(ms.flat_data).tobytes() == flat.tobytes()
        assert np.array_equal(h(ms.flat_indices), so.flat_indices)
        ys = sp.spmv("sell", ms, xd)
        if int(so.widths.max()) <= 256:  # every slice summed sequentially: bit-identical
            assert h(ys).tobytes() == port.spmv_sell(so, n, x).tobytes()
        else:  # wide power-law slices are split across a CTA (SPMVB_SELL_WIDE_COLS)
            check_within(ys, ref, bound)
            assert h(sp.spmv("sell", ms, xd, exact=True)).tobytes() == port.spmv_sell(so, n, x).tobytes()

    K, hi, hd, hn, tail = port.to_hyb(row, col, val, n)
    mh = sp.to_hyb(m)
    assert mh.k == K and np.array_equal(h(mh.ell.indices), hi)
    assert h(mh.ell.data.contiguous()).tobytes() == hd.tobytes()
    assert np.array_equal(h(mh.ell.row_nnz), hn)
    assert np.array_equal(h(mh.coo_tail.row), tail[0]) and np.array_equal(h(mh.coo_tail.col), tail[1])
    assert h(mh.coo_tail.data).tobytes() == tail[2].tobytes()
    check_within(sp.spmv("hyb", mh, xd), ref, bound)
    assert h(sp.spmv("hyb", mh, xd, exact=True)).tobytes() == port.spmv_hyb(K, hi, hd, tail, n, x).tobytes()

    f = sp.extract_features(m)
    assert f.as_array().tobytes() == np.array(port.extract_features(row, n, n)).tobytes()
    assert sp.coo_equal(sp.to_coo(sp.to_csr5(m, 32, 16)), a)


def test_c3_power_iteration(sp):
    """C3: 100 power-iteration steps x <- A x / ||A x|| (BASELINE configs[2])."""
    from paper_1805_11938_b200 import dist as spdist

    rr, cc, vv, n = host_triplets("C3")
    a = sp.canonicalize(rr, cc, vv, n, n)
    m = sp.to_csr5(a, 32, 16)
    x0 = torch.from_numpy(synth_ref.uniform(n, 23)).cuda()
    pi = spdist.PowerIteration(lambda x, out, s: sp.spmv("csr5", m, x, out=out, scale=s), [0, n], 0, 1,
                               torch.device("cuda"), x0)
    for _ in range(100):
        pi.step()
    row, col, val = port.canonicalize(rr, cc, vv, n, n)
    ptr, ind, dat = port.to_csr(row, col, val, n)
    x = synth_ref.uniform(n, 23)
    scale = 1.0
    for _ in range(100):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    np.testing.assert_allclose(h(pi.x), x, rtol=1e-9, atol=1e-12 * np.abs(x).max())
    assert float(pi.scale.item()) == pytest.approx(scale, rel=1e-12)


def test_c5_properties(sp):
    """C5 at full size (5.3e8 nnz) through size-independent properties."""
    from paper_1805_11938_b200 import synth

    cfg = synth.CONFIGS["C5"]
    r, c, v = synth.rmat_triplets(cfg["scale"], cfg["edge_factor"], cfg["seed"])
    n = 1 << cfg["scale"]
    a = sp.canonicalize(r, c, v, n, n)
    del r, c, v
    key = a.row.to(torch.int64) * n + a.col.to(torch.int64)
    assert bool((key[1:] > key[:-1]).all())  # strictly increasing: sorted and unique
    assert bool((a.data > 0).all()) and bool((a.data <= 1).all())
    # the first 4096 draws, regenerated on the host, are entries of A with
    # the value of their first occurrence
    hr, hc, hv = synth_ref.rmat_draws(cfg["scale"], cfg["edge_factor"] << cfg["scale"], cfg["seed"], lo=0, hi=4096)
    hk = hr * n + hc
    _, first = np.unique(hk, return_index=True)
    q = torch.from_numpy(hk[first]).cuda()
    pos = torch.searchsorted(key, q)
    assert bool(torch.equal(key[pos], q))
    assert h(a.data[pos]).tobytes() == hv[first].tobytes()
    del key, q, pos
    m = sp.to_csr(a)
    x = synth.uniform_vector(n, 29)
    ref = sp.dense_spmv_oracle(a, x)  # GPU restatement of coo.py:128-141 (bit-exact at small sizes)
    absA = sp.CooMatrix(a.n_rows, a.n_cols, a.row, a.col, a.data.abs())
    bound = sp.dense_spmv_oracle(absA, x.abs())
    del a, absA
    for tag, kw in [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("hyb", {})]:
        mm = sp.convert(tag, m, **kw)
        y = sp.spmv(tag, mm, x)
        assert bool(((y - ref).abs() <= TOL * bound).all()), tag
        y2 = sp.spmv(tag, mm, 2.0 * x)  # linearity under an exact scaling
        assert bool(torch.equal(y2, 2.0 * y)), tag
        assert bool(torch.equal(sp.spmv(tag, mm, x), y)), tag  # repeat bit-identity
        del mm, y, y2
        torch.cuda.empty_cache()
