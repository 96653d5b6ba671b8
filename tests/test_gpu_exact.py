"""``exact=True``: the reference-order SpMV kernels (csrc/spmv_exact.cu).

Bar: bit-identical to the y the reference itself produced
(tests/golden/cases.npz: ``csr/y``, ``csr5_*/y``, ``hyb/y``, ``sell_*/y``,
``ell/y``, written by spmvkit.spmv in tests/golden/make_golden.py) and, on
matrices with rows long enough for the CTA-per-row kernels (numpy's pairwise
tree cut at several depths, rows spanning thousands of CSR5 tiles, long HYB
tails, SELL slices past the wide threshold), to oracle/port.py, which is
pinned to the reference.  The full-size configs are covered in
test_gpu_configs.py.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu

CSR5_PARAMS = [(2, 2), (4, 16), (32, 16), (3, 5), (4, 3), (1, 1), (8, 4), (16, 2)]
SELL_PARAMS = [(4, 0), (2, 4), (3, 0), (4, 8), (32, 64), (1, 0), (2, 2)]


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def bits(t) -> bytes:
    a = t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return np.asarray(a, dtype=np.float64).tobytes()


def test_exact_equals_the_reference_outputs(sp, golden):
    for name in golden.names:
        g = golden.case(name)
        nr, nc = (int(t) for t in g["shape"])
        a = sp.canonicalize(g["in_row"], g["in_col"], g["in_val"], nr, nc)
        x = torch.from_numpy(g["x"]).cuda()
        assert bits(sp.spmv("csr", sp.to_csr(a), x, exact=True)) == bits(g["csr/y"]), name
        for om, sg in CSR5_PARAMS:
            y5 = sp.spmv("csr5", sp.to_csr5(a, om, sg), x, exact=True)
            assert bits(y5) == bits(g[f"csr5_{om}_{sg}/y"]), (name, om, sg)
        if int(g["ell/k"]) >= 0:
            assert bits(sp.spmv("ell", sp.to_ell(a), x, exact=True)) == bits(g["ell/y"]), name
        for cc, ss in SELL_PARAMS:
            ys = sp.spmv("sell", sp.to_sell(a, cc, ss), x, exact=True)
            assert bits(ys) == bits(g[f"sell_{cc}_{ss}/y"]), (name, cc, ss)
        assert bits(sp.spmv("hyb", sp.to_hyb(a), x, exact=True)) == bits(g["hyb/y"]), name


def long_row_matrix(rng, n_rows=3000, n_cols=300_000):
    """Short random rows plus rows of 257 ... 140001 entries: numpy's pairwise
    tree at depths 1-11 above its 128-element leaves, lengths that are and are
    not multiples of 8, a row of exactly 129 + 1 entries (rest = one leaf past
    the 128 boundary) and empty rows in between."""
    lens = rng.integers(0, 40, size=n_rows)
    lens[rng.random(n_rows) < 0.3] = 0
    for r, L in zip(rng.choice(n_rows, size=14, replace=False),
                    [257, 258, 264, 300, 513, 1025, 2047, 4096, 9999, 20001, 70000, 140001, 130, 129]):
        lens[r] = L
    rows = np.repeat(np.arange(n_rows), lens)
    cols = np.concatenate([np.sort(rng.choice(n_cols, size=int(L), replace=False)) for L in lens if L])
    vals = rng.normal(size=rows.size) * 10.0 ** rng.integers(-8, 9, size=rows.size)  # cancellation-prone
    return rows, cols, vals, n_rows, n_cols


def test_exact_long_rows_against_the_oracle(sp):
    rng = np.random.default_rng(7)
    r, c, v, nr, nc = long_row_matrix(rng)
    a = sp.canonicalize(r, c, v, nr, nc)
    row, col, val = port.canonicalize(r, c, v, nr, nc)
    ptr, ind, dat = port.to_csr(row, col, val, nr)
    x = rng.uniform(-1.0, 1.0, size=nc)
    xd = torch.from_numpy(x).cuda()
    m = sp.to_csr(a)
    want = port.spmv_csr(ptr, ind, dat, nr, x)
    got = sp.spmv("csr", m, xd, exact=True)
    assert bits(got) == bits(want)
    # the default kernel sums in another order: close, not identical, on these rows
    fast = sp.spmv("csr", m, xd).cpu().numpy()
    bound = port.dense_spmv_oracle(row, col, np.abs(val), nr, np.abs(x))
    assert np.all(np.abs(fast - want) <= 1e-12 * bound) and fast.tobytes() != want.tobytes()
    for om, sg in [(4, 16), (32, 16), (32, 8), (3, 5), (1, 1)]:
        o5 = port.to_csr5(ptr, ind, dat, nr, om, sg)
        assert bits(sp.spmv("csr5", sp.to_csr5(m, om, sg), xd, exact=True)) == bits(port.spmv_csr5(o5, nr, x)), (om, sg)
    K, hi, hd, hn, tail = port.to_hyb(row, col, val, nr)
    assert tail[0].size > 140000 - K  # the long rows live in the tail
    assert bits(sp.spmv("hyb", sp.to_hyb(m), xd, exact=True)) == bits(port.spmv_hyb(K, hi, hd, tail, nr, x))
    for cc, ss in [(32, 0), (4, 64)]:
        so = port.to_sell(ptr, ind, dat, nr, cc, ss, max_cells=1 << 34)
        ms = sp.to_sell(m, cc, ss, max_cells=1 << 34)
        assert int(so.widths.max()) > 4096
        assert bits(sp.spmv("sell", ms, xd, exact=True)) == bits(port.spmv_sell(so, nr, x)), (cc, ss)


def test_exact_scale_containers_and_repeat(sp):
    rng = np.random.default_rng(11)
    r, c, v, nr, nc = long_row_matrix(rng, n_rows=500, n_cols=200_000)
    a = sp.canonicalize(r, c, v, nr, nc)
    x = rng.uniform(-1.0, 1.0, size=nc)
    xd = torch.from_numpy(x).cuda()
    s = torch.tensor([0.37], dtype=torch.float64, device="cuda")
    for tag, kw in [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("hyb", {})]:
        m = sp.convert(tag, a, **kw)
        y = sp.spmv(tag, m, xd, exact=True)
        assert bits(sp.spmv(tag, m, xd, exact=True)) == bits(y)          # run to run
        assert bits(sp.spmv(tag, m, x, exact=True)) == bits(y)           # numpy in -> numpy out
        out = torch.empty(nr, dtype=torch.float64, device="cuda")
        assert sp.spmv(tag, m, xd, out=out, exact=True) is out and bits(out) == bits(y)
        assert bits(sp.spmv(tag, m, xd, scale=s, exact=True)) == bits(0.37 * y.cpu().numpy())
        with pytest.raises(ValueError, match="length"):
            sp.spmv(tag, m, np.ones(nc + 1), exact=True)
