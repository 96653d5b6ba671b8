"""Non-finite values follow the reference: canonicalize
drops only sums equal to +-0.0 -- NaN and +-inf entries, and duplicates that
sum to them, are KEPT -- and every SpMV propagates them as numpy does,
including through the padded slots of ELL / SELL / HYB (a pad is 0.0 times
x at the row's last column: NaN when that x entry is infinite).  NaN payload
bits differ between x86 and the GPU, so NaN positions are compared as a mask
and everything else bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def same_with_nan_mask(got, want) -> bool:
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    if got.shape != want.shape or not np.array_equal(np.isnan(got), np.isnan(want)):
        return False
    ok = ~np.isnan(want)
    return got[ok].tobytes() == want[ok].tobytes()


def test_canonicalize_keeps_nan_and_inf(sp):
    inf, nan = float("inf"), float("nan")
    r = np.array([0, 0, 1, 1, 2, 2, 3, 4, 4, 5, 5, 6, 6, 6, 7])
    c = np.array([0, 0, 1, 1, 2, 2, 3, 4, 4, 5, 5, 6, 6, 6, 7])
    v = np.array([inf, -inf,      # -> nan: kept
                  nan, 1.0,       # -> nan: kept
                  inf, 1.0,       # -> inf: kept
                  -0.0,           # dropped
                  1.5, -1.5,      # cancels: dropped
                  -inf, -inf,     # -> -inf: kept
                  1e308, 1e308, 1e308,  # overflows to inf: kept
                  nan])           # a lone NaN: kept, payload untouched
    with np.errstate(all="ignore"):
        want_r, want_c, want_v = port.canonicalize(r, c, v, 8, 8)
    assert want_r.tolist() == [0, 1, 2, 5, 6, 7]
    a = sp.canonicalize(r, c, v, 8, 8)
    assert np.array_equal(a.row.cpu().numpy(), want_r) and np.array_equal(a.col.cpu().numpy(), want_c)
    assert same_with_nan_mask(a.data.cpu().numpy(), want_v)
    assert a.data.cpu().numpy()[-1:].tobytes() == v[-1:].tobytes()  # no arithmetic on a lone entry


@pytest.mark.parametrize("exact", [False, True])
def test_spmv_propagates_nonfinite_like_numpy(sp, exact):
    rng = np.random.default_rng(21)
    nr, nc = 400, 300
    mask = rng.random((nr, nc)) < 0.04
    mask[7, :] = True                      # a dense row
    mask[20:30, :] = False                 # empty rows
    r, c = np.nonzero(mask)
    v = rng.normal(size=r.size)
    v[rng.choice(v.size, 6, replace=False)] = [np.inf, -np.inf, np.nan, np.inf, 1e308, -1e308]
    x = rng.uniform(-1.0, 1.0, size=nc)
    x[[3, 150, 299]] = [np.inf, np.nan, -np.inf]   # 299: many rows' LAST column -> their pads give 0 * -inf = NaN
    x[10] = 1e308
    a = sp.canonicalize(r, c, v, nr, nc)
    row, col, val = port.canonicalize(r, c, v, nr, nc)
    ptr, ind, dat = port.to_csr(row, col, val, nr)
    xd = torch.from_numpy(x).cuda()
    kw = dict(exact=True) if exact else {}
    with np.errstate(all="ignore"):
        want = {
            "csr": port.spmv_csr(ptr, ind, dat, nr, x),
            "csr5": port.spmv_csr5(port.to_csr5(ptr, ind, dat, nr, 4, 16), nr, x),
            "ell": port.spmv_ell(*port.to_ell(ptr, ind, dat, nr)[:3], x),
            "sell": port.spmv_sell(port.to_sell(ptr, ind, dat, nr, 4, 8), nr, x),
        }
        K, hi, hd, hn, tail = port.to_hyb(row, col, val, nr)
        want["hyb"] = port.spmv_hyb(K, hi, hd, tail, nr, x)
    # the padded formats poison rows the CSR formats leave finite
    assert np.isnan(want["ell"]).sum() > np.isnan(want["csr"]).sum() > 0
    for tag, p in [("csr", {}), ("csr5", dict(omega=4, sigma=16)), ("ell", {}), ("sell", dict(sell_c=4, sell_sigma=8)),
                   ("hyb", {})]:
        y = sp.spmv(tag, sp.convert(tag, a, **p), xd, **kw).cpu().numpy()
        assert np.array_equal(np.isnan(y), np.isnan(want[tag])), tag
        assert np.array_equal(np.isinf(y), np.isinf(want[tag])), tag
        if exact or tag in ("ell", "sell"):
            assert same_with_nan_mask(y, want[tag]), tag
        else:
            ok = np.isfinite(want[tag])
            assert np.allclose(y[ok], want[tag][ok], rtol=1e-12, atol=0.0), tag
