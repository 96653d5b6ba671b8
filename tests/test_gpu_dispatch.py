"""Prepared launches (kernels.bind / SpmvOperator) and the single-process
power-iteration fast path (dist.PowerIteration: bound SpMV + the fused
spmvb_norm_scale): the same kernels, so y is bit-identical to the generic
spmv entry point; the step's normalisation is summed in another fixed order,
so iterates agree with the generic path to rounding and with themselves
bit for bit (eager vs graph replay)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import port, synth_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


FORMATS = [("csr", {}), ("csr5", dict(omega=32, sigma=16)), ("csr5", dict(omega=4, sigma=16)), ("ell", {}),
           ("sell", dict(sell_c=32, sell_sigma=256)), ("sell", dict(sell_c=4, sell_sigma=0)), ("hyb", {})]


def _matrix(sp, kind):
    if kind == "rmat":
        r, c, v = sp.synth.rmat_triplets(12, 8, 5)
        n = 1 << 12
        return sp.canonicalize(r, c, v, n, n)
    return sp.synth.host_coo("C1")


@pytest.mark.parametrize("kind", ["rmat", "laplace"])
@pytest.mark.parametrize("tag,kw", FORMATS)
def test_bind_bit_identical(sp, kind, tag, kw):
    a = _matrix(sp, kind)
    try:
        m = sp.convert(tag, a, **kw)
    except sp.ConversionError:
        pytest.skip("grid too large for this matrix (as the reference)")
    x = sp.synth.uniform_vector(a.n_cols, 9)
    s = torch.full((1,), 0.75, dtype=torch.float64, device="cuda")
    out = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    call = sp.bind(tag, m, x, out, s)
    out.fill_(np.nan)
    call()
    want = sp.spmv(tag, m, x, scale=s)
    assert torch.equal(out, want)
    op = sp.SpmvOperator(tag, m)
    y2 = torch.empty_like(out)
    op(x, y2, s)
    assert torch.equal(y2, want)
    with pytest.raises(ValueError, match="does not match"):
        sp.bind("ell" if tag != "ell" else "csr", m, x, out)
    with pytest.raises(ValueError, match="contiguous float64"):
        sp.bind(tag, m, x[:-1], out)


def test_norm_scale_kernel(sp):
    from paper_1805_11938_b200.dist import GpuOps

    for n in (0, 1, 1000, 1 << 20, (1 << 22) + 3):
        y = sp.synth.uniform_vector(n, 3) if n else torch.empty(0, dtype=torch.float64, device="cuda")
        ss = torch.empty(1, dtype=torch.float64, device="cuda")
        sc = torch.empty(1, dtype=torch.float64, device="cuda")
        call = GpuOps.bind_norm_scale(y, ss, sc)
        call()
        first = (float(ss.item()), float(sc.item()))
        call()  # the ticket was reset: same result again
        assert (float(ss.item()), float(sc.item())) == first
        hy = y.cpu().numpy()
        want = float(np.dot(hy, hy))
        assert first[0] == pytest.approx(want, rel=1e-13, abs=0)
        assert first[1] == (1.0 / np.sqrt(first[0]) if first[0] > 0 else 1.0)


@pytest.mark.parametrize("tag,kw", [("ell", {}), ("csr5", dict(omega=32, sigma=16)), ("hyb", {})])
def test_fast_power_iteration(sp, tag, kw):
    from paper_1805_11938_b200 import dist as spdist

    rr, cc, vv, n = sp.synth.stencil27(g=24, seed=5)
    a = sp.canonicalize(rr, cc, vv, n, n)
    m = sp.convert(tag, a, **kw)
    x0 = torch.from_numpy(synth_ref.uniform(n, 23)).cuda()
    dev = torch.device("cuda")
    fast = spdist.PowerIteration(sp.SpmvOperator(tag, m), [0, n], 0, 1, dev, x0)
    slow = spdist.PowerIteration(lambda x, o, s: sp.spmv(tag, m, x, out=o, scale=s), [0, n], 0, 1, dev, x0)
    assert fast._fast_ok and not slow._fast_ok
    for _ in range(30):
        fast.step()
        slow.step()
    xs = slow.x.cpu().numpy()
    np.testing.assert_allclose(fast.x.cpu().numpy(), xs, rtol=1e-12, atol=1e-13 * np.abs(xs).max())
    assert float(fast.scale.item()) == pytest.approx(float(slow.scale.item()), rel=1e-13)
    # graph replay of the fast path: bit-identical to its eager steps
    g = spdist.PowerIteration(sp.SpmvOperator(tag, m), [0, n], 0, 1, dev, x0)
    g.run(30, graph=True)
    assert torch.equal(g.x, fast.x) and torch.equal(g.scale, fast.scale)
    # against the CPU oracle (reference CSR algorithm)
    row, col, val = port.canonicalize(rr, cc, vv, n, n)
    ptr, ind, dat = port.to_csr(row, col, val, n)
    x, scale = synth_ref.uniform(n, 23), 1.0
    for _ in range(30):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    np.testing.assert_allclose(fast.x.cpu().numpy(), x, rtol=1e-9, atol=1e-12 * np.abs(x).max())


@pytest.mark.parametrize("tag,kw", [("csr5", dict(omega=32, sigma=16)), ("csr5", dict(omega=32, sigma=8)),
                                    ("sell", dict(sell_c=32, sell_sigma=0)), ("sell", dict(sell_c=8, sell_sigma=64))])
def test_bind_range_bit_identical(sp, tag, kw):
    """Prepared row ranges (bind_range, used by the multi-GPU overlap) over a
    range plan == one SpMV, bit for bit."""
    a = _matrix(sp, "rmat")
    m = sp.convert(tag, a, **kw)
    x = sp.synth.uniform_vector(a.n_cols, 9)
    s = torch.full((1,), 1.5, dtype=torch.float64, device="cuda")
    want = sp.spmv(tag, m, x, scale=s)
    if tag == "csr5":
        tb, rb = m.range_plan(4)
        k = len(tb) - 1
        plan = [(int(rb[i]), int(rb[i + 1]) if i + 1 < k else m.n_rows, int(tb[i]), int(tb[i + 1])) for i in range(k)]
    else:
        plan = m.range_plan(4)
    y = torch.full((a.n_rows,), 3.0, dtype=torch.float64, device="cuda")
    calls = [sp.bind_range(tag, m, x, y, r, s) for r in plan[::-1]]
    for c in calls:
        c()
    assert torch.equal(y, want)
    with pytest.raises(ValueError, match="row ranges"):
        sp.bind_range("hyb", sp.to_hyb(a), x, y, plan[0])
