"""Out-of-bounds detection without compute-sanitizer (closed on this GPU
pool: runs under it left GPUs needing a reset).

Every CUDA tensor created through ``torch.empty`` / ``torch.zeros`` /
``torch.full`` / ``torch.empty_like`` while a test runs -- the library's
output and scratch buffers, the matrices' arrays, x and y -- is carved out
of a larger allocation whose guard bands on both sides hold a sentinel (NaN
payload for float64, 0x7f7f7f7f for 32/64-bit integers, 0xA5 for bytes).
The parity tests then run unchanged, and afterwards every guard band must
be intact: a kernel that writes past either end of any of those buffers
fails the test.  A kernel that READS past an end picks up a sentinel: NaN
poisons y and the oracle comparison fails; a sentinel index gathers far out
of range and faults.  (Library-internal stream-ordered temporaries are not
covered; the radix sort's and the conversions' outputs are.)"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import test_gpu_dispatch as tdisp
import test_gpu_exact as texact
import test_gpu_p2p as tp2p
import test_gpu_parity as tpar
import test_gpu_relabel as trel

pytestmark = pytest.mark.gpu

GUARD = 256  # elements on each side (keeps 256-byte alignment for every dtype)
_REAL_EMPTY = torch.empty
_SENT = {torch.float64: float("nan"), torch.float32: float("nan"),
         torch.int32: 0x7F7F7F7F, torch.int64: 0x7F7F7F7F7F7F7F7F, torch.uint8: 0xA5, torch.bool: True,
         torch.int16: 0x7F7F}


class Guards:
    def __init__(self):
        self.live = []  # (base allocation, elements in the view, the guard band's bytes)
        self.checked = 0

    def make(self, shape, dtype, device, fill=None):
        shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list, torch.Size)) else (shape,)))
        n = int(np.prod(shape)) if shape else 1
        base = _REAL_EMPTY(n + 2 * GUARD, dtype=dtype, device=device)
        base.fill_(_SENT.get(dtype, 0))
        head = base[:GUARD].clone()
        view = base[GUARD:GUARD + n]
        if fill is not None:
            view.fill_(fill)
        view = view.view(shape)
        self.live.append((base, n, head))
        return view

    def check(self):
        live, self.live = self.live, []
        bad = []
        for base, n, head in live:
            lo, hi = base[:GUARD], base[GUARD + n:]
            same = lambda a, b: torch.equal(a.view(torch.uint8) if a.dtype != torch.bool else a,  # noqa: E731
                                            b.view(torch.uint8) if b.dtype != torch.bool else b)
            if not (same(lo, head) and same(hi, head)):
                bad.append(f"{base.dtype}[{n}]")
            self.checked += 1
        assert not bad, f"guard band overwritten next to {len(bad)} buffer(s): {', '.join(bad[:8])}"


@pytest.fixture
def guarded(monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    g = Guards()
    real_empty, real_zeros, real_full, real_empty_like = torch.empty, torch.zeros, torch.full, torch.empty_like

    def is_cuda(kw):
        d = kw.get("device")
        return d is not None and torch.device(d).type == "cuda"

    def split(args):
        return args[0] if len(args) == 1 and isinstance(args[0], (tuple, list, torch.Size)) else args

    def empty(*args, **kw):
        if not is_cuda(kw) or kw.get("pin_memory") or "out" in kw:
            return real_empty(*args, **kw)
        return g.make(split(args), kw.get("dtype") or torch.get_default_dtype(), kw["device"])

    def zeros(*args, **kw):
        if not is_cuda(kw) or "out" in kw:
            return real_zeros(*args, **kw)
        return g.make(split(args), kw.get("dtype") or torch.get_default_dtype(), kw["device"], fill=0)

    def full(size, fill_value, **kw):
        if not is_cuda(kw) or "out" in kw:
            return real_full(size, fill_value, **kw)
        dt = kw.get("dtype") or (torch.float64 if isinstance(fill_value, float) else torch.int64)
        return g.make(size, dt, kw["device"], fill=fill_value)

    def empty_like(t, **kw):
        if not t.is_cuda or kw.get("device") not in (None, t.device) or kw.get("memory_format"):
            return real_empty_like(t, **kw)
        return g.make(t.shape, kw.get("dtype") or t.dtype, t.device)

    monkeypatch.setattr(torch, "empty", empty)
    monkeypatch.setattr(torch, "zeros", zeros)
    monkeypatch.setattr(torch, "full", full)
    monkeypatch.setattr(torch, "empty_like", empty_like)
    yield g
    torch.cuda.synchronize()
    monkeypatch.undo()
    g.check()
    assert g.checked > 0


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def test_guarded_golden_cases(guarded, sp, golden):
    tpar.test_every_case_matches_reference(sp, golden)
    guarded.check()
    tpar.test_demo_hand_results(sp)


def test_guarded_random_sweep(guarded, sp):
    tpar.test_random_sweep_against_oracle(sp, np.random.default_rng(7))


@pytest.mark.parametrize("rts", ["0", "1"])
def test_guarded_canonicalize_many_tiles(guarded, sp, monkeypatch, rts):
    tpar.test_canonicalize_many_tiles(sp, np.random.default_rng(11), monkeypatch, rts, (1 << 24, 3_000_017))


def test_guarded_wide_rows(guarded, sp):
    tpar.test_wide_rows_sell_hyb(sp, np.random.default_rng(5))


def test_guarded_degenerate_shapes(guarded, sp):
    tpar.test_new_entry_points_on_degenerate_shapes(sp)


@pytest.mark.parametrize("sigma,push_off", [(16, 0), (16, 3), (8, 1)])
def test_guarded_fused_push(guarded, sp, sigma, push_off):
    tp2p.test_fused_spmv_push_to_local_peers(sp, np.random.default_rng(3), sigma, push_off)
    tp2p.test_push_rows_to_local_peers(sp, np.random.default_rng(4))


def test_guarded_power_iteration_and_dispatch(guarded, sp):
    tp2p.test_power_iteration_graph_replay_identical(sp, np.random.default_rng(9))
    tdisp.test_norm_scale_kernel(sp)
    tdisp.test_bind_bit_identical(sp, "rmat", "csr5", dict(omega=32, sigma=16))
    tdisp.test_bind_bit_identical(sp, "laplace", "hyb", {})


def test_guarded_relabel(guarded, sp):
    trel.test_prefix_csr5_spmv(sp, 32, 16)
    trel.test_prefix_csr5_spmv(sp, 4, 16)
    trel.test_relabelled_power_iteration_matches_oracle(sp)


def test_guarded_exact_mode(guarded, sp, golden):
    """The reference-order kernels (csrc/spmv_exact.cu): golden cases, the
    CTA-per-long-row paths and the containers under guard bands."""
    texact.test_exact_equals_the_reference_outputs(sp, golden)
    guarded.check()
    texact.test_exact_long_rows_against_the_oracle(sp)
    guarded.check()
    texact.test_exact_scale_containers_and_repeat(sp)


def test_guard_detects_an_overrun(guarded, sp):
    """The harness itself: a deliberate one-element overrun is caught."""
    y = torch.empty(1000, dtype=torch.float64, device="cuda")
    base = guarded.live[-1][0]
    base[GUARD + 1000] = 1.0  # one past the end
    with pytest.raises(AssertionError, match="guard band"):
        guarded.check()
    del y
    guarded.checked = 1


def test_guarded_shadow_layout_paths(guarded, sp):
    """The round-2 kernels under guard bands: SELL on a degree-ordered
    matrix (empty-tail path, wide pieces incl. hub slices, slice ranges),
    CSR5 sigma 8 at 5 blocks/SM with its ranges, ELL with the x prefetch,
    the fused norm; all against the one-shot results / the oracle."""
    from oracle import port, synth_ref

    r, c, v = synth_ref.rmat(16, 16, 61)
    n = 1 << 16
    rng = np.random.default_rng(8)  # three rows of 40000 entries: a hub slice (> 32 pieces of 1024 columns)
    hub_r = np.repeat(np.array([100, 2000, 30000]), 40000)
    hub_c = np.concatenate([rng.choice(n, 40000, replace=False) for _ in range(3)])
    row, col, val = port.canonicalize(np.concatenate([r, hub_r]), np.concatenate([c, hub_c]),
                                      np.concatenate([v, rng.uniform(0.1, 1.0, hub_r.size)]), n, n)
    a = sp.canonicalize(row, col, val, n, n)
    order = sp.DegreeOrder(a)
    shadow = order.matrix(a)
    x = torch.from_numpy(synth_ref.uniform(n, 2)).cuda()
    xp = order.to_new(x)
    ref = port.dense_spmv_oracle(row, col, val, n, synth_ref.uniform(n, 2))
    bound = port.dense_spmv_oracle(row, col, np.abs(val), n, np.abs(synth_ref.uniform(n, 2)))
    for tag, kw in [("sell", dict(sell_c=32, sell_sigma=0)), ("csr5", dict(omega=32, sigma=8)),
                    ("sell", dict(sell_c=4, sell_sigma=64))]:
        m = sp.convert(tag, shadow, **kw)
        if tag == "sell":
            if kw["sell_c"] == 32:
                assert m.wide_plan()[8] > 0  # hub slices exist
            plan = m.range_plan(3)
        else:
            tb, rb = m.range_plan(3)
            k = len(tb) - 1
            plan = [(int(rb[i]), int(rb[i + 1]) if i + 1 < k else n, int(tb[i]), int(tb[i + 1])) for i in range(k)]
        y = sp.spmv(tag, m, xp)
        got = order.to_old(y).cpu().numpy()
        assert np.all(np.abs(got - ref) <= 1e-12 * bound), tag
        yr = torch.empty(n, dtype=torch.float64, device="cuda")
        for rr in plan:
            sp.bind_range(tag, m, xp, yr, rr)()
        assert torch.equal(yr, y), tag
    me = sp.to_ell(sp.synth.host_coo("C1"))
    xe = sp.synth.uniform_vector(me.n_cols, 4)
    assert torch.equal(sp.spmv("ell", me, xe), sp.spmv("ell", me, xe))
