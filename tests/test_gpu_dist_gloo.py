"""Row-block power iteration with the REAL CUDA kernels in a multi-process run.

Two (or three) processes share the one GPU of the test box, each owning an
nnz-balanced row block (dist.nnz_balanced_bounds), converted on the device
by the library (dist.row_block -> to_csr5 omega 32 sigma 16 / to_hyb), its
SpMV the library kernel (spmv, or the row-aligned tile ranges of
spmv_csr5_tiles for the overlapped all-gatherv).  The exchange runs over
gloo with host staging (PowerIteration stages through pinned host copies
when the group's backend has no device transport), so no rank's kernel
waits on another's.  Checked against the serial power iteration of
oracle/port.py (the reference's CSR algorithm, kernels.py:76-95) and
against each other: the overlapped ranges are bit-identical to the
single-shot shard SpMV (reference task plan: kernels.py:61-66)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port, synth_ref

pytestmark = pytest.mark.gpu

SCALE, EF, SEED = 13, 8, 41


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _host_matrix():
    hr, hc, hv = synth_ref.rmat(SCALE, EF, SEED)
    n = 1 << SCALE
    r, c, v = port.canonicalize(hr, hc, hv, n, n)
    return (hr, hc, hv), port.to_csr(r, c, v, n), n


def _worker(rank, world, port_no, steps, out, exchange, tag, n_ranges):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import dist as spdist

    (hr, hc, hv), _, n = _host_matrix()
    dev = torch.device("cuda", 0)
    csr = sp.to_csr(sp.canonicalize(hr, hc, hv, n, n, device=dev))
    bounds = spdist.nnz_balanced_bounds(csr.ptr, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    shard = spdist.row_block(csr, lo, hi)
    kw = {"csr5": dict(omega=32, sigma=16), "sell": dict(sell_c=32, sell_sigma=64)}.get(tag, {})
    m = sp.convert(tag, shard, **kw)

    def local_spmv(x, out_view, scale):
        sp.spmv(tag, m, x, out=out_view, scale=scale)

    ranges, range_fn = None, None
    if n_ranges and tag == "sell":
        splan = m.range_plan(n_ranges)[::-1]
        ranges = [(r_[6], r_[7]) for r_ in splan]

        def range_fn(k, x, out_view, scale):
            sp.spmv_sell_range(m, x, out_view, splan[k], scale=scale)
    elif n_ranges:
        tb, rb = m.range_plan(n_ranges)
        k_all = len(tb) - 1
        plan = [(int(rb[k]), int(rb[k + 1]) if k + 1 < k_all else m.n_rows, int(tb[k]), int(tb[k + 1]))
                for k in range(k_all)][::-1]
        ranges = [(a, b) for a, b, _, _ in plan]
        carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=dev)

        def range_fn(k, x, out_view, scale):
            a, b, t0, t1 = plan[k]
            sp.spmv_csr5_tiles(m, x, out_view, t0, t1, a, b, scale=scale, carry=carry)

    x0 = torch.from_numpy(synth_ref.uniform(n, 7)).to(dev)
    pi = spdist.PowerIteration(local_spmv, bounds, rank, world, dev, x0, exchange=exchange,
                               local_cols=shard.indices if exchange == "sparse" else None,
                               local_ranges=ranges, local_spmv_range=range_fn)
    assert pi._staged
    launches0 = sp._lib.load().spmvb_launch_count()
    for _ in range(steps):
        pi.step()
    launches = sp._lib.load().spmvb_launch_count() - launches0
    own = pi.x[lo:hi].cpu().numpy().copy()
    full = pi.gather_full().cpu().numpy().copy()
    out[rank] = (full, own, float(pi.scale.item()), (lo, hi), int(launches))
    dist.destroy_process_group()


def _run(world, steps, exchange, tag="csr5", n_ranges=0):
    mgr = mp.get_context("spawn").Manager()  # no fork of a CUDA-initialised process
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), steps, out, exchange, tag, n_ranges), nprocs=world, join=True)
    return dict(out)


def _serial(steps):
    _, (ptr, ind, dat), n = _host_matrix()
    x = synth_ref.uniform(n, 7)
    scale = 1.0
    for _ in range(steps):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    return x, scale


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


STEPS = 10


@pytest.mark.parametrize("world,exchange,tag,n_ranges", [
    (2, "allgatherv", "csr5", 0),
    (2, "allgatherv", "csr5", 4),
    (3, "allgatherv", "csr5", 3),
    (2, "sparse", "csr5", 0),
    (2, "allgatherv", "hyb", 0),
    (2, "allgatherv", "sell", 3),
])
def test_gloo_ranks_real_kernels_match_serial(cuda, world, exchange, tag, n_ranges):
    got = _run(world, STEPS, exchange, tag, n_ranges)
    want_x, want_scale = _serial(STEPS)
    tol = 1e-9
    for rank in range(world):
        full, own, scale, (lo, hi), launches = got[rank]
        assert launches >= STEPS  # the library's kernels ran on every step
        np.testing.assert_allclose(full, want_x, rtol=tol, atol=1e-12 * np.abs(want_x).max())
        assert scale == pytest.approx(want_scale, rel=1e-12)
    # every rank holds the same gathered iterate
    for rank in range(1, world):
        assert got[rank][0].tobytes() == got[0][0].tobytes()


def test_gloo_overlapped_ranges_bit_identical(cuda):
    """The overlapped all-gatherv (tile ranges, each sent as soon as done)
    gives the same iterate, bit for bit, as single-shot shard SpMVs."""
    a = _run(2, STEPS, "allgatherv", "csr5", 0)
    b = _run(2, STEPS, "allgatherv", "csr5", 4)
    for rank in range(2):
        assert a[rank][0].tobytes() == b[rank][0].tobytes()
        assert a[rank][2] == b[rank][2]


def _dealt_worker(rank, world, port_no, steps, out, tag, n_ranges):
    """The N > 1 headline layout: DegreeOrder(parts=world) dealt row blocks,
    each rank sending only its non-empty prefix (send_rows); the iterate is
    mapped back to the original ids."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import dist as spdist

    (hr, hc, hv), _, n = _host_matrix()
    dev = torch.device("cuda", 0)
    csr = sp.to_csr(sp.canonicalize(hr, hc, hv, n, n, device=dev))
    order = sp.DegreeOrder(csr, parts=world)
    mat = order.matrix(csr)
    bounds = order.part_bounds
    lo, hi = bounds[rank], bounds[rank + 1]
    shard = spdist.row_block(mat, lo, hi)
    rowdeg = torch.diff(shard.ptr)
    send_rows = int((rowdeg > 0).sum().item())
    assert bool((rowdeg[:send_rows] > 0).all()) and bool((rowdeg[send_rows:] == 0).all())
    kw = {"csr5": dict(omega=32, sigma=8), "sell": dict(sell_c=32, sell_sigma=0)}[tag]
    m = sp.convert(tag, shard, **kw)
    ranges, range_fn = None, None
    if n_ranges:
        if tag == "sell":
            plan = m.range_plan(n_ranges)[::-1]
            ranges = [(r_[6], r_[7]) for r_ in plan]
        else:
            tb, rb = m.range_plan(n_ranges)
            k_all = len(tb) - 1
            plan = [(int(rb[k]), int(rb[k + 1]) if k + 1 < k_all else m.n_rows, int(tb[k]), int(tb[k + 1]))
                    for k in range(k_all)][::-1]
            ranges = [(a, b) for a, b, _, _ in plan]

        def range_fn(k, x, out_view, scale):
            sp.bind_range(tag, m, x, out_view, plan[k], scale)()
    x0 = order.to_new(torch.from_numpy(synth_ref.uniform(n, 7)).to(dev))
    pi = spdist.PowerIteration(sp.SpmvOperator(tag, m), bounds, rank, world, dev, x0, local_ranges=ranges,
                               local_spmv_range=range_fn, send_rows=send_rows)
    for _ in range(STEPS):
        pi.step()
    out[rank] = (order.to_old(pi.gather_full()).cpu().numpy().copy(), float(pi.scale.item()), send_rows, hi - lo)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,tag,n_ranges", [(2, "sell", 3), (3, "csr5", 2), (2, "csr5", 0)])
def test_gloo_dealt_layout_sends_only_nonempty_rows(cuda, world, tag, n_ranges):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_dealt_worker, args=(world, _free_port(), STEPS, out, tag, n_ranges), nprocs=world, join=True)
    want_x, want_scale = _serial(STEPS)
    for rank in range(world):
        full, scale, send_rows, rows = out[rank]
        assert send_rows < rows  # there is an empty tail that did not travel
        np.testing.assert_allclose(full, want_x, rtol=1e-9, atol=1e-12 * np.abs(want_x).max())
        assert scale == pytest.approx(want_scale, rel=1e-12)
    for rank in range(1, world):
        assert out[rank][0].tobytes() == out[0][0].tobytes()
