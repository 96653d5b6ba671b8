"""Peer-memory exchange on one GPU: the push kernel against local stand-in
"peer" buffers (every alignment of offset and length), and the whole
exchange="p2p" power-iteration step (symmetric memory, device barrier, norm
slots) at world size 1 against the plain iteration.  Multi-rank runs need
more GPUs than this harness has; the rank-to-rank ordering argument is in
dist.PowerIteration._plan_p2p."""

from __future__ import annotations

import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


def test_push_rows_to_local_peers(sp, rng):
    from paper_1805_11938_b200 import _lib

    n = 1000
    src_full = torch.from_numpy(rng.normal(size=n)).cuda()
    peers = [torch.full((n,), -7.0, dtype=torch.float64, device="cuda") for _ in range(3)]
    ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for a, b in [(0, 1000), (1, 2), (3, 10), (10, 11), (5, 5), (2, 999), (999, 1000)]:
        for p in peers:
            p.fill_(-7.0)
        _lib.check(_lib.load().spmvb_push_rows(src_full[a:].data_ptr(), b - a, ptrs.data_ptr(), 3, a, stream))
        want = np.full(n, -7.0)
        want[a:b] = src_full.cpu().numpy()[a:b]
        for p in peers:
            assert np.array_equal(p.cpu().numpy(), want), (a, b)


def test_p2p_power_iteration_world1(sp, rng):
    import torch.distributed as dist

    from paper_1805_11938_b200 import dist as spdist

    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    r, c, v = sp.synth.rmat_triplets(scale=12, edge_factor=8, seed=5)
    n = 1 << 12
    a = sp.canonicalize(r, c, v, n, n)
    m = sp.to_csr5(a, 32, 16)
    x0 = torch.from_numpy(rng.uniform(0.5, 1.0, size=n)).cuda()

    def local(xv, out, scale):
        sp.spmv("csr5", m, xv, out=out, scale=scale)

    tb, rb = m.range_plan(4)
    plan = [(int(rb[k]), int(rb[k + 1]) if k + 1 < len(tb) - 1 else n, int(tb[k]), int(tb[k + 1]))
            for k in range(len(tb) - 1)][::-1]

    def range_fn(k, xv, out, scale):
        a0, b0, t0, t1 = plan[k]
        sp.spmv_csr5_tiles(m, xv, out, t0, t1, a0, b0, scale=scale)

    ref = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0)
    p2p = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0, exchange="p2p")
    p2r = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0, exchange="p2p",
                                local_ranges=[(a0, b0) for a0, b0, _, _ in plan], local_spmv_range=range_fn)
    p2f = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0, exchange="p2p",
                                local_spmv_push=lambda xv, out, scale, peers, off: sp.spmv_csr5_push(
                                    m, xv, out, peers, off, scale=scale))
    assert p2p.exchange == "p2p"
    for _ in range(7):
        ref.step()
        p2p.step()
        p2r.step()
        p2f.step()
    torch.cuda.synchronize()
    want = ref.x.cpu().numpy()
    assert p2f.gather_full().cpu().numpy().tobytes() == p2p.gather_full().cpu().numpy().tobytes()
    for pi in (p2p, p2r, p2f):
        got = pi.gather_full().cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=0)
        assert float(pi.scale.item()) == pytest.approx(float(ref.scale.item()), rel=1e-14)


def test_power_iteration_graph_replay_identical(sp, rng):
    """PowerIteration.run(graph=True) (two steps captured in a CUDA graph,
    replayed) gives bit-identical iterates to eager steps, odd counts too."""
    from paper_1805_11938_b200 import dist as spdist

    r, c, v = sp.synth.rmat_triplets(scale=12, edge_factor=8, seed=6)
    n = 1 << 12
    a = sp.canonicalize(r, c, v, n, n)
    x0 = torch.from_numpy(rng.uniform(0.5, 1.0, size=n)).cuda()
    for tag, kw in [("csr5", dict(omega=32, sigma=16)), ("csr", {}), ("ell", dict(max_cells=1 << 30)),
                    ("hyb", {})]:
        m = sp.convert(tag, a, **kw)

        def local(xv, out, scale, m=m, tag=tag):
            sp.spmv(tag, m, xv, out=out, scale=scale)

        eager = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0)
        graph = spdist.PowerIteration(local, [0, n], 0, 1, torch.device("cuda", 0), x0)
        eager.run(21, graph=False)
        graph.run(6, graph=True)
        graph.run(7, graph=True)  # leaves the buffers swapped relative to the capture
        graph.run(8, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(eager.x, graph.x), tag
        assert torch.equal(eager.scale, graph.scale), tag
        # rebinding the iterate to fresh tensors forces a re-capture
        graph.x, graph.x_next = graph.x.clone(), graph.x_next.clone()
        eager.run(5, graph=False)
        graph.run(5, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(eager.x, graph.x), tag
        # "auto" measures eager vs replay on its first run of >= 16 steps
        eager.run(23, graph=False)
        graph.run(23, graph="auto")
        torch.cuda.synchronize()
        assert graph._graph_auto in (True, False), tag
        assert torch.equal(eager.x, graph.x), tag
        assert torch.equal(eager.scale, graph.scale), tag
        # the default is eager
        eager.run(3)
        graph.run(3)
        torch.cuda.synchronize()
        assert torch.equal(eager.x, graph.x), tag


def test_power_iteration_graph_capture_failure_falls_back(sp, rng):
    """A local_spmv that syncs with the host cannot be captured: run(graph=True)
    warns and finishes eagerly with the same iterate as eager steps."""
    from paper_1805_11938_b200 import dist as spdist

    r, c, v = sp.synth.rmat_triplets(scale=10, edge_factor=8, seed=7)
    n = 1 << 10
    m = sp.to_csr5(sp.canonicalize(r, c, v, n, n), 32, 16)
    x0 = torch.from_numpy(rng.uniform(0.5, 1.0, size=n)).cuda()

    def syncing(xv, out, scale):
        sp.spmv("csr5", m, xv, out=out, scale=scale)
        float(out[0].item())  # host sync: illegal inside a capture

    eager = spdist.PowerIteration(syncing, [0, n], 0, 1, torch.device("cuda", 0), x0)
    graph = spdist.PowerIteration(syncing, [0, n], 0, 1, torch.device("cuda", 0), x0)
    eager.run(9)
    with pytest.warns(RuntimeWarning, match="capture failed"):
        graph.run(9, graph=True)
    torch.cuda.synchronize()
    assert torch.equal(eager.x, graph.x)
    assert torch.equal(eager.scale, graph.scale)


@pytest.mark.parametrize("sigma", [16, 8])
@pytest.mark.parametrize("push_off", [0, 1, 1001])
def test_fused_spmv_push_to_local_peers(sp, rng, sigma, push_off):
    """spmvb_spmv_csr5_push: y equals the plain CSR5 SpMV bit for bit and
    every stand-in peer buffer holds y at [push_off, push_off + n) with the
    rest untouched -- empty rows, rows spanning several tiles and blocks,
    and odd offsets (the 16-byte store path) included."""
    n, nc = 30_000, 20_000
    counts = np.where(rng.random(n) < 0.4, 0, rng.integers(1, 30, n))
    counts[[5, 17_000, 29_999]] = [9_000, 3_000, 700]  # rows across many tiles / blocks, last row long
    rr = np.repeat(np.arange(n), counts)
    cc = np.concatenate([np.sort(rng.choice(nc, size=k, replace=False)) for k in counts if k])
    vv = rng.normal(size=rr.size)
    a = sp.canonicalize(torch.from_numpy(rr).int(), torch.from_numpy(cc).int(), vv, n, nc)
    m = sp.to_csr5(a, 32, sigma)
    x = torch.from_numpy(rng.normal(size=nc)).cuda()
    scale = torch.tensor([0.75], dtype=torch.float64, device="cuda")
    ref = sp.spmv_csr5(m, x, scale=scale)
    peers = [torch.full((push_off + n + 3,), -7.0, dtype=torch.float64, device="cuda") for _ in range(3)]
    ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device="cuda")
    y = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    sp.spmv_csr5_push(m, x, y, ptrs, push_off, scale=scale)
    torch.cuda.synchronize()
    assert y.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()
    for p in peers:
        h = p.cpu().numpy()
        assert h[push_off:push_off + n].tobytes() == y.cpu().numpy().tobytes()
        assert np.all(h[:push_off] == -7.0) and np.all(h[push_off + n:] == -7.0)


def test_fused_spmv_push_rejects_other_shapes(sp, rng):
    rr = np.array([0, 1, 2]); cc = np.array([0, 1, 2]); vv = np.ones(3)
    m = sp.to_csr5(sp.canonicalize(rr, cc, vv, 3, 3), 4, 16)
    p = torch.zeros(3, dtype=torch.float64, device="cuda")
    ptrs = torch.tensor([p.data_ptr()], dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="omega"):
        sp.spmv_csr5_push(m, torch.ones(3, dtype=torch.float64, device="cuda"), None, ptrs, 0)
