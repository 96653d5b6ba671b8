"""Two GPUs, one process each, NCCL (skipped on boxes with fewer GPUs; the
round-end boxes of this project have one).  The three exchanges of the
row-block power iteration (dist.py) -- the NCCL all-gatherv overlapped with
CSR5 tile ranges, the sparse exchange and the peer-memory exchange (p2p, our
kernels over NVLink through symmetric memory: fused SpMV + peer store, and
the separate push kernel) and the C ABI's spmvb_dist_* step -- must give
the same iterate as the serial power iteration of oracle/port.py (the reference CSR algorithm,
kernels.py:76-95, partitioned as kernels.py:61-66 does per task)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port, synth_ref

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                       reason="needs two CUDA devices"),
]

SCALE, EF, SEED, STEPS = 16, 8, 43, 12


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, out, exchange, fused):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import dist as spdist

    n = 1 << SCALE
    r, c, v = sp.synth.rmat_triplets(SCALE, EF, SEED, dev)
    csr = sp.to_csr(sp.canonicalize(r, c, v, n, n))
    bounds = spdist.nnz_balanced_bounds(csr.ptr, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    shard = spdist.row_block(csr, lo, hi)
    m = sp.to_csr5(shard, 32, 16)
    tb, rb = m.range_plan(4)
    k_all = len(tb) - 1
    plan = [(int(rb[k]), int(rb[k + 1]) if k + 1 < k_all else m.n_rows, int(tb[k]), int(tb[k + 1]))
            for k in range(k_all)][::-1]
    carry = torch.empty(max(m.num_tiles, 1), dtype=torch.float64, device=dev)

    def range_fn(k, x, o, s):
        a, b, t0, t1 = plan[k]
        sp.spmv_csr5_tiles(m, x, o, t0, t1, a, b, scale=s, carry=carry)

    push = None
    if exchange == "p2p" and fused:
        def push(x, o, s, peers, off):
            sp.spmv_csr5_push(m, x, o, peers, off, scale=s, carry=carry)

    x0 = synth_ref.uniform(n, 7)
    if exchange == "native-dealt":  # the bench's N > 1 path: dealt shadow layout, C-ABI ranges, send_rows
        order = sp.DegreeOrder(csr, parts=world)
        mat = order.matrix(csr)
        b = order.part_bounds
        shard_d = spdist.row_block(mat, b[rank], b[rank + 1])
        md = sp.to_sell(shard_d, 32, 0)
        plan_d = md.range_plan(4)[::-1]
        rowdeg = torch.diff(shard_d.ptr)
        ne = int((rowdeg > 0).sum().item())
        comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
        pi = spdist.NativePowerIteration(
            sp.SpmvOperator("sell", md), b, rank, world, dev, order.to_new(torch.from_numpy(x0).to(dev)), comm,
            ranges=[(r_[6], r_[7]) for r_ in plan_d],
            range_op=lambda k, xv, o, sc: sp.bind_range("sell", md, xv, o, plan_d[k], sc), send_rows=ne)
        for _ in range(STEPS):
            pi.step()
        torch.cuda.synchronize()
        out[rank] = (order.to_old(pi.x).cpu().numpy().copy(), float(pi.scale.item()))
        pi.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    if exchange == "native":  # the C ABI's spmvb_dist_* over torch's NCCL communicator
        comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
        pi = spdist.NativePowerIteration(sp.SpmvOperator("csr5", m), bounds, rank, world, dev,
                                         torch.from_numpy(x0).to(dev), comm)
        for _ in range(STEPS):
            pi.step()
        torch.cuda.synchronize()
        out[rank] = (pi.x.cpu().numpy().copy(), float(pi.scale.item()))
        pi.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    pi = spdist.PowerIteration(sp.SpmvOperator("csr5", m), bounds, rank, world, dev, torch.from_numpy(x0).to(dev),
                               exchange=exchange, local_cols=shard.indices if exchange == "sparse" else None,
                               local_ranges=[(a, b) for a, b, _, _ in plan], local_spmv_range=range_fn,
                               local_spmv_push=push)
    for _ in range(STEPS):
        pi.step()
    torch.cuda.synchronize()
    out[rank] = (pi.gather_full().cpu().numpy().copy(), float(pi.scale.item()))
    dist.barrier()
    dist.destroy_process_group()


def _serial():
    hr, hc, hv = synth_ref.rmat(SCALE, EF, SEED)
    n = 1 << SCALE
    row, col, val = port.canonicalize(hr, hc, hv, n, n)
    ptr, ind, dat = port.to_csr(row, col, val, n)
    x, scale = synth_ref.uniform(n, 7), 1.0
    for _ in range(STEPS):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    return x, scale


@pytest.mark.parametrize("exchange,fused", [("allgatherv", False), ("sparse", False), ("p2p", True),
                                            ("p2p", False), ("native", False), ("native-dealt", False)])
def test_two_gpu_exchanges_match_serial(exchange, fused):
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), out, exchange, fused), nprocs=2, join=True)
    want_x, want_scale = _serial()
    for rank in range(2):
        x, scale = out[rank]
        np.testing.assert_allclose(x, want_x, rtol=1e-9, atol=1e-12 * np.abs(want_x).max())
        assert scale == pytest.approx(want_scale, rel=1e-12)
    assert out[0][0].tobytes() == out[1][0].tobytes()
