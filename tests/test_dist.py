"""Multi-process (world_size 2, gloo, CPU) test of the row-block power
iteration driver (paper_1805_11938_b200/dist.py): nnz-balanced partition,
grouped P2P all-gatherv of the y shards, ||y||^2 all-reduce, deferred
normalisation.  The local SpMV is the CPU oracle (test injection); on GPUs
the same driver calls the library kernels over NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(seed=3, n=300, density=0.03):
    rng = np.random.default_rng(seed)
    nnz = int(density * n * n)
    flat = rng.choice(n * n, size=nnz, replace=False)
    r, c, v = port.canonicalize(flat // n, flat % n, rng.uniform(0.1, 1.0, nnz), n, n)
    # a few heavy rows make the nnz-balanced shards very different in rows
    return port.to_csr(r, c, v, n), n


def _serial(ptr, ind, dat, n, x0, steps):
    x = x0.copy()
    scale = 1.0
    for _ in range(steps):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    return x, scale


def _worker(rank, world, port_no, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_11938_b200 import dist as spdist

    (ptr, ind, dat), n = _matrix()
    bounds = spdist.nnz_balanced_bounds(ptr, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    sub_ptr = ptr[lo:hi + 1] - ptr[lo]
    sub_ind, sub_dat = ind[ptr[lo]:ptr[hi]], dat[ptr[lo]:ptr[hi]]

    def local_spmv(x, out_view, scale):
        y = port.spmv_csr(sub_ptr, sub_ind, sub_dat, hi - lo, x.numpy())
        out_view.copy_(torch.from_numpy(y) * scale)

    def sumsq(y, out_t):
        out_t.fill_(float(torch.dot(y, y)))

    def inv_sqrt(s, scale):
        scale.fill_(1.0 / float(torch.sqrt(s)))

    x0 = torch.from_numpy(np.linspace(-1.0, 1.0, n))
    pi = spdist.PowerIteration(local_spmv, bounds, rank, world, torch.device("cpu"), x0, sumsq=sumsq,
                               inv_sqrt=inv_sqrt)
    for _ in range(steps):
        pi.step()
    out[rank] = (pi.x.numpy().copy(), float(pi.scale.item()), [int(b) for b in bounds])
    dist.destroy_process_group()


def test_partition_is_nnz_balanced_and_covers_rows():
    from paper_1805_11938_b200 import dist as spdist

    (ptr, ind, dat), n = _matrix()
    for parts in (1, 2, 3, 8, 64):
        b = spdist.nnz_balanced_bounds(ptr, parts)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0) and len(b) == parts + 1
        nnz = ptr[-1]
        for p in range(1, parts):
            # first row whose start reaches p * nnz / P
            assert ptr[b[p]] >= -(-p * nnz // parts)
            assert b[p] == 0 or ptr[b[p] - 1] < -(-p * nnz // parts)


def test_two_rank_power_iteration_matches_serial():
    world, steps = 2, 12
    mgr = mp.Manager()
    out = mgr.dict()
    port_no = _free_port()
    mp.spawn(_worker, args=(world, port_no, steps, out), nprocs=world, join=True)
    (ptr, ind, dat), n = _matrix()
    want_x, want_scale = _serial(ptr, ind, dat, n, np.linspace(-1.0, 1.0, n), steps)
    for rank in range(world):
        x, scale, bounds = out[rank]
        # every rank holds the full gathered iterate
        np.testing.assert_allclose(x, want_x, rtol=1e-12, atol=1e-300)
        assert scale == pytest.approx(want_scale, rel=1e-12)
    assert out[0][2] == out[1][2]
