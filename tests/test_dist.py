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


def _matrix(seed=3, n=300, density=0.03, kind="random"):
    rng = np.random.default_rng(seed)
    if kind == "banded":
        # band |i-j| <= 6 plus a few long-range entries: shards read few columns
        i = np.repeat(np.arange(n), 13)
        j = i + np.tile(np.arange(-6, 7), n)
        keep = (j >= 0) & (j < n)
        extra = rng.integers(0, n, size=(40, 2))
        r = np.concatenate([i[keep], extra[:, 0]])
        c = np.concatenate([j[keep], extra[:, 1]])
        r, c, v = port.canonicalize(r, c, rng.uniform(0.1, 1.0, r.size), n, n)
        return port.to_csr(r, c, v, n), n
    nnz = int(density * n * n)
    flat = rng.choice(n * n, size=nnz, replace=False)
    r, c, v = port.canonicalize(flat // n, flat % n, rng.uniform(0.1, 1.0, nnz), n, n)
    # a few heavy rows make the nnz-balanced shards very different in rows
    return port.to_csr(r, c, v, n), n


class CpuOps:
    """CPU stand-ins for dist.GpuOps (same contracts)."""

    @staticmethod
    def sumsq(y, out_t):
        out_t.fill_(float(torch.dot(y, y)))

    @staticmethod
    def inv_sqrt(s, scale):
        scale.fill_(1.0 / float(torch.sqrt(s)))

    @staticmethod
    def column_set(cols, n_cols):
        return torch.unique(cols.long()).to(torch.int32)

    @staticmethod
    def gather(src, base, idx, dst):
        dst[: idx.numel()] = src[idx.long() - base]

    @staticmethod
    def scatter(src, idx, dst):
        dst[idx.long()] = src[: idx.numel()]


def _serial(ptr, ind, dat, n, x0, steps):
    x = x0.copy()
    scale = 1.0
    for _ in range(steps):
        y = scale * port.spmv_csr(ptr, ind, dat, n, x)
        scale = 1.0 / np.sqrt(np.dot(y, y))
        x = y
    return x, scale


def _worker(rank, world, port_no, steps, out, exchange="allgatherv", kind="random", ranges=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_11938_b200 import dist as spdist

    (ptr, ind, dat), n = _matrix(kind=kind)
    bounds = spdist.nnz_balanced_bounds(ptr, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    sub_ptr = ptr[lo:hi + 1] - ptr[lo]
    sub_ind, sub_dat = ind[ptr[lo]:ptr[hi]], dat[ptr[lo]:ptr[hi]]

    def local_spmv(x, out_view, scale):
        y = port.spmv_csr(sub_ptr, sub_ind, sub_dat, hi - lo, x.numpy())
        out_view.copy_(torch.from_numpy(y) * scale)

    spans, range_fn = None, None
    if ranges:
        # uneven spans (rank-dependent count), executed last to first
        cuts = np.unique(np.linspace(0, hi - lo, ranges + rank + 1).astype(int))
        spans = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])][::-1]

        def range_fn(k, x, out_view, scale):
            a, b = spans[k]
            p = sub_ptr[a:b + 1] - sub_ptr[a]
            y = port.spmv_csr(p, sub_ind[sub_ptr[a]:sub_ptr[b]], sub_dat[sub_ptr[a]:sub_ptr[b]], b - a, x.numpy())
            out_view[a:b].copy_(torch.from_numpy(y) * scale)

    x0 = torch.from_numpy(np.linspace(-1.0, 1.0, n))
    pi = spdist.PowerIteration(local_spmv, bounds, rank, world, torch.device("cpu"), x0, ops=CpuOps,
                               exchange=exchange, local_cols=torch.from_numpy(sub_ind.astype(np.int32)),
                               local_ranges=spans, local_spmv_range=range_fn)
    for _ in range(steps):
        pi.step()
    partial = pi.x.numpy().copy()
    vol = getattr(pi, "exchange_volume", None)
    full = pi.gather_full().numpy().copy()
    out[rank] = (full, float(pi.scale.item()), [int(b) for b in bounds], partial, np.unique(sub_ind), (lo, hi), vol)
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


def test_cost_balanced_bounds():
    from paper_1805_11938_b200 import dist as spdist

    (ptr, ind, dat), n = _matrix()
    for parts in (1, 2, 3, 8):
        for w in (0.0, 1.5, 10.0):
            b = spdist.cost_balanced_bounds(ptr, parts, row_weight=w)
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0) and len(b) == parts + 1
            cost = ptr + w * np.arange(n + 1)
            for p in range(1, parts):
                assert cost[b[p]] >= p * cost[-1] / parts
                assert b[p] == 0 or cost[b[p] - 1] < p * cost[-1] / parts


def test_two_rank_power_iteration_matches_serial():
    world, steps = 2, 12
    mgr = mp.Manager()
    out = mgr.dict()
    port_no = _free_port()
    mp.spawn(_worker, args=(world, port_no, steps, out), nprocs=world, join=True)
    (ptr, ind, dat), n = _matrix()
    want_x, want_scale = _serial(ptr, ind, dat, n, np.linspace(-1.0, 1.0, n), steps)
    for rank in range(world):
        x, scale, bounds = out[rank][:3]
        # every rank holds the full gathered iterate
        np.testing.assert_allclose(x, want_x, rtol=1e-12, atol=1e-300)
        assert scale == pytest.approx(want_scale, rel=1e-12)
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("world,kind", [(2, "banded"), (3, "banded"), (2, "random")])
def test_sparse_exchange_matches_serial(world, kind):
    """exchange='sparse': each rank receives only the x entries its shard's
    columns read; those entries (and its own rows) match the serial
    iteration every step, and gather_full() restores the whole iterate."""
    steps = 9
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), steps, out, "sparse", kind), nprocs=world, join=True)
    (ptr, ind, dat), n = _matrix(kind=kind)
    want_x, want_scale = _serial(ptr, ind, dat, n, np.linspace(-1.0, 1.0, n), steps)
    for rank in range(world):
        full, scale, bounds, partial, cols, (lo, hi), vol = out[rank]
        np.testing.assert_allclose(full, want_x, rtol=1e-12, atol=1e-300)
        assert scale == pytest.approx(want_scale, rel=1e-12)
        read = np.union1d(cols, np.arange(lo, hi))
        np.testing.assert_allclose(partial[read], want_x[read], rtol=1e-12, atol=1e-300)
        remote = cols[(cols < lo) | (cols >= hi)]
        assert vol["recv_entries"] == remote.size
        if kind == "banded":
            assert vol["recv_entries"] < vol["allgatherv_recv_entries"] / 4


@pytest.mark.parametrize("world", [2, 3])
def test_overlapped_ranges_match_serial(world):
    """All-gatherv overlapped with the local SpMV: each rank computes its rows
    in (uneven, rank-dependent) spans and sends every span as soon as it is
    done; the iterate matches the serial power iteration."""
    steps = 8
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), steps, out, "allgatherv", "random", 3), nprocs=world, join=True)
    (ptr, ind, dat), n = _matrix()
    want_x, want_scale = _serial(ptr, ind, dat, n, np.linspace(-1.0, 1.0, n), steps)
    for rank in range(world):
        full, scale = out[rank][:2]
        np.testing.assert_allclose(full, want_x, rtol=1e-12, atol=1e-300)
        assert scale == pytest.approx(want_scale, rel=1e-12)
