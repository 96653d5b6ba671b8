"""GPU kernels of the sparse x exchange (dist.GpuOps): column sets, the
owner-side gather and the receiver-side scatter, against numpy."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1805_11938_b200.dist import GpuOps

    return GpuOps


def test_column_set(ops, rng):
    for n_cols, nnz in [(1, 0), (1, 5), (1000, 1), (1000, 20000), (1 << 20, 300000)]:
        cols = rng.integers(0, n_cols, size=nnz).astype(np.int32)
        got = ops.column_set(torch.from_numpy(cols).cuda(), n_cols)
        assert got.dtype == torch.int32
        assert np.array_equal(got.cpu().numpy(), np.unique(cols))


def test_gather_scatter(ops, rng):
    n = 5000
    y = torch.from_numpy(rng.normal(size=n)).cuda()
    base = 1234
    idx = np.sort(rng.choice(n, size=700, replace=False)).astype(np.int32) + base
    buf = torch.empty(700, dtype=torch.float64, device="cuda")
    ops.gather(y, base, torch.from_numpy(idx).cuda(), buf)
    assert np.array_equal(buf.cpu().numpy(), y.cpu().numpy()[idx - base])
    x = torch.zeros(n + base, dtype=torch.float64, device="cuda")
    ops.scatter(buf, torch.from_numpy(idx).cuda(), x)
    want = np.zeros(n + base)
    want[idx] = y.cpu().numpy()[idx - base]
    assert np.array_equal(x.cpu().numpy(), want)
