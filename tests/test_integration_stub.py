"""The ctypes stub a spmvkit maintainer would add runs as
written: it is extracted from INTEGRATION.md, pointed at the in-tree
libspmvb.so and checked against the CPU oracle."""

from __future__ import annotations

import types
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    start = text.index("# spmvkit/_gpu.py")
    end = text.index("```", start)
    lib = ROOT / "paper_1805_11938_b200" / "libspmvb.so"
    return text[start:end].replace('ctypes.CDLL("libspmvb.so")', f'ctypes.CDLL("{lib}")')


def test_stub_matches_oracle(rng):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ns: dict = {}
    exec(compile(_stub_source(), "INTEGRATION.md:_gpu.py", "exec"), ns)
    spmv_csr_gpu = ns["spmv_csr_gpu"]
    for n_rows, n_cols, density in [(300, 200, 0.05), (1000, 1000, 0.002), (50, 70, 0.0), (5000, 40, 0.3)]:
        nnz = int(density * n_rows * n_cols)
        flat = rng.choice(n_rows * n_cols, size=nnz, replace=False)
        r, c, v = port.canonicalize(flat // n_cols, flat % n_cols, rng.normal(size=nnz), n_rows, n_cols)
        ptr, ind, dat = port.to_csr(r, c, v, n_rows)
        m = types.SimpleNamespace(n_rows=n_rows, n_cols=n_cols, ptr=ptr, indices=ind, data=dat)
        x = rng.uniform(-1, 1, size=n_cols)
        y = spmv_csr_gpu(m, x)
        ref = port.dense_spmv_oracle(r, c, v, n_rows, x)
        bound = port.dense_spmv_oracle(r, c, np.abs(v), n_rows, np.abs(x))
        assert np.all(np.abs(y - ref) <= 1e-12 * bound)
        with pytest.raises(ValueError, match="length"):
            spmv_csr_gpu(m, np.ones(n_cols + 1))
