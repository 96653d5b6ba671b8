from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "cases.npz"

# The paper's Fig. 1 / Table 1 running example (reference tests/conftest.py:8-28):
#   [[0, 6, 1, 0],
#    [2, 0, 8, 3],
#    [0, 0, 4, 0],
#    [0, 7, 5, 0]]
DEMO_ENTRIES = [(0, 1, 6.0), (0, 2, 1.0), (1, 0, 2.0), (1, 2, 8.0), (1, 3, 3.0), (2, 2, 4.0), (3, 1, 7.0), (3, 2, 5.0)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libspmvb.so")


class Golden:
    """Fixtures produced by the reference (tests/golden/make_golden.py)."""

    def __init__(self, path: Path):
        with np.load(path, allow_pickle=False) as z:
            self.d = {k: z[k] for k in z.files}
        self.names = [str(n) for n in self.d["__names__"]]

    def case(self, name: str) -> dict:
        p = name + "/"
        return {k[len(p):]: v for k, v in self.d.items() if k.startswith(p)}


@pytest.fixture(scope="session")
def golden() -> Golden:
    return Golden(GOLDEN)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def demo_triplets():
    r, c, v = zip(*DEMO_ENTRIES)
    return list(r), list(c), list(v)


def random_triplets(rng, n_rows=None, n_cols=None, density=None, max_dim=256):
    """Random canonical-ready triplets (own generator; shapes like the
    reference helpers: dims <= max_dim, density 0.1-20%, values +-U(0.1, 3))."""
    n_rows = int(rng.integers(1, max_dim + 1)) if n_rows is None else n_rows
    n_cols = int(rng.integers(1, max_dim + 1)) if n_cols is None else n_cols
    density = float(rng.uniform(0.001, 0.2)) if density is None else density
    nnz = min(n_rows * n_cols, max(0, round(density * n_rows * n_cols)))
    flat = rng.choice(n_rows * n_cols, size=nnz, replace=False)
    vals = rng.uniform(0.1, 3.0, size=nnz) * rng.choice([-1.0, 1.0], size=nnz)
    return flat // n_cols, flat % n_cols, vals, n_rows, n_cols
