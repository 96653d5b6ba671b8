"""The C ABI library loads and exports every symbol include/spmvb.h declares
(no compute calls: runs without a GPU)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "spmvb.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spmvb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ["spmvb_canonicalize_begin", "spmvb_coo_to_csr", "spmvb_csr_to_csr5", "spmvb_csr_to_ell",
                 "spmvb_sell_plan", "spmvb_hyb_plan", "spmvb_spmv_csr", "spmvb_spmv_csr5", "spmvb_spmv_ell",
                 "spmvb_spmv_sell", "spmvb_spmv_hyb", "spmvb_csr_features"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_1805_11938_b200 import _lib

    lib = ctypes.CDLL(str(_lib.library_path()))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_1805_11938_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_error_string():
    from paper_1805_11938_b200 import _lib

    lib = _lib.load()
    assert lib.spmvb_abi_version() == 1
    assert isinstance(_lib.last_error(), str)


def test_library_is_sm100a():
    import subprocess, shutil

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    from paper_1805_11938_b200 import _lib

    out = subprocess.run([cuobjdump, "--list-elf", str(_lib.library_path())], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_package_refuses_to_run_without_cuda():
    import torch
    import paper_1805_11938_b200 as sp

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        sp.canonicalize([0], [0], [1.0], 1, 1)
