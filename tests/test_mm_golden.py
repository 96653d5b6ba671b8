"""Matrix Market ingestion pinned to the REFERENCE reader.

``tests/golden/mm_cases.json`` holds 51 texts run through
``spmvkit.read_matrix_market`` (/root/reference/pkg/src/spmvkit/coo.py:158-263)
by ``tests/golden/make_mm_golden.py``: the canonical triplets (values as
float.hex) or the exact ``MatrixMarketError`` message.

CPU: both of our parse paths -- the native multithreaded tokenizer
(``_fast_triplets``, csrc/mmio.cpp) whenever it accepts the text, and the
reference-semantics parser (``_parse_text_triplets``) always -- followed by
the oracle's canonicalize give the reference's triplets bit for bit; the
public ``read_matrix_market`` raises the reference's message for every error
(errors are raised before anything touches the GPU).
GPU: the public ``read_matrix_market`` (tokenizer -> GPU canonicalize) gives
the reference's triplets bit for bit.
"""

from __future__ import annotations

import base64
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import port
from paper_1805_11938_b200.coo import MatrixMarketError, _fast_triplets, _parse_text_triplets, read_matrix_market

CASES = json.loads((Path(__file__).resolve().parent / "golden" / "mm_cases.json").read_text())
OK = [c for c in CASES if "error" not in c]
ERR = [c for c in CASES if "error" in c]


def _raw(case) -> bytes:
    return base64.b64decode(case["text_b64"])


def _expected(case):
    data = np.array([float.fromhex(h) for h in case["data_hex"]], dtype=np.float64)
    return np.array(case["row"], dtype=np.int64), np.array(case["col"], dtype=np.int64), data


def _same(case, row, col, data):
    er, ec, ed = _expected(case)
    assert np.asarray(row).tolist() == er.tolist()
    assert np.asarray(col).tolist() == ec.tolist()
    assert np.asarray(data, dtype=np.float64).tobytes() == ed.tobytes()


def test_fixture_covers_the_reference_cases():
    assert len(CASES) >= 50 and len(ERR) >= 20
    names = {c["name"] for c in CASES}
    for must in ("demo", "crlf", "symmetric_expansion", "pattern_general", "integer_field", "err_too_many"):
        assert must in names


@pytest.mark.parametrize("case", OK, ids=[c["name"] for c in OK])
def test_parsers_then_oracle_canonicalize_match_reference(case):
    raw = _raw(case)
    rows, cols, vals, nr, nc = _parse_text_triplets(raw.decode("utf-8"))
    assert (nr, nc) == (case["n_rows"], case["n_cols"])
    _same(case, *port.canonicalize(np.array(rows, np.int64), np.array(cols, np.int64),
                                   np.array(vals, np.float64), nr, nc))
    fast = _fast_triplets(raw)
    if fast is not None:  # the native tokenizer accepted the text: same triplets
        fr, fc, fv, fnr, fnc = fast
        assert (fnr, fnc) == (nr, nc)
        _same(case, *port.canonicalize(fr, fc, fv, fnr, fnc))


def test_native_tokenizer_takes_the_ordinary_texts():
    # the fast path must not hand every text back to Python
    taken = [c["name"] for c in OK if _fast_triplets(_raw(c)) is not None]
    for must in ("demo", "crlf", "symmetric_expansion", "pattern_general", "integer_field", "random0", "random1"):
        assert must in taken, taken


@pytest.mark.parametrize("case", ERR, ids=[c["name"] for c in ERR])
def test_errors_match_reference_message(case):
    raw = _raw(case)
    assert _fast_triplets(raw) is None
    with pytest.raises(MatrixMarketError) as err:
        read_matrix_market(raw)
    assert str(err.value) == case["error"]
    with pytest.raises(MatrixMarketError) as err2:
        _parse_text_triplets(raw.decode("utf-8"))
    assert str(err2.value) == case["error"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", OK, ids=[c["name"] for c in OK])
def test_read_matrix_market_gpu_matches_reference(case):
    a = read_matrix_market(_raw(case))
    assert (a.n_rows, a.n_cols) == (case["n_rows"], case["n_cols"])
    _same(case, a.row.cpu().numpy(), a.col.cpu().numpy(), a.data.cpu().numpy())
