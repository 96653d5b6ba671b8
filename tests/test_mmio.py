"""Native Matrix Market tokenizer (csrc/mmio.cpp) versus the reference-
semantics Python parser (coo.py:166-262 restated), host only (no GPU):
same triplets on every accepted input; every error and every unusual text
is handed back (None) so the Python parser raises the reference's exact
MatrixMarketError."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1805_11938_b200.coo import MatrixMarketError, _fast_triplets, _parse_text_triplets


def _same(raw: bytes):
    fast = _fast_triplets(raw)
    assert fast is not None
    r, c, v, nr, nc = _parse_text_triplets(raw.decode())
    fr, fc, fv, fnr, fnc = fast
    assert (fnr, fnc) == (nr, nc)
    assert fr.tolist() == r and fc.tolist() == c
    assert np.asarray(v, dtype=np.float64).tobytes() == fv.tobytes()


def _text(rng, n_rows, n_cols, nnz, field="real", symmetry="general", crlf=False, noise=False):
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}", "% generated"]
    if noise:
        lines += ["", "   % indented comment", "\t"]
    lines.append(f"{n_rows} {n_cols} {nnz}")
    for k in range(nnz):
        i = int(rng.integers(1, n_rows + 1))
        j = int(rng.integers(1, n_cols + 1)) if symmetry == "general" else int(rng.integers(1, i + 1))
        if field == "pattern":
            lines.append(f"{i} {j}")
        elif field == "integer":
            lines.append(f"{i} {j} {int(rng.integers(-9, 10))}")
        else:
            val = rng.choice([f"{rng.normal():.17g}", f"{rng.uniform(-5, 5):e}", "inf", "-0.0", "1e-310", "5."])
            lines.append(f"  {i}\t{j}   {val} ")
        if noise and k % 7 == 0:
            lines += ["% mid comment", ""]
    sep = "\r\n" if crlf else "\n"
    return (sep.join(lines) + sep).encode()


@pytest.mark.parametrize("field", ["real", "integer", "pattern"])
@pytest.mark.parametrize("symmetry", ["general", "symmetric"])
def test_fast_parser_matches_reference_semantics(rng, field, symmetry):
    for trial in range(6):
        n = int(rng.integers(1, 50))
        _same(_text(rng, n, n, int(rng.integers(0, 200)), field, symmetry, crlf=trial % 2 == 1, noise=trial > 2))


def test_large_multithreaded_input(rng):
    _same(_text(rng, 5000, 4000, 120_000))  # > 1 MiB of entries: the threaded path


@pytest.mark.parametrize(
    "raw",
    [
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 9\n",  # out of bounds
        b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 9\n",  # too few
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 9\n2 2 4\n",  # too many
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",  # fields
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 2\n",  # number
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1_0\n",  # Python-only spelling
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\r1 1 2\n",  # lone CR separator
        b"%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",  # header error
        b"%%MatrixMarket matrix coordinate real general\nbogus\n",  # size line error
    ],
)
def test_errors_and_unusual_text_go_to_the_reference_parser(raw):
    assert _fast_triplets(raw) is None


def test_reference_parser_messages_name_the_line():
    with pytest.raises(MatrixMarketError, match="line 3"):
        _parse_text_triplets("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 9\n")
    r, c, v, nr, nc = _parse_text_triplets("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1_0\n")
    assert v == [10.0]
