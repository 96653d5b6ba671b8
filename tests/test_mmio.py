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


def test_native_writer_matches_the_python_expression():
    """write_matrix_market's entry lines come from the native formatter
    (spmvb_mm_format_*): byte for byte the reference's
    f"{i + 1} {j + 1} {v:.17g}" (coo.py:266-278), over magnitudes from
    denormals to 1e308, integers, signed zeros, shortest-repr ties and
    non-finite values; multithreaded chunks join in order."""
    from paper_1805_11938_b200 import coo

    rng = np.random.default_rng(5)
    n = 200_000  # above the single-thread cutoff
    with np.errstate(over="ignore"):
        v = rng.normal(size=n) * 10.0 ** rng.integers(-320, 309, size=n).astype(np.float64)
    special = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1e16, 1e17, 123456789012345678.0, 1e-5, 1e-4, 5e-324,
                        1.7976931348623157e308, 2.0 ** 53, 1 / 3, float("inf"), float("-inf"), float("nan"),
                        100.0, 1e15, 0.5, 2.5e-7])
    v[: special.size] = special
    r = rng.integers(0, 2**31 - 1, size=n)
    c = rng.integers(0, 2**31 - 1, size=n)
    want = "".join(f"{i + 1} {j + 1} {x:.17g}\n" for i, j, x in zip(r.tolist(), c.tolist(), v.tolist()))
    got = bytes(coo._format_entries(r, c, v)).decode("ascii")
    assert got == want
    assert bytes(coo._format_entries(r[:0], c[:0], v[:0])) == b""
    assert bytes(coo._format_entries(r[:3], c[:3], v[:3])).decode() == want[: sum(len(s) + 1 for s in want.split("\n")[:3])]


def test_write_matrix_market_streams_and_paths(tmp_path):
    """Text stream, binary stream and path destinations give the same bytes,
    and the tokenizer reads them back (no GPU: triplets only)."""
    import io
    from types import SimpleNamespace

    from paper_1805_11938_b200 import coo

    rng = np.random.default_rng(6)
    a = SimpleNamespace(n_rows=50, n_cols=70, row=np.sort(rng.integers(0, 50, 300)), col=rng.integers(0, 70, 300),
                        data=rng.normal(size=300))
    s, b = io.StringIO(), io.BytesIO()
    coo.write_matrix_market(a, s)
    coo.write_matrix_market(a, b)
    coo.write_matrix_market(a, tmp_path / "m.mtx")
    text = s.getvalue()
    assert text.encode() == b.getvalue() == (tmp_path / "m.mtx").read_bytes()
    assert text.startswith("%%MatrixMarket matrix coordinate real general\n50 70 300\n")
    rows, cols, vals, nr, nc = coo._fast_triplets(text.encode())
    assert (nr, nc) == (50, 70) and np.array_equal(rows, a.row) and np.array_equal(cols, a.col)
    assert vals.tobytes() == a.data.tobytes()
