"""Golden Matrix Market fixtures made by running the REFERENCE reader.

Run in the build container (where /root/reference exists):

    python tests/golden/make_mm_golden.py

Every text below goes through ``spmvkit.read_matrix_market``
(/root/reference/pkg/src/spmvkit/coo.py:158-263); the canonical triplets it
returns (values as float.hex, so bit-exact) or the exact
``MatrixMarketError`` message are stored in ``tests/golden/mm_cases.json``
with the input bytes (base64).  The texts cover real / integer / pattern
fields, general / symmetric storage, comments and blank lines, CRLF and the
other line breaks Python's ``str.splitlines`` honours, unusual number
spellings, duplicates and cancellations, and every error branch of the
reference reader (pinned by /root/reference/pkg/tests/test_coo.py:35-104).
"""

from __future__ import annotations

import base64
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().with_name("mm_cases.json")
H = "%%MatrixMarket matrix coordinate"


def _texts(rng):
    yield "demo", (f"{H} real general\n% the 4x4 running example\n4 4 8\n1 2 6\n1 3 1\n2 1 2\n2 3 8\n"
                   "2 4 3\n3 3 4\n4 2 7\n4 3 5\n").encode()
    yield "empty_3x3", f"{H} real general\n3 3 0\n".encode()
    yield "zero_by_zero", f"{H} real general\n0 0 0\n".encode()
    yield "symmetric_expansion", f"{H} real symmetric\n3 3 2\n2 1 5\n3 3 7\n".encode()
    yield "pattern_general", f"{H} pattern general\n2 2 2\n1 1\n2 2\n".encode()
    yield "pattern_symmetric", f"{H} pattern symmetric\n4 4 4\n1 1\n3 1\n4 2\n4 4\n".encode()
    yield "integer_field", f"{H} integer general\n2 2 1\n2 1 -3\n".encode()
    yield "integer_symmetric", f"{H} integer symmetric\n3 3 3\n1 1 4\n2 1 -1\n3 2 -1\n".encode()
    yield "duplicates_cancel", f"{H} real general\n2 2 3\n1 1 2\n1 1 -2\n2 2 5\n".encode()
    yield "duplicate_run_order", f"{H} real general\n1 1 4\n1 1 0.1\n1 1 0.2\n1 1 0.3\n1 1 1e-17\n".encode()
    yield "symmetric_mirror_duplicates", f"{H} real symmetric\n2 2 3\n2 1 1.5\n2 1 2.25\n2 2 -0.0\n".encode()
    yield "negative_zero_dropped", f"{H} real general\n2 3 2\n1 3 -0.0\n2 1 0.0\n".encode()
    yield "comments_blank_lines", f"{H} real general\n% c\n\n2 2 1\n% c\n1 2 3\n\n".encode()
    yield "crlf", f"{H} real general\r\n% crlf\r\n3 3 3\r\n1 1 1.5\r\n2 3 -2\r\n3 2 4e-3\r\n".encode()
    yield "lone_cr", f"{H} real general\r2 2 2\r1 1 2\r2 2 3\r".encode()
    yield "form_feed_and_vt", f"{H} real general\n2 2 2\n1 1 2\x0c2 2 3\x0b".encode()
    yield "unicode_line_sep", f"{H} real general\n2 2 2\n1 1 2 2 2 3\n".encode()
    yield "upper_case_banner", b"%%MATRIXMARKET MATRIX Coordinate REAL General\n2 2 1\n2 2 9\n"
    yield "leading_space_banner", f"   {H} real general\n1 1 1\n1 1 2\n".encode()
    yield "tabs_and_padding", f"{H} real general\n\t 3 2\t2  \n  1\t2   0.5 \n\t3 1 -7\t\n".encode()
    yield "no_trailing_newline", f"{H} real general\n2 2 1\n2 1 3.25".encode()
    yield "number_spellings", (f"{H} real general\n3 3 8\n1 1 +5\n1 2 .5\n1 3 5.\n2 1 1E-310\n2 2 -1e+3\n"
                               "2 3 1_0\n3 1 inf\n3 3 1.0000000000000002\n").encode()
    yield "nan_kept", f"{H} real general\n2 2 2\n1 1 nan\n2 2 1\n".encode()
    yield "rect_1x5", f"{H} real general\n1 5 3\n1 5 1\n1 1 2\n1 3 3\n".encode()
    yield "rect_5x1", f"{H} integer general\n5 1 2\n5 1 1\n2 1 -2\n".encode()
    # seeded random texts (17 significant digits, shuffled entry order)
    for k, (nr, nc, nnz, sym) in enumerate([(30, 40, 150, False), (25, 25, 90, True), (64, 7, 60, False)]):
        lines = [f"{H} real {'symmetric' if sym else 'general'}", "% seeded", f"{nr} {nc} {nnz}"]
        for _ in range(nnz):
            i = int(rng.integers(1, nr + 1))
            j = int(rng.integers(1, (i if sym else nc) + 1))
            lines.append(f"{i} {j} {rng.normal():.17g}")
        yield f"random{k}", ("\n".join(lines) + "\n").encode()
    # error branches (coo.py:166-262)
    yield "err_empty_input", b""
    yield "err_complex", f"{H} complex general\n1 1 1\n1 1 1 0\n".encode()
    yield "err_object", b"%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n"
    yield "err_array_format", b"%%MatrixMarket matrix array real general\n1 1\n1\n"
    yield "err_malformed_header", b"not a header\n1 1 0\n"
    yield "err_header_tokens", b"%%MatrixMarket matrix coordinate real\n1 1 0\n"
    yield "err_field", f"{H} hermitian general\n1 1 0\n".encode()
    yield "err_symmetry", f"{H} real skew-symmetric\n1 1 0\n".encode()
    yield "err_size_line", f"{H} real general\nbogus\n".encode()
    yield "err_size_negative", f"{H} real general\n2 -2 0\n".encode()
    yield "err_size_fields", f"{H} real general\n2 2\n".encode()
    yield "err_missing_size", f"{H} real general\n% only comments\n\n".encode()
    yield "err_exceeds_32bit", f"{H} real general\n4294967296 2 0\n".encode()
    yield "err_out_of_bounds", f"{H} real general\n2 2 1\n3 1 9\n".encode()
    yield "err_zero_index", f"{H} real general\n2 2 1\n0 1 9\n".encode()
    yield "err_too_few", f"{H} real general\n2 2 2\n1 1 9\n".encode()
    yield "err_too_many", f"{H} real general\n2 2 1\n1 1 9\n2 2 4\n".encode()
    yield "err_fields", f"{H} real general\n2 2 1\n1 1\n".encode()
    yield "err_pattern_fields", f"{H} pattern general\n2 2 1\n1 1 1\n".encode()
    yield "err_number", f"{H} real general\n2 2 1\n1 x 2\n".encode()
    yield "err_float_index", f"{H} real general\n2 2 1\n1.0 1 2\n".encode()
    yield "err_value", f"{H} real general\n2 2 1\n1 1 abc\n".encode()
    yield "err_crlf_too_few", f"{H} real general\r\n3 3 2\r\n1 1 1\r\n".encode()


def main():
    sys.path.insert(0, str(REF))
    from spmvkit import MatrixMarketError, read_matrix_market

    rng = np.random.default_rng(20261020)
    cases = []
    for name, raw in _texts(rng):
        rec = {"name": name, "text_b64": base64.b64encode(raw).decode()}
        try:
            a = read_matrix_market(raw)
            rec.update(n_rows=int(a.n_rows), n_cols=int(a.n_cols), row=a.row.tolist(), col=a.col.tolist(),
                       data_hex=[float(v).hex() for v in a.data.tolist()])
        except MatrixMarketError as exc:
            rec["error"] = str(exc)
        cases.append(rec)
    OUT.write_text(json.dumps(cases, indent=1) + "\n")
    print(f"wrote {len(cases)} cases ({sum('error' in c for c in cases)} errors) to {OUT}")


if __name__ == "__main__":
    main()
