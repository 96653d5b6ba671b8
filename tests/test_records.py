"""Benchmark-record format and label helpers against fixtures produced by
the reference (tests/golden/make_records.py -> records.json), plus the GPU
corpus benchmark that turns Matrix Market files into B200 label records."""

from __future__ import annotations

import io
import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_1805_11938_b200 import harness
from paper_1805_11938_b200.formats import FormatTag

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "records.json").read_text())


def _rec(d):
    def num(v):
        return float(v) if isinstance(v, str) else v

    return harness.BenchRecord(d["matrix_id"], FormatTag(d["format"]), d["reps"], num(d["mean_time_s"]),
                               num(d["ci_low_s"]), num(d["ci_high_s"]), num(d["gflops"]), num(d["bandwidth_bps"]),
                               d["converted_ok"])


def _same(a: harness.BenchRecord, b: harness.BenchRecord) -> bool:
    for f in harness._RECORD_FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        if isinstance(x, float) and math.isnan(x):
            if not (isinstance(y, float) and math.isnan(y)):
                return False
        elif x != y:
            return False
    return True


def test_record_lines_match_reference():
    recs = [_rec(d) for d in GOLD["records"]]
    assert [harness.record_to_line(r) for r in recs] == GOLD["lines"]
    for r, line in zip(recs, GOLD["lines"]):
        assert _same(harness.record_from_line(line), r)
    buf = io.StringIO()
    harness.write_records(recs, buf)
    back = harness.read_records(io.StringIO(buf.getvalue()))
    assert len(back) == len(recs) and all(_same(a, b) for a, b in zip(back, recs))
    with pytest.raises(ValueError, match="bad record line"):
        harness.record_from_line("matrix_id:x format:csr reps:abc")


def test_labels_and_times_match_reference():
    recs = [_rec(d) for d in GOLD["records"]]
    assert {k: v.value for k, v in harness.best_labels(recs).items()} == GOLD["best_labels"]
    got = {m: {t.value: repr(x) for t, x in d.items()} for m, d in harness.times_by_matrix(recs).items()}
    assert got == GOLD["times_by_matrix"]


def test_discover_corpus(tmp_path):
    for rel in ["b/m2.mtx", "a/m1.mtx", "c.mtx", "ignore.txt"]:
        p = tmp_path / rel
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_text("x")
    assert [mid for mid, _ in harness.discover_corpus(tmp_path)] == ["a/m1", "b/m2", "c"]


@pytest.mark.gpu
def test_bench_corpus_on_gpu(tmp_path, rng):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    for name, (n, dens) in {"small/banded": (400, 0.02), "small/random": (300, 0.05)}.items():
        k = int(n * n * dens)
        flat = rng.choice(n * n, size=k, replace=False)
        a = sp.canonicalize(flat // n, flat % n, rng.normal(size=k), n, n)
        path = tmp_path / f"{name}.mtx"
        path.parent.mkdir(parents=True, exist_ok=True)
        sp.write_matrix_market(a, path)
    (tmp_path / "broken.mtx").write_text("not a matrix market file\n")
    cfg = harness.BenchConfig(fixed_reps=3, warmup_reps=1)
    records, labels, skipped = harness.bench_corpus(tmp_path, cfg)
    assert len(skipped) == 1 and "broken" in skipped[0]
    assert len(records) == 2 * len(FormatTag)
    assert set(labels) == {"small/banded", "small/random"}
    assert all(r.converted_ok and r.reps == 3 and r.mean_time_s > 0 for r in records)
    buf = io.StringIO()
    harness.write_records(records, buf)
    assert [harness.record_to_line(r) for r in harness.read_records(io.StringIO(buf.getvalue()))] == \
        [harness.record_to_line(r) for r in records]
    # in-memory corpus, a subset of formats
    a = sp.canonicalize(np.arange(50), np.arange(50), np.ones(50), 50, 50)
    recs2, labels2, _ = harness.bench_corpus([("diag", a)], cfg, formats=["csr", "ell"])
    assert [r.format for r in recs2] == [FormatTag.CSR, FormatTag.ELL] and "diag" in labels2
