"""Golden fixtures for the benchmark-record format and label helpers,
produced by the REFERENCE package (spmvkit.bench) in the build container:

    python tests/golden/make_records.py

Writes records.json: a list of seeded BenchRecord field sets (converted and
failed ones, ties, NaN/inf), the reference's record_to_line for each, and
its best_labels / times_by_matrix over the list.  Tests compare the GPU
package's record I/O and label helpers against it (no /root/reference at
test time)."""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from spmvkit import bench  # noqa: E402
from spmvkit.formats import FormatTag  # noqa: E402

OUT = Path(__file__).resolve().with_name("records.json")


def main():
    rng = np.random.default_rng(2024)
    recs = []
    for mi in range(6):
        mid = f"group{mi % 2}/matrix_{mi}"
        for tag in FormatTag:
            failed = rng.random() < 0.15
            if failed:
                nan = float("nan")
                recs.append(bench.BenchRecord(mid, tag, 0, nan, nan, nan, nan, nan, False))
                continue
            mean = float(rng.choice([1e-3, 2e-3, 1e-3 * (1 + rng.random())]))  # ties happen
            recs.append(bench.BenchRecord(mid, tag, int(rng.integers(5, 1000)), mean, mean * 0.98, mean * 1.02,
                                          float(rng.random() * 100), float(rng.random() * 1e12), True))
    recs.append(bench.BenchRecord("inf_case", FormatTag.ELL, 3, 0.0, 0.0, 0.0, math.inf, math.inf, True))

    def enc(v):
        if isinstance(v, float) and not math.isfinite(v):
            return repr(v)
        return v.value if isinstance(v, FormatTag) else v

    data = {
        "records": [{k: enc(getattr(r, k)) for k in bench.RECORD_FIELDS} for r in recs],
        "lines": [bench.record_to_line(r) for r in recs],
        "best_labels": {k: v.value for k, v in bench.best_labels(recs).items()},
        "times_by_matrix": {m: {t.value: repr(x) for t, x in d.items()} for m, d in bench.times_by_matrix(recs).items()},
    }
    OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({len(recs)} records)")


if __name__ == "__main__":
    main()
