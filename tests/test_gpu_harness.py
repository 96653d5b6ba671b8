"""run_bench on the GPU kernels with the reference's stopping rule
(bench.py:178-253; reference tests test_bench.py:35-118 restated with our
own fake clocks).  GPU: run_bench converts and launches SpMVs."""

from __future__ import annotations

import itertools
import math
import statistics

import numpy as np
import pytest
import torch

from conftest import demo_triplets, random_triplets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1805_11938_b200 as sp

    return sp


class Durations:
    """Clock whose (start, end) pairs measure the given durations in a cycle."""

    def __init__(self, durations):
        self.it = itertools.cycle(durations)
        self.start = True

    def __call__(self):
        self.start = not self.start
        return next(self.it) if self.start else 0.0


def replay(durations, min_reps, max_reps, level, gap):
    """Independent replay of the CI stopping rule with the statistics module."""
    from scipy import stats

    samples = []
    for d in itertools.cycle(durations):
        samples.append(d)
        n = len(samples)
        if n >= min_reps:
            half = float(stats.t.ppf((1 + level) / 2, n - 1)) * statistics.stdev(samples) / math.sqrt(n)
            if 2 * half < gap * statistics.fmean(samples):
                return n
        if n >= max_reps:
            return n


@pytest.fixture
def demo(sp):
    r, c, v = demo_triplets()
    return sp.canonicalize(r, c, v, 4, 4)


def test_zero_variance_stops_at_min_reps(sp, demo):
    rec = sp.run_bench(demo, "csr", sp.BenchConfig(min_reps=5), "demo", clock=Durations([1e-3]))
    assert rec.reps == 5 and rec.ci_low_s == rec.mean_time_s == rec.ci_high_s == 1e-3


@pytest.mark.parametrize("durations", [(1e-3, 1.2e-3), (1e-3, 1.05e-3), (2e-3, 2.1e-3, 1.9e-3)])
def test_reps_match_offline_replay(sp, demo, durations):
    cfg = sp.BenchConfig(min_reps=5, max_reps=1000)
    rec = sp.run_bench(demo, "csr5", cfg, "demo", clock=Durations(durations))
    assert rec.reps == replay(durations, 5, 1000, cfg.ci_level, cfg.ci_gap)


def test_caps_fixed_reps_and_failures(sp, demo):
    assert sp.run_bench(demo, "ell", sp.BenchConfig(min_reps=2, max_reps=12, ci_gap=1e-9), "d",
                        clock=Durations([1e-3, 9e-3])).reps == 12
    assert sp.run_bench(demo, "hyb", sp.BenchConfig(fixed_reps=17), "d", clock=Durations([1e-3])).reps == 17
    failed = sp.run_bench(demo, "ell", sp.BenchConfig(max_grid_cells=2), "d")
    assert not failed.converted_ok and math.isnan(failed.mean_time_s)
    with pytest.raises(ValueError, match="min_reps"):
        sp.BenchConfig(min_reps=1)


def test_gflops_identity_and_byte_model(sp, rng):
    for i in range(5):
        rr, cc, vv, nr, nc = random_triplets(rng, max_dim=40)
        a = sp.canonicalize(rr, cc, vv, nr, nc)
        if a.nnz == 0:
            continue
        step = float(rng.uniform(1e-5, 1e-2))
        rec = sp.run_bench(a, "sell", sp.BenchConfig(min_reps=3, warmup_reps=0), f"m{i}", clock=Durations([step]))
        assert abs(rec.gflops * (rec.mean_time_s * 1e9) - 2.0 * a.nnz) <= math.ulp(2.0 * a.nnz)


def test_device_clock_and_labels(sp, demo):
    recs = [sp.run_bench(demo, t, sp.BenchConfig(min_reps=3, max_reps=20), "demo") for t in sp.FormatTag]
    assert all(r.converted_ok and r.mean_time_s > 0 for r in recs)
    assert sp.best_labels(recs)["demo"] in set(sp.FormatTag)
    tie = [sp.BenchRecord("m", t, 3, 1.0, 1.0, 1.0, 1.0, 1.0, True) for t in reversed(list(sp.FormatTag))]
    assert sp.best_labels(tie)["m"] is sp.FormatTag.CSR
