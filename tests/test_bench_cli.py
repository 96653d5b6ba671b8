"""bench.py's rank launcher (--gpus N): the world must match, and a box with
fewer GPUs than asked fails with a clear message instead of silently
running one rank."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=300)


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2"], {"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=3" in r.stderr and r.stdout == ""


@pytest.mark.skipif(torch.cuda.device_count() >= 64, reason="box has that many GPUs")
def test_too_few_gpus_is_a_clear_error():
    r = _run(["--gpus", "64"])
    assert r.returncode == 2
    assert "needs 64 visible CUDA devices" in r.stderr and r.stdout == ""


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("formats", ["csr5,hyb", "sell"])
def test_two_rank_bench_code_path_over_gloo(formats):
    """bench.py --gpus 2 end to end (torchrun re-exec, row blocks, relabelled
    shards, overlapped all-gatherv, sparse exchange, e2e, max-over-ranks
    timing) with two ranks sharing this box's GPU over gloo: a check of the
    N > 1 code path the driver's scaling run takes with NCCL, not a
    measurement."""
    import json

    r = _run(["--gpus", "2", "--dist-backend", "gloo", "--workload", "C4", "--steps", "3", "--warmup", "3",
              "--no-configs", "--no-cpu-baseline", "--kernel-reps", "3", "--clock-ramp-s", "0.05", "--e2e-steps", "2",
              "--formats", formats])
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "rowblock2"
    assert line["config"]["format"] in formats.split(",")
    assert line["exchange"]["overlap_ranges"] > 1 or line["config"]["format"] not in ("csr5", "sell")
    assert "ms_per_step_allgatherv" in line["exchange"] and "ms_per_step_sparse" in line["exchange"]
    assert line["gpu_launches"] > 0 and line["value"] > 0
