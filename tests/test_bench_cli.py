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
