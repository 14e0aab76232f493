"""bench.py's launch contract on a box without the requested GPUs: --gpus N must
fail loudly (never a silent single-GPU run labelled N)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]


def _bench(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=e)


def test_gpus_more_than_visible_fails_loudly():
    import torch
    if has_gpu() and torch.cuda.device_count() >= 64:
        pytest.skip("64 GPUs visible")
    r = _bench("--gpus", "64", "--steps", "1", "--warmup", "0")
    assert r.returncode == 2
    assert "GPU(s) visible" in r.stderr


def test_world_size_mismatch_fails_loudly():
    r = _bench("--gpus", "2", "--steps", "1", "--warmup", "0", env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr


def test_cpu_variants_small_config():
    """The CPU baseline legs (reference composition and C port, all cores and 1
    thread) on a small input: every variant reports a time or a reason."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2605_26599_b200 import generators as G
    cfg = dict(family="sym-uniform", n=2048, batch=0, workload="test")
    d, e = G.generate("sym-uniform", 2048)
    head, var = bench.cpu_variants(cfg, d, e, budget_s=20)
    assert {v["kind"] for v in var} == {"reference", "port"}
    for v in var:
        assert ("value" in v and v["value"] > 0) or "skipped" in v
    assert head is None or head["kind"] == "reference"
