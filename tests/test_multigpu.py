"""Multi-GPU decomposition over real NCCL: two ranks through
brgpu_create_distributed -- phase-1 subtrees per rank, the grouped in-place
broadcast, the root-range split with in-place all-gathers (exchange_nccl /
exchange_allgather) -- bitwise equal to the single-GPU solve.  Needs >= 2
visible GPUs (skipped otherwise; the gloo tests cover the host-side schedule)."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2605_26599_b200 import generators as G

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _ngpu() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_ranks_nccl_bitwise(solver, tmp_path):
    out = tmp_path / "dist.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", str(ROOT / "tests" / "helpers" / "dist_solve.py"),
           str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = np.load(out)
    for key in res.files:
        fam, n, _ = key.rsplit("_", 2)
        d, e = G.generate(fam, int(n))
        assert np.array_equal(res[key], solver.eigvals(d, e)), key
