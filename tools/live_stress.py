"""Live-tier stress: many families / sizes / scalings, GPU vs checker bit-exact (and tier use)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

rng = np.random.default_rng(11)
cases = []
for n in [32768, 40001, 65535, 65536, 70001, 131071, 200000, 262144]:
    cases.append(("sym-uniform", n, None))
    cases.append(("normal", n, None))
for n in [50000, 131072]:
    for fam in ("uniform", "clustered", "toeplitz121", "wilkinson"):
        cases.append((fam, n, None))
# hand-made: graded diagonal, tiny off-diagonals, repeated diagonal, +-1 spikes
def special(kind, n):
    if kind == "graded":
        d = np.exp(-np.linspace(0, 30, n)) * rng.uniform(-1, 1, n); e = rng.uniform(-1, 1, n - 1) * 1e-3
    elif kind == "tiny-e":
        d = rng.uniform(-1, 1, n); e = rng.uniform(-1, 1, n - 1) * 1e-9
    elif kind == "repeated":
        d = np.round(rng.uniform(-1, 1, n), 2); e = rng.uniform(-1, 1, n - 1) * 0.3
    elif kind == "spikes":
        d = rng.uniform(-1, 1, n); d[::97] *= 1e6; e = rng.uniform(-1, 1, n - 1)
    elif kind == "ones":
        d = np.ones(n); e = rng.uniform(0.5, 1, n - 1)
    return d, e
for kind in ("graded", "tiny-e", "repeated", "spikes", "ones"):
    for n in (65536, 100001):
        cases.append((kind, n, "special"))
bad = 0
s = br.Solver(0)
for fam, n, tag in cases:
    d, e = special(fam, n) if tag else G.generate(fam, n)
    ref = O.eigvals(d, e).w
    w = s.eigvals(d, e)
    prof = s.profile_kernels(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"))
    live = prof.get("live_level", (0, 0))[1] > 0
    ok = np.array_equal(w.view(np.int64), ref.view(np.int64))
    bad += not ok
    print(f"{fam:12s} n={n:7d} live={int(live)} bit-exact={ok}" + ("" if ok else f" maxdiff {np.max(np.abs(w-ref)):.3e}"), flush=True)
s.close()
print("FAILURES", bad)
