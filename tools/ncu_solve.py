"""Small driver for ncu captures: `reps` solves of one BASELINE config on cuda:0
(graph disabled so every kernel is a separate, attributable launch)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="sym-uniform")
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
d, e = G.generate(a.family, a.n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0, br.BrOptions(use_graph=bool(a.graph)))
for _ in range(a.reps):
    w = s.eigvals_device(td, te)
torch.cuda.synchronize()
print("launches per solve", s.stats()["kernel_launches"], "device_ms", s.timing())
