"""Determinism stress of the live tier's dataflow (k_live_flow) and cluster
(k_live_cluster) launches: many graph replays and eager solves of the same
inputs must give the same bits as the checker every time (a missed dependency
or DSMEM race would show up as a run-to-run difference)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

bad = 0
for fam, n, reps in [("sym-uniform", 1 << 20, 60), ("normal", 1 << 18, 100), ("sym-uniform", 3_000_017, 10)]:
    d, e = G.generate(fam, n)
    ref = O.eigvals(d, e).w
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    for graph in (True, False):
        s = br.Solver(0, br.BrOptions(use_graph=graph))
        diffs = 0
        for _ in range(reps):
            w = s.eigvals_device(td, te).cpu().numpy()
            diffs += not np.array_equal(w, ref)
        s.close()
        print(fam, n, "graph" if graph else "eager", reps, "solves, mismatches:", diffs, flush=True)
        bad += diffs
print("TOTAL mismatches", bad)
sys.exit(1 if bad else 0)
