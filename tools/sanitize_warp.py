"""Warp tier under compute-sanitizer: Toeplitz n = 16384 (K > 1024 below the
root: split secular / refreshed weights / rows with cp.async tiles), a glued
Wilkinson case and requested rows through the same tier."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

with br.Solver(0, br.BrOptions(use_graph=False)) as s:
    for fam, n in [("toeplitz121", 16384), ("wilkinson", 20000)]:
        d, e = G.generate(fam, n)
        w = s.eigvals(d, e)
        assert np.all(np.diff(w) >= 0)
        print(fam, n, "ok", flush=True)
    d, e = G.generate("toeplitz121", 16384)
    w, R = s.eigvals_rows(d, e, [0, 8191, 16383])
    print("rows ok", flush=True)
