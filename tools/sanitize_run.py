"""Small solves of every family for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
import os
SMALL = os.environ.get("SAN_SMALL") == "1"
cases = [("sym-uniform", 4000 if SMALL else 40000), ("toeplitz121", 3000 if SMALL else 12000), ("wilkinson", 5000 if SMALL else 30000), ("clustered", 2000 if SMALL else 5000), ("uniform", 3000 if SMALL else 9000)]
with br.Solver(0, br.BrOptions(use_graph=False)) as s:
    for fam, n in cases:
        d, e = G.generate(fam, n)
        w = s.eigvals(d, e)
        assert np.all(np.diff(w) >= 0)
        print(fam, n, "ok", flush=True)
    db, eb = G.generate_batch("sym-uniform", 16, 1024)
    s.eigvals_batched(db, eb)
    print("batched ok")
with br.Solver(0, br.BrOptions(use_graph=False, virtual_ranks=4)) as s:
    d, e = G.generate("toeplitz121", 16384)
    s.eigvals(d, e)
    print("virtual ok")
with br.Solver(0, br.BrOptions(use_graph=False, subtree=False)) as s:
    d, e = G.generate("wilkinson", 20000)
    s.eigvals(d, e)
    print("grid-only ok")
with br.Solver(0) as s:  # requested rows (sigma.cu), incl. the split tier and several blocks
    for fam, n in [("sym-uniform", 3000 if SMALL else 20000), ("toeplitz121", 2000 if SMALL else 10000)]:
        d, e = G.generate(fam, n)
        e[n // 3] = 0.0
        w, R = s.eigvals_rows(d, e, [0, n // 3, n // 3 + 1, n - 1, 7, 7])
        assert np.allclose((R * R).sum(1), 1.0, atol=1e-12)
    print("rows ok")
