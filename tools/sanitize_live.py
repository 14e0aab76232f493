"""Live-tier solves for compute-sanitizer: lane levels as the dataflow launch
(k_live_flow) and split-rule levels on clusters (k_live_cluster), checked
against the checker (memcheck / racecheck / synccheck runs)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
for graph in (False, True):
    with br.Solver(0, br.BrOptions(use_graph=graph)) as s:
        for fam, n in [("sym-uniform", 1 << 16), ("normal", 40000)]:
            d, e = G.generate(fam, n)
            w = s.eigvals(d, e)
            assert np.array_equal(w, O.eigvals(d, e).w), fam
            print(fam, n, "graph" if graph else "eager", "ok", flush=True)
