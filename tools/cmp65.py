import sys; sys.path.insert(0,'.')
import numpy as np, oracle as O, paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
d,e = G.generate("sym-uniform", 1<<16)
ref = O.eigvals(d,e).w
for live in (False, True):
    s = br.Solver(0, br.BrOptions(live=live))
    w = s.eigvals(d,e)
    print("live", live, "equal", np.array_equal(w, ref), "maxdiff", np.max(np.abs(w-ref)), "n diff", np.sum(w != ref))
    s.set_trace(True); s.eigvals(d,e); t = s.trace(); s.close()
    rt = O.eigvals(d,e,trace=True).trace
    bad = [(a,b) for a,b in zip(t, rt) if a != b]
    print("  trace records differing:", len(bad), bad[:3])
