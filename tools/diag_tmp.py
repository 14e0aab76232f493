import os, sys, ctypes as C, numpy as np
sys.path.insert(0, '.')
import oracle as O, paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
s = br.Solver(0)
bad = C.c_uint64(0)
if hasattr(s._lib, "brgpu_selftest_rcp"):
    print("selftest rc", s._lib.brgpu_selftest_rcp(s._h, 1 << 26, 777, C.byref(bad)), "mismatches", bad.value)
for fam, n in [("toeplitz121", 1000), ("toeplitz121", 4096), ("sym-uniform", 4096), ("wilkinson", 3000)]:
    d, e = G.generate(fam, n)
    w = s.eigvals(d, e)
    r = O.eigvals(d, e)
    print(os.environ.get("BRGPU_LIB", "main"), fam, n, "equal", np.array_equal(w, r.w), "maxdiff", np.max(np.abs(w - r.w)))
