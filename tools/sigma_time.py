"""Timing of the requested-rows solve (brgpu_eigvals_rows) beside the
eigenvalue-only solve, host buffers in and out (wall clock, 3 repeats)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time
import numpy as np
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
s = br.Solver(0)
for n, ns in [(1<<20, 2), (1<<20, 16), (1<<16, 64)]:
    d, e = G.generate("sym-uniform", n)
    sel = np.linspace(0, n-1, ns).astype(np.int64)
    s.eigvals_rows(d, e, sel)
    t = time.perf_counter(); 
    for _ in range(3): w, R = s.eigvals_rows(d, e, sel)
    t1 = (time.perf_counter() - t) / 3
    s.eigvals(d, e)
    t = time.perf_counter()
    for _ in range(3): s.eigvals(d, e)
    t0 = (time.perf_counter() - t) / 3
    s.eigvals_rows(d, e, sel)
    tm = s.timing()
    print(f"n={n} nsel={ns}: device {tm}")
    print(f"n={n} nsel={ns}: rows {t1*1e3:.2f} ms  eigvals-only {t0*1e3:.2f} ms  row-norm err {np.abs((R*R).sum(1)-1).max():.1e}")
