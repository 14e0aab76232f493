"""Live-list tier vs dense tiers: bit-identical eigenvalues and traces, timing."""
import sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
cases = [("sym-uniform", 1 << 20), ("sym-uniform", 1 << 16), ("sym-uniform", 100003), ("uniform", 1 << 17),
         ("normal", 1 << 17), ("toeplitz121", 1 << 16), ("wilkinson", 1 << 18), ("clustered", 1 << 16)]
if len(sys.argv) > 1:
    cases = [(sys.argv[1], int(sys.argv[2]))]
for fam, n in cases:
    d, e = G.generate(fam, n)
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    res = {}
    for live in (False, True):
        s = br.Solver(0, br.BrOptions(live=live))
        s.set_trace(True)
        w = s.eigvals_device(td, te).cpu().numpy()
        tr = s.trace()
        s.set_trace(False)
        ts = []
        for _ in range(6):
            s.eigvals_device(td, te)
            ts.append(s.timing()["device_ms"])
        res[live] = (w, tr, min(ts), s.stats() if hasattr(s, "stats") else None)
        s.close()
    w0, t0, m0, _ = res[False]
    w1, t1, m1, _ = res[True]
    same = np.array_equal(w0.view(np.int64), w1.view(np.int64))
    print(f"{fam} n={n}: bit-identical {same} (max diff {np.max(np.abs(w0 - w1)):.3e}) trace equal {t0 == t1} "
          f"dense {m0:.3f} ms live {m1:.3f} ms", flush=True)
