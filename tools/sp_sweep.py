"""Sparse vs dense bit-identity over a size sweep (debug)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
fam = sys.argv[1] if len(sys.argv) > 1 else "sym-uniform"
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [512, 1000, 1024, 2048, 3000, 4096, 5000, 8192, 10000, 16384, 20000, 32768, 65536]
sd = br.Solver(0, br.BrOptions(sparse=False, use_graph=False))
ss = br.Solver(0, br.BrOptions(sparse=True, use_graph=False))
ss.set_trace(True); sd.set_trace(True)
for n in sizes:
    d, e = G.generate(fam, n)
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    a = sd.eigvals_device(td, te).cpu().numpy(); ta = sd.trace()
    try:
        b = ss.eigvals_device(td, te).cpu().numpy(); tb = ss.trace()
    except Exception as ex:
        print(n, "ERROR", ex, flush=True); break
    diffs = [(x, y) for x, y in zip(ta, tb) if x != y]
    print(n, "identical", np.array_equal(a, b), int(np.sum(a != b)), "sorted", bool(np.all(np.diff(b) >= 0)),
          "trace diffs", len(diffs), diffs[:2], flush=True)
