"""One solve of a family (debug under compute-sanitizer)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
fam, n = sys.argv[1], int(sys.argv[2])
graph = int(sys.argv[3]) if len(sys.argv) > 3 else 0
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0, br.BrOptions(use_graph=bool(graph)))
w = s.eigvals_device(td, te).cpu().numpy()
print(fam, n, "sorted", bool(np.all(np.diff(w) >= 0)))
