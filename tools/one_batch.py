"""One batched solve (ncu launch lists): tools/one_batch.py batch n"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2605_26599_b200 as br
batch, n = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
d = torch.tensor(rng.uniform(-1, 1, (batch, n)), device="cuda")
e = torch.tensor(rng.uniform(-1, 1, (batch, n - 1)), device="cuda")
s = br.Solver(0, br.BrOptions(use_graph=False))
s.eigvals_batched_device(d, e)
torch.cuda.synchronize()
