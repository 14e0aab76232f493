"""Per-class device ms of a batched solve: tools/prof_batch.py batch n"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
batch, n = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
d = rng.uniform(-1, 1, (batch, n)); e = rng.uniform(-1, 1, (batch, n - 1))
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
for _ in range(3): s.eigvals_batched_device(td, te)
prof = s.profile_kernels(td, te, batch)
print(f"batch {batch} x {n}: classes sum {sum(v[0] for v in prof.values()):.3f} ms")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"   {k:16s} {v[0]:.4f} ms  {v[1:]}")
