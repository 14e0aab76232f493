"""A/B timing of library variants (BRGPU_LIB) on one config: mean device ms over reps."""
import os, sys, statistics
sys.path.insert(0, '.')
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
fam = sys.argv[1] if len(sys.argv) > 1 else "sym-uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
for _ in range(3):
    s.eigvals_device(td, te)
ts = []
for _ in range(10):
    s.eigvals_device(td, te)
    ts.append(s.timing()["device_ms"])
prof = s.profile_kernels(td, te)
top = sorted(prof.items(), key=lambda kv: -kv[1][0])[:4]
print(f"{os.environ.get('BRGPU_LIB','main'):28s} {fam} n={n}: {statistics.mean(ts):.3f} ms (min {min(ts):.3f})  ",
      "  ".join(f"{k}={v[0]:.3f}" for k, v in top))
