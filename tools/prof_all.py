"""Per-kernel-class profile (events between launches, no graph) of one config."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
fam = sys.argv[1] if len(sys.argv) > 1 else "sym-uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
for _ in range(2):
    s.eigvals_device(td, te)
p = s.profile_kernels(td, te)
tot = sum(v[0] for v in p.values())
print(f"{fam} n={n}: total {tot:.3f} ms")
for k, (ms, c) in sorted(p.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:22s} {ms:8.3f} ms  {c:4d} launches")
