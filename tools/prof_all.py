"""Per-class device ms (profile_kernels) of the default solver: tools/prof_all.py fam n [fam n ...]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
args = sys.argv[1:] or ["sym-uniform", str(1 << 20)]
for fam, n in zip(args[::2], args[1::2]):
    n = int(n)
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
    print(f"{fam} n={n}: {min(ts):.3f} ms  classes sum {sum(v[0] for v in prof.values()):.3f}")
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:16s} {v[0]:.4f} ms  {v[1:]}")
    s.close()
