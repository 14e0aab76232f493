"""A/B of one BrOptions field inside one process: device ms per variant and bitwise equality.

python tools/ab_opt.py FIELD [family] [n] [reps]   e.g.  tools/ab_opt.py live_cluster sym-uniform 1048576
"""
import dataclasses
import statistics
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

field = sys.argv[1]
fam = sys.argv[2] if len(sys.argv) > 2 else "sym-uniform"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
out = {}
for rnd in range(2):
    for v in (True, False):
        s = br.Solver(0, dataclasses.replace(br.BrOptions(), **{field: v}))
        for _ in range(3):
            w = s.eigvals_device(td, te)
        ts = []
        for _ in range(reps):
            w = s.eigvals_device(td, te)
            ts.append(s.timing()["device_ms"])
        out[v] = w.cpu().numpy()
        prof = s.profile_kernels(td, te)
        top = sorted(prof.items(), key=lambda kv: -kv[1][0])[:5]
        print(f"{field}={v!s:5s} {fam} n={n}: {statistics.mean(ts):.3f} ms (min {min(ts):.3f} med {statistics.median(ts):.3f})  ",
              "  ".join(f"{k}={v2[0]:.3f}" for k, v2 in top), flush=True)
        s.close()
print("bitwise equal:", bool(np.array_equal(out[True], out[False])))
