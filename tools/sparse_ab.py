"""Sparse vs dense grid levels: bit-identity and device time on a set of inputs.
python tools/sparse_ab.py [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cases = [("sym-uniform", 1 << 20, {}), ("sym-uniform", 4096, {}), ("sym-uniform", 100000, {}),
         ("sym-uniform", 1 << 17, {}), ("wilkinson", 1 << 18, {}), ("wilkinson", 1 << 18, {"glue": 2.0 ** -26}),
         ("toeplitz121", 1 << 16, {}), ("normal", 300001, {}), ("clustered", 1 << 16, {}),
         ("uniform", 1 << 16, {})]
bad = 0
for fam, n, kw in cases:
    try:
        d, e = G.generate(fam, n, **kw)
    except Exception as ex:  # noqa: BLE001
        print(fam, n, "skip", ex)
        continue
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    res = {}
    for sp in (False, True):
        s = br.Solver(0, br.BrOptions(sparse=sp))
        w = s.eigvals_device(td, te)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            w = s.eigvals_device(td, te)
            torch.cuda.synchronize()
            ts.append(s.timing()["device_ms"])
        res[sp] = (w.cpu().numpy(), min(ts), s.stats()["kernel_launches"])
        s.close()
    same = np.array_equal(res[False][0], res[True][0])
    nd = int(np.sum(res[False][0] != res[True][0]))
    bad += not same
    print(f"{fam:12s} n={n:8d} {kw} identical={same} ndiff={nd} dense {res[False][1]:.3f} ms "
          f"({res[False][2]} launches)  sparse {res[True][1]:.3f} ms ({res[True][2]} launches)", flush=True)
print("MISMATCHES", bad)
