"""Debug: state after the first k levels, dense vs sparse (BRGPU_DEBUG_STOP_LEVEL)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
fam = sys.argv[1]; n = int(sys.argv[2])
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
for k in range(1, 20):
    os.environ["BRGPU_DEBUG_STOP_LEVEL"] = str(k)
    r = []
    for sp in (0, 1):
        s = br.Solver(0, br.BrOptions(sparse=bool(sp), use_graph=False))
        try:
            r.append(s.eigvals_device(td, te).cpu().numpy())
        except Exception as ex:
            r.append(None); print(k, sp, "ERR", ex)
        s.close()
    if r[0] is None or r[1] is None: break
    dif = np.nonzero(r[0] != r[1])[0]
    print("levels", k, "identical", len(dif) == 0, len(dif), dif[:10], flush=True)
    if len(dif):
        i = dif[0]
        print(" dense", r[0][max(0,i-3):i+4]); print(" sparse", r[1][max(0,i-3):i+4])
        break
