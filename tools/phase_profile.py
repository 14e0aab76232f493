"""Phase split of the fused level kernels (build with -DBRGPU_PHASE_PROF; run with
BRGPU_LIB=tools/libphase.so): SM-cycle shares of deflation / secular / refreshed
weights / rows + placement, and the FP64 fraction of each phase when its share of
the fused kernels' time is applied to the algorithmic work of that phase."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "sym-uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
peak = float(sys.argv[3]) if len(sys.argv) > 3 else 17.1e12
d, e = G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
for _ in range(3):
    s.eigvals_device(td, te)
s.set_trace(True)
s.eigvals_device(td, te)
st = s.stats()
s.set_trace(False)
s.eigvals_device(td, te)
cyc = (C.c_uint64 * 4)()
assert s._lib.brgpu_phase_cycles(s._h, cyc) == 0
prof = s.profile_kernels(td, te)
fused_ms = prof.get("fused_level", (0.0, 0))[0]
tot = sum(cyc)
shares = [c / tot for c in cyc] if tot else [0] * 4
ops = {"secular": 11 * st["pole_terms_fused"], "zhat": 10 * st["k2_nonroot_fused"],
       "rows": 11 * st["k2_nonroot_fused"]}
out = {"config": f"{fam} n={n}", "fused_ms": fused_ms,
       "phase_share": dict(zip(["deflation", "secular", "zhat", "rows+placement"], shares))}
for k, i in (("secular", 1), ("zhat", 2), ("rows", 3)):
    t = shares[i] * fused_ms * 1e-3
    out[f"{k}_fp64_frac"] = ops[k] / t / peak if t > 0 else None
print(json.dumps(out))
