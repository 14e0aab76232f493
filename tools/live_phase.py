"""Phase cycles of the few-merge live levels (BRGPU_LIB=tools/liblprof.so, -DBRGPU_LIVE_PROF)."""
import ctypes as C, sys
sys.path.insert(0, '.')
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
d, e = G.generate("sym-uniform", 1 << 20)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
for _ in range(2):
    s.eigvals_device(td, te)
cyc = (C.c_uint64 * 4)()
s._lib.brgpu_phase_cycles(s._h, cyc)
ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 64 + 32 + 16 + 8 + 4 + 2 + 1
print(f"per-CTA avg cycles over {ctas} CTAs:",
      {k: round(v / ctas) for k, v in zip(["deflation", "secular", "zhat", "rows+out"], cyc)})
