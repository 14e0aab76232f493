import os, sys, ctypes as C
sys.path.insert(0, '.')
os.environ["BRGPU_LIB"] = "tools/libdbg.so"
import torch, numpy as np
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
d, e = G.generate("sym-uniform", 1 << 20)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
s = br.Solver(0)
s.eigvals_device(td, te)
lib = s._lib
buf = (C.c_ulonglong * 16)()
lib.brgpu_debug_phases(buf)
s.eigvals_device(td, te)
lib.brgpu_debug_phases(buf)
names = ["load", "tol", "scatter", "flags+scan", "walk", "surv-compact", "secular", "zhat", "rows+defl"]
tot = sum(buf[i] for i in range(9))
for i, nm in enumerate(names):
    print(f"{nm:14s} {buf[i]/tot*100:6.1f}%")
