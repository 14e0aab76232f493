"""Per-launch-group device times of one solve (events between launches, no graph):
    BRGPU_PROF_DUMP=1 python tools/prof_dump.py [family] [n] [batch]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("BRGPU_PROF_DUMP", "1")
import torch  # noqa: E402

import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "sym-uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 0
d, e = G.generate_batch(fam, batch, n) if batch else G.generate(fam, n)
td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
with br.Solver(0) as s:
    for _ in range(3):
        (s.eigvals_batched_device(td, te) if batch else s.eigvals_device(td, te))
    torch.cuda.synchronize()
    s.profile_kernels(td, te, batch)
    s.profile_kernels(td, te, batch)
    (s.eigvals_batched_device(td, te) if batch else s.eigvals_device(td, te))
    torch.cuda.synchronize()
    print("graph device ms", s.timing())
