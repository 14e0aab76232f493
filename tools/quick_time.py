"""Device ms (best of R) of the default solver on a few BASELINE configs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
R = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cases = [("c5", "sym-uniform", 1 << 20, {}), ("c1", "sym-uniform", 4096, {}), ("c3", "toeplitz121", 1 << 16, {}),
         ("c4", "wilkinson", 1 << 18, {}), ("c4s", "wilkinson", 1 << 18, {"glue": 2.0 ** -26})]
for name, fam, n, kw in cases:
    d, e = G.generate(fam, n, **kw)
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    s = br.Solver(0)
    for _ in range(3):
        s.eigvals_device(td, te)
    ts = []
    for _ in range(R):
        s.eigvals_device(td, te)
        torch.cuda.synchronize()
        ts.append(s.timing()["device_ms"])
    ts.sort()
    print(f"{name} n={n} best {ts[0]:.3f} ms median {ts[len(ts)//2]:.3f} ms", flush=True)
    s.close()
