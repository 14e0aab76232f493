"""Device ms of a batched solve, live tier on vs off: tools/ab_batch.py batch n"""
import sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2605_26599_b200 as br
batch, n = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
d = torch.tensor(rng.uniform(-1, 1, (batch, n)), device="cuda")
e = torch.tensor(rng.uniform(-1, 1, (batch, n - 1)), device="cuda")
for rep in range(2):
    for live in (True, False):
        s = br.Solver(0, br.BrOptions(live=live))
        for _ in range(3): s.eigvals_batched_device(d, e)
        ts = []
        for _ in range(10):
            s.eigvals_batched_device(d, e)
            ts.append(s.timing()["device_ms"])
        print(f"batch {batch} x {n} live={live}: {statistics.mean(ts):.3f} ms (min {min(ts):.3f})", flush=True)
        s.close()
