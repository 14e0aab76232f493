import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
d, e = G.generate("sym-uniform", 1 << 20)
s = br.Solver(0)
n = len(d)
hd = torch.from_numpy(d).pin_memory(); he = torch.from_numpy(e).pin_memory(); hw = torch.empty(n, dtype=torch.float64).pin_memory()
for _ in range(5): s._lib.brgpu_eigvals(s._h, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr())
ts = []
for _ in range(50):
    t0 = time.perf_counter(); s._lib.brgpu_eigvals(s._h, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr()); ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e3
print(f"e2e ms: min {ts.min():.3f} median {np.median(ts):.3f} mean {ts.mean():.3f} max {ts.max():.3f}")
x = torch.empty(n * 2, dtype=torch.float64, device="cuda"); hx = torch.empty(n * 2, dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
for name, f in [("h2d 16MB", lambda: x.copy_(hx, non_blocking=True)), ("d2h 8MB", lambda: hx[:n].copy_(x[:n], non_blocking=True))]:
    ts = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, f"{np.median(ts)*1e3:.3f} ms")
print("device", s.timing())
