"""One requested-rows solve at n = 2^20, 16 rows (for an ncu launch list)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

s = br.Solver(0)
d, e = G.generate("sym-uniform", 1 << 20)
sel = np.linspace(0, (1 << 20) - 1, int(sys.argv[1]) if len(sys.argv) > 1 else 16).astype(np.int64)
s.eigvals_rows(d, e, sel)
