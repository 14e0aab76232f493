"""Generate tests/golden/config_vectors.npz from the REFERENCE itself at the
BASELINE sizes the reference can still run in seconds to minutes.

* every golden family at n = 2048 and 4096 (BASELINE config 1 is sym-uniform
  n = 4096): the reference BR composition (oracle/_ref: the unmodified
  /root/reference/proj/src blocks composed per SPEC.md:312-380) and the shipped
  ``br::eigenvalues_qrql`` (proj/src/qrql.cpp:386-394);
* the reference's Jacobi ``dense_eig`` (proj/src/oracle_jacobi.cpp) at n = 2048
  for every family and at n = 4096 for config 1 (SPEC.md:597 names qrql / the
  dense oracle as the truth for n <= 65536; Jacobi at 4096 takes ~70 s here,
  too slow for a test, so it is frozen as a fixture).

Inputs are not stored: they are regenerated bit for bit by
paper_2605_26599_b200.generators (xorshift64*).  Run in the build
container (where /root/reference exists); the .npz is committed.

    python tests/golden/make_config_golden.py
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

FAMILIES = ["sym-uniform", "uniform", "normal", "toeplitz", "toeplitz121", "clustered", "wilkinson"]
SIZES = [2048, 4096]


def main() -> None:
    store: dict[str, np.ndarray] = {}
    names = []
    for fam in FAMILIES:
        for n in SIZES:
            d, e = G.generate(fam, n)
            key = f"{fam}:{n}"
            names.append(key)
            t0 = time.time()
            store[key + ":br"] = O.ref_eigvals(d, e, threads=1)
            store[key + ":qrql"] = O.ref_qrql(d, e)
            if n == 2048 or (fam == "sym-uniform" and n == 4096):
                store[key + ":dense"] = O.ref_dense(d, e)
            print(f"{key}: {time.time() - t0:.1f} s", flush=True)
    store["names"] = np.array(names)
    out = Path(__file__).parent / "config_vectors.npz"
    np.savez_compressed(out, **store)
    print(out, out.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
