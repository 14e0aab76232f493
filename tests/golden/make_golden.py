"""Generate tests/golden/reference_vectors.npz from the REFERENCE itself.

Runs the unmodified reference building blocks compiled from /root/reference
(oracle/_ref/libbrref.so: the SPEC.md:312-380 driver composed from
leaf_eig / build_z / deflate_merge / apply_prep_to_rows / solve_root /
refreshed_weights / secular_column / dot, plus eigenvalues_qrql and the Jacobi
dense_eig) on fixed inputs and stores inputs and outputs.  Run in the build
container (where /root/reference exists); the .npz is committed and is what the
GPU box checks against.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

CASES = []
for fam in ["sym-uniform", "uniform", "normal", "toeplitz", "toeplitz121", "clustered", "wilkinson"]:
    for n in [1, 2, 3, 5, 25, 26, 27, 51, 64, 100, 257, 512, 1000]:
        CASES.append((fam, n))


def special_cases():
    rng = np.random.default_rng(12345)
    out = []
    # exact zero couplings -> several irreducible blocks (tridiagonal.cpp:45-58)
    d = rng.uniform(-1, 1, 300); e = rng.uniform(-1, 1, 299); e[[10, 40, 41, 200]] = 0.0
    out.append(("zeros-e", d, e))
    # all off-diagonals zero: n blocks of size 1
    out.append(("diag-only", rng.uniform(-1, 1, 80), np.zeros(79)))
    # negative couplings (split_sign = -1 everywhere)
    out.append(("neg-e", rng.uniform(-1, 1, 200), -np.abs(rng.uniform(0.1, 1, 199))))
    # constant diagonal, tiny coupling: heavy close-pole deflation
    out.append(("const-d", np.ones(160), np.full(159, 1e-9)))
    # repeated identical blocks glued weakly (mirror spectra)
    blk = rng.uniform(-1, 1, 33)
    d = np.tile(blk, 6); e = np.full(len(d) - 1, 0.5); e[32::33] = 1e-7
    out.append(("mirror", d, e))
    # large magnitudes (block scaling)
    out.append(("scaled", 1e6 * rng.uniform(-1, 1, 150), 1e6 * rng.uniform(-1, 1, 149)))
    # tiny magnitudes
    out.append(("tiny", 1e-6 * rng.uniform(-1, 1, 150), 1e-6 * rng.uniform(-1, 1, 149)))
    return out


def main() -> None:
    store: dict[str, np.ndarray] = {}
    names = []
    for fam, n in CASES:
        d, e = G.generate(fam, n)
        names.append(f"{fam}:{n}")
        key = f"c{len(names) - 1}"
        store[key + "_d"] = d
        store[key + "_e"] = e
        store[key + "_br"] = O.ref_eigvals(d, e, threads=1)
        if n <= 512:
            store[key + "_qrql"] = O.ref_qrql(d, e)
        if n <= 257:
            store[key + "_dense"] = O.ref_dense(d, e)
    for name, d, e in special_cases():
        names.append(name)
        key = f"c{len(names) - 1}"
        store[key + "_d"] = d
        store[key + "_e"] = e
        store[key + "_br"] = O.ref_eigvals(d, e, threads=1)
        store[key + "_qrql"] = O.ref_qrql(d, e)
    # secular micro-cases: reference solve_root (unpatched) on random problems
    rng = np.random.default_rng(7)
    sec = []
    for t in range(40):
        k = int(rng.integers(1, 40))
        dd = np.sort(rng.uniform(-1, 1, k))
        dd = np.unique(dd)
        k = len(dd)
        z = rng.uniform(-1, 1, k)
        rho = float(rng.uniform(0.05, 2))
        for j in range(k):
            o, tau = O.ref_solve_root(dd, z, rho, j)
            sec.append((t, j, o, tau))
        store[f"s{t}_d"] = dd
        store[f"s{t}_z"] = z
        store[f"s{t}_rho"] = np.array([rho])
    store["sec_roots"] = np.array([(a, b, c) for a, b, c, _ in sec], dtype=np.int64)
    store["sec_tau"] = np.array([x for *_, x in sec])
    store["names"] = np.array(names)
    np.savez_compressed(Path(__file__).parent / "reference_vectors.npz", **store)
    print(f"{len(names)} solver cases, {len(sec)} secular roots")


if __name__ == "__main__":
    main()
