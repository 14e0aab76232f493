"""Pin the CPU checker (oracle/br_oracle.c) before trusting it.

1. Against the committed golden vectors produced by the reference itself
   (tests/golden/make_golden.py -> oracle/_ref, the unmodified reference blocks):
   the restatement in reference-arithmetic mode must reproduce the reference's
   eigenvalues BIT FOR BIT, and its secular roots (unpatched stop) bit for bit.
2. Against the live reference library when it is present (this container).
3. The GPU-arithmetic mode (the product's specification, tau-relative stop)
   must sit within the BASELINE tolerance 8 n eps ||T|| of LAPACK dsterf
   (scipy) and of the dense Jacobi oracle.
4. SPEC.md known-answer examples.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import scipy.linalg as sl

import oracle as O
from paper_2605_26599_b200 import generators as G

GOLD = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")
NAMES = [str(x) for x in GOLD["names"]]


def _case(i):
    return GOLD[f"c{i}_d"], GOLD[f"c{i}_e"]


@pytest.mark.parametrize("i", range(len(NAMES)), ids=NAMES)
def test_refmode_matches_reference_golden_bitwise(i):
    d, e = _case(i)
    w = O.eigvals(d, e, ref_arith=True, patched=False, threads=1).w
    ref = GOLD[f"c{i}_br"]
    assert np.array_equal(w, ref), f"max diff {np.max(np.abs(w - ref))}"


@pytest.mark.parametrize("i", range(len(NAMES)), ids=NAMES)
def test_gpu_arith_within_tolerance_of_lapack(i):
    d, e = _case(i)
    n = len(d)
    w = O.eigvals(d, e, threads=1).w
    assert np.all(np.diff(w) >= 0)
    tol = G.tolerance(d, e)
    truth = sl.eigvalsh_tridiagonal(d, e) if n > 1 else d
    assert np.max(np.abs(w - truth)) <= tol
    if f"c{i}_dense" in GOLD:  # reference Jacobi oracle (oracle_jacobi.cpp:144-157)
        assert np.max(np.abs(w - GOLD[f"c{i}_dense"])) <= tol
    if f"c{i}_qrql" in GOLD:  # reference eigenvalues_qrql (qrql.cpp:386-394)
        assert np.max(np.abs(w - GOLD[f"c{i}_qrql"])) <= tol


def test_secular_roots_match_reference_bitwise():
    roots = GOLD["sec_roots"]
    taus = GOLD["sec_tau"]
    for (t, j, o), tau in zip(roots, taus):
        d, z, rho = GOLD[f"s{t}_d"], GOLD[f"s{t}_z"], float(GOLD[f"s{t}_rho"][0])
        og, tg, _ = O.solve_root(d, z, rho, int(j), patched=False, ref_arith=True)
        assert og == o and tg == tau


def test_patched_stop_keeps_tau_relative_accuracy():
    # near-pole roots: the tau-relative stop must give tau to ~ulp relative accuracy
    d = np.array([0.0, 1e-3, 1.0, 2.0])
    z = np.array([1e-9, 0.5, 0.5, 0.5])
    for j in range(4):
        o, tau, _ = O.solve_root(d, z, 1.0, j, patched=True)
        # residual of the secular function at the root, in the shifted variable
        lam_delta = (d - d[o]) - tau
        f = 1.0 + np.sum(z * z / lam_delta)
        assert abs(f) < 1e-10 * (1 + np.sum(np.abs(z * z / lam_delta)))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("fam", ["sym-uniform", "uniform", "toeplitz121", "wilkinson", "clustered"])
@pytest.mark.parametrize("n", [64, 1000, 4096])
def test_refmode_matches_live_reference(fam, n):
    d, e = G.generate(fam, n)
    assert np.array_equal(O.eigvals(d, e, ref_arith=True, patched=False, threads=1).w,
                          O.ref_eigvals(d, e, threads=1))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_leaf_matches_reference_leaf_eig():
    rng = np.random.default_rng(3)
    for m in [1, 2, 3, 7, 16, 25]:
        for _ in range(10):
            d, e = rng.uniform(-1, 1, m), rng.uniform(-1, 1, max(m - 1, 0))
            lam, blo, bhi = O.leaf(d, e, ref_arith=True)
            rl, rb, rh = O.ref_leaf(d, e)
            assert np.array_equal(lam, rl)
            # eigenvector column signs are canonicalised by the reference only
            assert np.array_equal(np.abs(blo), np.abs(rb)) and np.array_equal(np.abs(bhi), np.abs(rh))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_deflation_matches_reference():
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(2, 60))
        d = np.round(rng.uniform(-1, 1, n), 2)  # ties and close poles
        z = rng.uniform(-1, 1, n) * (rng.uniform(0, 1, n) > 0.2)
        a = O.deflate(d, z, ref_arith=True)
        b = O.ref_deflate(d, z)
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_refreshed_weights_match_reference():
    rng = np.random.default_rng(9)
    for _ in range(20):
        k = int(rng.integers(1, 30))
        d = np.unique(rng.uniform(-1, 1, k))
        k = len(d)
        z = rng.uniform(-1, 1, k)
        roots = [O.solve_root(d, z, 0.7, j, patched=True, ref_arith=True) for j in range(k)]
        org = [r[0] for r in roots]
        tau = [r[1] for r in roots]
        a = O.refreshed_weights(d, z, org, tau, ref_arith=True)
        b = O.ref_refreshed_weights(d, z, 0.7, org, tau)
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ SPEC known answers
def test_spec_secular_2x2():
    # SPEC.md:264-266 / acceptance 8: D=[0,2], z=[1/sqrt2, 1/sqrt2], rho=1 -> (3 +- sqrt5)/2
    d = np.array([0.0, 2.0])
    z = np.array([1.0, 1.0]) / np.sqrt(2.0)
    lam = [d[o] + t for o, t, _ in (O.solve_root(d, z, 1.0, j) for j in range(2))]
    assert np.allclose(lam, [(3 - np.sqrt(5)) / 2, (3 + np.sqrt(5)) / 2], atol=1e-15)


def test_spec_deflation_examples():
    # SPEC.md:194-196
    da, za, df, nrot, _ = O.deflate([1.0, 3.0], [0.0, 0.5])
    assert list(da) == [3.0] and list(za) == [0.5] and list(df) == [1.0]
    da, za, df, nrot, _ = O.deflate([2.0, 2.0], [3.0, 4.0])
    assert list(da) == [2.0] and za[0] == pytest.approx(5.0) and nrot == 1 and list(df) == [2.0]
    da, za, df, nrot, _ = O.deflate([0.0, 2.0], [1.0, 1.0])
    assert len(da) == 2 and nrot == 0


def test_spec_qrql_examples():
    # SPEC.md:129-131
    assert list(O.qrql([5.0], [])) == [5.0]
    assert np.allclose(O.qrql([2.0, 2.0], [0.25]), [1.75, 2.25], atol=1e-15)
    k = np.arange(1, 5)
    assert np.allclose(O.qrql(np.full(4, 2.0), np.full(3, 0.25)), np.sort(2 + 0.5 * np.cos(k * np.pi / 5)),
                       atol=1e-15)


def test_spec_toeplitz_analytic_n1024():
    # acceptance criterion 3: Toeplitz(0.25, 2, 0.25), n = 1024, <= 1e-12
    n = 1024
    d, e = G.generate("toeplitz", n)
    k = np.arange(1, n + 1)
    exact = np.sort(2 + 0.5 * np.cos(k * np.pi / (n + 1)))
    assert np.max(np.abs(O.eigvals(d, e).w - exact)) <= 1e-12


def test_spec_br_examples():
    # SPEC.md:345-347, 354-356
    assert list(O.eigvals([3.0], []).w) == [3.0]
    d = np.full(4, 2.0)
    e = np.full(3, 0.25)
    k = np.arange(1, 5)
    assert np.allclose(O.eigvals(d, e, leaf_cutoff=5).w, np.sort(2 + 0.5 * np.cos(k * np.pi / 5)))


def test_determinism_thread_count():
    # SPEC.md:362 / acceptance 5: bitwise identical for 1 vs max workers
    d, e = G.generate("sym-uniform", 20000)
    a = O.eigvals(d, e, threads=1).w
    b = O.eigvals(d, e, threads=0).w
    assert np.array_equal(a, b)


def test_sturm_certificate_sample():
    d, e = G.generate("sym-uniform", 30000)
    w = O.eigvals(d, e).w
    tol = G.tolerance(d, e)
    for i in np.linspace(0, len(w) - 1, 25).astype(int):
        assert O.sturm_count(d, e, w[i] - tol) <= i
        assert O.sturm_count(d, e, w[i] + tol) >= i + 1


@pytest.mark.parametrize("fam,n", [("sym-uniform", 2000), ("wilkinson", 1000), ("clustered", 800)])
@pytest.mark.parametrize("scale", [2.0 ** -1010, 2.0 ** -1040, 2.0 ** 1000])
def test_gpu_arith_extreme_scales(fam, n, scale):
    """GPU mode lifts tiny blocks by an exact power of two (block scale rule), so
    tiny and huge matrices keep the relative tolerance; the reference's max(.,1)
    rule never enlarges a block and overflows the boundary-row sums instead."""
    d, e = G.generate(fam, n)
    d, e = d * scale, e * scale
    w = O.eigvals(d, e, threads=1).w
    assert np.all(np.isfinite(w))
    truth = sl.eigvalsh_tridiagonal(d / scale, e / scale) * scale
    assert np.max(np.abs(w - truth)) <= G.tolerance(d, e) * (1 + 1e-12) + 64 * 2.0 ** -1074


CG = np.load(Path(__file__).parent / "golden" / "config_vectors.npz")
CNAMES = [str(x) for x in CG["names"]]


@pytest.mark.parametrize("key", CNAMES)
def test_checker_pinned_at_config_sizes(key):
    """BASELINE config 1 (sym-uniform:4096) and every family at 2048 / 4096
    (tests/golden/config_vectors.npz, from the reference itself): reference-arithmetic
    mode reproduces the reference BR composition bit for bit; the product's
    arithmetic is within 8 n eps ||T|| of the reference's qrql and Jacobi solvers."""
    fam, n = key.split(":")
    d, e = G.generate(fam, int(n))
    assert np.array_equal(O.eigvals(d, e, ref_arith=True, patched=False).w, CG[key + ":br"])
    w = O.eigvals(d, e).w
    tol = G.tolerance(d, e)
    assert np.max(np.abs(w - CG[key + ":qrql"])) <= tol
    if key + ":dense" in CG:
        assert np.max(np.abs(w - CG[key + ":dense"])) <= tol
