"""The opt-in sparse grid tier (BRGPU_OPT_SPARSE, csrc/sparse.cu) against the
checker and against the dense grid tier: bit-exact eigenvalues, identical
per-merge deflation traces, stable across the profile-driven re-planning of the
second solve, and the dense fallback on levels whose merges keep more than C
non-negligible poles (Toeplitz)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sparse_solver():
    s = br.Solver(0, br.BrOptions(sparse=True))
    yield s
    s.close()


@pytest.mark.parametrize("fam", ["sym-uniform", "normal", "uniform", "wilkinson", "clustered", "toeplitz121"])
@pytest.mark.parametrize("n", [4096, 20000, 65536])
def test_sparse_bitwise_vs_checker(sparse_solver, fam, n):
    d, e = G.generate(fam, n)
    ref = O.eigvals(d, e).w
    for _ in range(2):  # the second solve runs the re-planned configuration
        w = sparse_solver.eigvals(d, e)
        assert np.array_equal(w, ref), f"max diff {np.max(np.abs(w - ref)):.3e}"


@pytest.mark.parametrize("fam,n", [("sym-uniform", 100000), ("normal", 300001), ("wilkinson", 1 << 18)])
def test_sparse_matches_dense(sparse_solver, solver, fam, n):
    d, e = G.generate(fam, n)
    sparse_solver.set_trace(True)
    solver.set_trace(True)
    try:
        for _ in range(2):
            ws = sparse_solver.eigvals(d, e)
            wd = solver.eigvals(d, e)
            assert np.array_equal(ws, wd)
            assert sparse_solver.trace() == solver.trace()
    finally:
        sparse_solver.set_trace(False)
        solver.set_trace(False)


def test_sparse_c5(sparse_solver, solver):
    d, e = G.generate("sym-uniform", 1 << 20)
    for _ in range(2):
        assert np.array_equal(sparse_solver.eigvals(d, e), solver.eigvals(d, e))


def test_sparse_batched(sparse_solver):
    d, e = G.generate_batch("sym-uniform", 64, 1024)
    w = sparse_solver.eigvals_batched(d, e)
    for b in (0, 17, 63):
        assert np.array_equal(w[b], O.eigvals(d[b], e[b]).w)
