"""Requested eigenvector rows (Algorithm 1's sigma).

CPU part: the checker's rows (oracle.eigvals_rows) against LAPACK (numpy eigh):
with sigma = every row they form an eigenvector matrix Q of T, so T Q = Q diag(w)
and Q^T Q = I must hold to a few ulps on every family, including heavy
deflation (Toeplitz, glued Wilkinson), ties across irreducible blocks and
blocks <= the leaf cutoff; duplicates and order of sigma are pure gathers.
SPEC's split_row_request examples are checked verbatim.

GPU part: brgpu_eigvals_rows against the checker, BIT-EXACT (rows and
eigenvalues), and the eigenvalues equal those of the eigenvalue-only path.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2605_26599_b200 import generators as G


def _dense(d, e):
    return np.diag(d) + np.diag(e, 1) + np.diag(e, -1)


def _cases():
    rng = np.random.default_rng(11)
    out = []
    for fam, n in [("sym-uniform", 300), ("toeplitz121", 257), ("clustered", 200), ("normal", 120)]:
        out.append((f"{fam}-{n}",) + G.generate(fam, n))
    i = np.arange(315)
    out.append(("glued-wilkinson", np.abs(i % 21 - 10).astype(float),
                np.where((i[:-1] % 21) == 20, 1e-10, 1.0)))
    base_d, base_e = rng.uniform(-1, 1, 40), rng.uniform(-1, 1, 39)
    out.append(("tied-blocks", np.tile(base_d, 5), np.tile(np.r_[base_e, 0.0], 5)[:-1]))
    d, e = rng.uniform(-1, 1, 200), rng.uniform(-1, 1, 199)
    e[[3, 10, 11, 12, 150]] = 0.0  # blocks of 1..26 rows next to big ones
    out.append(("small-blocks", d, e))
    out.append(("leaf-only", rng.uniform(-1, 1, 20), rng.uniform(-1, 1, 19)))
    out.append(("n1", np.array([0.7]), np.zeros(0)))
    return out


CASES = _cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_checker_rows_are_eigenvectors(case):
    _, d, e = case
    n = len(d)
    w, Q = O.eigvals_rows(d, e, np.arange(n))
    assert np.array_equal(w, O.eigvals(d, e).w)  # rows do not perturb the eigenvalues
    T = _dense(d, e)
    nrm = max(G.inf_norm(d, e), 1e-300)
    assert np.max(np.abs(T @ Q - Q * w)) <= 64 * n * np.finfo(float).eps * nrm
    assert np.max(np.abs(Q.T @ Q - np.eye(n))) <= 64 * n * np.finfo(float).eps
    # against LAPACK, column by column up to sign, where eigenvalues are well separated
    wl, V = np.linalg.eigh(T)
    gap = np.minimum(np.r_[np.inf, np.diff(wl)], np.r_[np.diff(wl), np.inf])
    ok = gap > 1e-6 * nrm
    diff = np.minimum(np.abs(Q - V).max(0), np.abs(Q + V).max(0))
    assert np.all(diff[ok] <= 1e-9)


def test_checker_rows_duplicates_and_order():
    d, e = G.generate("sym-uniform", 100)
    sel = [5, 1, 5, 99, 0, 5]
    _, R = O.eigvals_rows(d, e, sel)
    _, Q = O.eigvals_rows(d, e, np.arange(100))
    for r, i in enumerate(sel):
        assert np.array_equal(R[r], Q[i])


def test_checker_rows_reject_bad_index():
    d, e = G.generate("sym-uniform", 50)
    with pytest.raises(O.OracleError):
        O.eigvals_rows(d, e, [50])
    with pytest.raises(O.OracleError):
        O.eigvals_rows(d, e, [-1])


def test_split_row_request_spec_examples():
    from paper_2605_26599_b200 import RowRequest, split_row_request
    # SPEC.md:331-333
    L, R = split_row_request((1, 5, 3), 3)
    assert L.sigma == (1, 3, 3) and R.sigma == (2, 1)
    L, R = split_row_request((), 2)
    assert L.sigma == (2,) and R.sigma == (1,)
    L, R = split_row_request(RowRequest((2, 2)), 4)
    assert L.sigma == (2, 2, 4) and R.sigma == (1,)


def test_split_row_request_matches_child_rows():
    """Merging the children's selected rows at their original positions
    reproduces the parent selection: with a zero cut, T =
    T_L (+) T_R, and each requested row of T is the row its child request
    returns, placed at the child's eigenvalues in the global order (bitwise:
    both blocks scale by 1)."""
    from paper_2605_26599_b200 import split_row_request
    rng = np.random.default_rng(3)
    dl, el = rng.uniform(-1, 1, 30), rng.uniform(-1, 1, 29)
    dr, er = rng.uniform(-1, 1, 34), rng.uniform(-1, 1, 33)
    sigma = (31, 2, 30, 64, 2)
    L, R = split_row_request(sigma, 30, size=64)
    assert L.sigma == (2, 30, 2, 30) and R.sigma == (1, 34, 1)  # boundary rows last
    wl, QL = O.eigvals_rows(dl, el, np.asarray(L.sigma) - 1)
    wr, QR = O.eigvals_rows(dr, er, np.asarray(R.sigma) - 1)
    w, Q = O.eigvals_rows(np.r_[dl, dr], np.r_[el, 0.0, er], np.asarray(sigma) - 1)
    order = np.argsort(np.r_[wl, wr], kind="stable")
    assert np.array_equal(w, np.r_[wl, wr][order])
    inv = np.empty(64, dtype=np.int64)
    inv[order] = np.arange(64)
    li = ri = 0
    for r, s_ in enumerate(sigma):
        want = np.zeros(64)
        if s_ <= 30:
            want[inv[:30]] = QL[li]
            li += 1
        else:
            want[inv[30:]] = QR[ri]
            ri += 1
        assert np.array_equal(Q[r], want)


# ------------------------------------------------------------------------------ GPU
GPU_CASES = [("sym-uniform", 1000), ("sym-uniform", 4096), ("toeplitz121", 2048), ("wilkinson", 3000),
             ("clustered", 1500), ("normal", 777), ("uniform", 26)]


@pytest.mark.gpu
@pytest.mark.parametrize("fam,n", GPU_CASES)
def test_gpu_rows_bitwise_vs_checker(solver, fam, n):
    d, e = G.generate(fam, n)
    rng = np.random.default_rng(n)
    sel = np.r_[0, n - 1, rng.integers(0, n, 6), n // 2, n // 2]
    w, R = solver.eigvals_rows(d, e, sel)
    wc, Rc = O.eigvals_rows(d, e, sel)
    assert np.array_equal(w, wc)
    assert np.array_equal(w, solver.eigvals(d, e))
    assert np.array_equal(R, Rc), f"max diff {np.max(np.abs(R - Rc)):.3e}"


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gpu_all_rows_bitwise(solver, case):
    _, d, e = case
    n = len(d)
    w, Q = solver.eigvals_rows(d, e, np.arange(n))
    wc, Qc = O.eigvals_rows(d, e, np.arange(n))
    assert np.array_equal(w, wc)
    assert np.array_equal(Q, Qc), f"max diff {np.max(np.abs(Q - Qc)):.3e}"


@pytest.mark.gpu
def test_gpu_rows_large_split_tier(solver):
    """n = 2^16 random: the top merges run the warp-per-root (split) tier."""
    d, e = G.generate("sym-uniform", 1 << 16)
    sel = np.array([0, 12345, 32767, 32768, 65535])
    w, R = solver.eigvals_rows(d, e, sel)
    wc, Rc = O.eigvals_rows(d, e, sel)
    assert np.array_equal(w, wc) and np.array_equal(R, Rc)
    assert np.allclose((R * R).sum(1), 1.0, atol=1e-12)  # rows of an orthogonal matrix


@pytest.mark.gpu
def test_gpu_rows_errors_and_plan_switch(solver):
    import paper_2605_26599_b200 as br
    d, e = G.generate("sym-uniform", 500)
    with pytest.raises(br.InvalidArgument):
        solver.eigvals_rows(d, e, [500])
    w0 = solver.eigvals(d, e)
    w1, _ = solver.eigvals_rows(d, e, [7])
    w2 = solver.eigvals(d, e)  # back to the cached eigenvalue-only plan
    assert np.array_equal(w0, w1) and np.array_equal(w0, w2)
    w3, R3 = solver.eigvals_rows(d, e, [])
    assert np.array_equal(w0, w3) and R3.shape == (0, 500)


@pytest.mark.gpu
@pytest.mark.parametrize("opts,chk", [(dict(zhat=False), dict(zhat=False)),
                                      (dict(patched_stop=False), dict(patched=False)),
                                      (dict(leaf_cutoff=8), dict(leaf_cutoff=8)),
                                      (dict(exact_passes=True), {})])
def test_gpu_rows_options(opts, chk):
    import paper_2605_26599_b200 as br
    d, e = G.generate("sym-uniform", 3000)
    sel = [0, 1, 1499, 1500, 2999, 1500]
    with br.Solver(0, br.BrOptions(**opts)) as s:
        w, R = s.eigvals_rows(d, e, sel)
    wc, Rc = O.eigvals_rows(d, e, sel, **chk)
    assert np.array_equal(w, wc) and np.array_equal(R, Rc)


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [2.0 ** -1040, 2.0 ** 1000])
def test_gpu_rows_extreme_scales(solver, scale):
    d, e = G.generate("sym-uniform", 2000)
    d, e = d * scale, e * scale
    sel = [3, 1000, 1999]
    w, R = solver.eigvals_rows(d, e, sel)
    wc, Rc = O.eigvals_rows(d, e, sel)
    assert np.array_equal(w, wc) and np.array_equal(R, Rc)
    assert np.allclose((R * R).sum(1), 1.0, atol=1e-12)


@pytest.mark.gpu
def test_gpu_rows_leaf_cutoff_32():
    import paper_2605_26599_b200 as br
    d, e = G.generate("sym-uniform", 2500)
    e[[40, 41, 100]] = 0.0  # blocks of 1 and 59 rows beside the big one
    sel = [0, 40, 41, 60, 2499]
    with br.Solver(0, br.BrOptions(leaf_cutoff=32)) as s:
        w, R = s.eigvals_rows(d, e, sel)
    wc, Rc = O.eigvals_rows(d, e, sel, leaf_cutoff=32)
    assert np.array_equal(w, wc) and np.array_equal(R, Rc)
