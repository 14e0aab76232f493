"""Theorem 1 (Algorithm 1): every boundary-row merge hands
deflation the same secular problem a full-eigenvector D&C would -- the poles are the
children's eigenvalues and z = (sign * last row of Q_L, first row of Q_R) is formed from
the children's true eigenvectors -- although BR never stores Q.  Checked on the CPU
restatement (which the GPU reproduces bit for bit, tests/test_gpu_parity.py) against
dense eigendecompositions of every child: poles to 1e-13 ||T||, and z to 1e-11 through its
eigenspace-invariant part (the squared norm of z over each group of equal child
eigenvalues, so column signs and rotations inside clusters do not matter)."""
import numpy as np
import pytest

import oracle as O
from paper_2605_26599_b200 import generators as G


def internal_nodes(n, cutoff=25):
    """(offset, size) of every internal node -- merge_tree.cpp:34-60 (split at size // 2)."""
    out = []

    def rec(o, sz):
        if sz <= cutoff:
            return
        out.append((o, sz))
        nl = sz // 2
        rec(o, nl)
        rec(o + nl, sz - nl)

    rec(0, n)
    return out


def child_diagonal(d, e, nodes, off, size):
    """Diagonal of the child matrix at (off, size): the Cuppen cuts of its ancestors
    only (merge_tree.cpp:62-76) -- the cuts inside the child belong to its subtree."""
    dc = d.copy()
    for o, sz in nodes:
        if o <= off and off + size <= o + sz and (o, sz) != (off, size):
            m = o + sz // 2 - 1
            rho = abs(e[m])
            dc[m] -= rho
            dc[m + 1] -= rho
    return dc


def child_eig(dc, e, off, size):
    T = np.diag(dc[off:off + size]) + np.diag(e[off:off + size - 1], 1) + np.diag(e[off:off + size - 1], -1)
    return np.linalg.eigh(T)


def groups(lam, gap):
    """Index groups of consecutive sorted values closer than gap."""
    out, cur = [], [0]
    for i in range(1, len(lam)):
        if lam[i] - lam[i - 1] <= gap:
            cur.append(i)
        else:
            out.append(cur)
            cur = [i]
    out.append(cur)
    return out


@pytest.mark.parametrize("fam,n", [("uniform", 256), ("normal", 200), ("toeplitz", 256), ("sym-uniform", 240),
                                   ("clustered", 128), ("wilkinson", 210)])
def test_br_merges_equal_full_dc(fam, n):
    d0, e0 = G.generate(fam, n)
    # the solver works on the block scaled by max(|d|, |e|, 1); one block here
    sc = max(float(np.max(np.abs(d0))), float(np.max(np.abs(e0))), 1.0)
    d, e = d0 / sc, e0 / sc
    tn = float(np.max(np.abs(d) + np.r_[np.abs(e), 0] + np.r_[0, np.abs(e)]))
    nodes = internal_nodes(n)
    recs = O.merge_inputs(d0, e0)
    assert recs, "no merges"
    for off, size, nl, D, z in recs:
        lamL, QL = child_eig(child_diagonal(d, e, nodes, off, nl), e, off, nl)
        lamR, QR = child_eig(child_diagonal(d, e, nodes, off + nl, size - nl), e, off + nl, size - nl)
        sign = -1.0 if e[off + nl - 1] < 0 else 1.0
        poles = np.concatenate([lamL, lamR])
        zf = np.concatenate([sign * QL[-1, :], QR[0, :]])
        order = np.argsort(poles, kind="stable")
        poles, zf = poles[order], zf[order]
        assert np.max(np.abs(D - poles)) <= 1e-13 * tn, (off, size)
        for g in groups(poles, 1e-7 * tn):
            # z carries the accumulated rounding of the boundary rows below this merge
            assert abs(np.sum(z[g] ** 2) - np.sum(zf[g] ** 2)) <= 1e-11, (off, size, g[:3])


@pytest.mark.parametrize("fam,n", [("uniform", 256), ("toeplitz", 256), ("clustered", 128), ("sym-uniform", 4096)])
def test_full_dc_restatement_matches_checker(fam, n):
    """oracle/full_dc.py (the conventional D&C of the GPU Theorem 1 check,
    tests/test_theorem1_gpu.py): same deflation decisions at every merge as the
    checker, eigenvalues within a few ulps of ||T||."""
    from oracle.full_dc import full_dc_trace
    d, e = G.generate(fam, n)
    lam, recs = full_dc_trace(d, e)
    r = O.eigvals(d, e, trace=True, threads=1)
    tr = sorted(r.trace, key=lambda t: (t[0], t[2]))
    assert [t[5] for t in tr] == [x[3] for x in recs]
    tn = float(np.max(np.abs(d) + np.r_[np.abs(e), 0] + np.r_[0, np.abs(e)]))
    assert np.max(np.abs(lam - r.w)) <= 64 * 2.0 ** -52 * tn
