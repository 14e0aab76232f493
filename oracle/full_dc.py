"""Conventional full-eigenvector divide and conquer -- TEST INFRASTRUCTURE ONLY.

The Theorem 1 check (PAPER.md: "constructs the same secular problem as
conventional D&C"; SPEC.md:403-420 full_dc_eigen / compare_traces, acceptance
criterion 2 at SPEC.md:611): every node's FULL eigenvector matrix is
materialised, and each merge's secular problem (rho, D_active, z_active, K) is
built from the last row of Q_L and the first row of Q_R -- where the BR path
only ever carried those two rows.

Same split tree (merge_tree.cpp:34-60), Cuppen cuts, leaf QL/QR (the checker's
sweeps with every row tracked, oracle.leaf_full), deflation rule and close-pole
group arithmetic (the checker's deflate_walk, applied to whole columns),
secular roots and refreshed weights (the checker's solve_root /
refreshed_weights), and parent ordering as the BR driver; the parent matrix is
Q_parent = blockdiag(Q_L, Q_R) P G U with U formed explicitly and multiplied
with BLAS -- independent of the BR path's streamed boundary-row dots, so the
per-merge agreement is a real check, not an identity.  The reference declares
full_dc_eigen (proj/include/br/oracle.hpp:53) but ships no implementation.
Single irreducible block, lane (non-split) arithmetic: n <= 8192.
"""
from __future__ import annotations

import numpy as np

from . import leaf_full, refreshed_weights, solve_root

U_RND = 2.0 ** -53


def _walk(D, Z, X, tol):
    """The checker's deflate_walk (GPU arithmetic) on whole columns: D, Z in
    merged order, X (rows x n) the merged columns; returns (act, defl)."""
    n = len(D)
    act, defl = [], []
    prev, L = -1, 0
    Q = 0.0
    S = None

    def close():
        if prev >= 0 and L > 0:
            R = np.sqrt(Q)
            iR = 1.0 / R
            Z[prev] = R
            X[:, prev] = S * iR

    for k in range(n):
        if abs(Z[k]) <= tol:
            defl.append(k)
            continue
        if prev >= 0 and abs(D[k] - D[prev]) <= tol:
            zk = Z[k]
            xk = X[:, k].copy()
            Qn = Q + zk * zk
            rp, Rn = np.sqrt(Q), np.sqrt(Qn)
            irp, iRn = 1.0 / rp, 1.0 / Rn
            c, sn = rp * iRn, zk * iRn
            X[:, k] = c * xk - sn * (S * irp)
            Q = Qn
            S = S + zk * xk
            Z[k] = 0.0
            L += 1
            defl.append(k)
            continue
        close()
        prev = k
        act.append(k)
        zs = Z[k]
        L = 0
        Q = zs * zs
        S = zs * X[:, k]
    close()
    return np.array(act, dtype=int), np.array(defl, dtype=int)


def full_dc_trace(d0, e0, cutoff: int = 25, tol_scale: float = 1.0, zhat: bool = True):
    """(eigenvalues, records): records[i] = (level, offset, size, K, rho,
    D_active, z_active) for every merge, in (level, offset) order."""
    d0 = np.asarray(d0, dtype=np.float64)
    e0 = np.asarray(e0, dtype=np.float64)
    n = len(d0)
    sc = max(float(np.max(np.abs(d0))), float(np.max(np.abs(e0))) if n > 1 else 0.0, 1.0)
    d, e = d0 / sc, e0 / sc
    recs = []

    def rec(off, size, dmod, root):
        if size <= cutoff:
            lam, Q = leaf_full(dmod[off:off + size], e[off:off + size - 1] if size > 1 else np.zeros(1))
            return lam, Q, 0
        nl = size // 2
        m = off + nl - 1
        rho = abs(e[m])
        dm = dmod.copy()
        dm[m] -= rho
        dm[m + 1] -= rho
        lamL, QL, hL = rec(off, nl, dm, False)
        lamR, QR, hR = rec(off + nl, size - nl, dm, False)
        level = 1 + max(hL, hR)
        sign = -1.0 if e[m] < 0 else 1.0
        zL, zR = QL[-1, :], QR[0, :]
        tol = 8.0 * U_RND * max(np.max(np.abs(np.r_[lamL, lamR])), np.max(np.abs(np.r_[zL, zR]))) * tol_scale
        # stable merge of the sorted children, left first on ties (deflate.cpp:62-66)
        Dc = np.r_[lamL, lamR]
        order = np.argsort(Dc, kind="stable")
        D = Dc[order]
        Z = np.r_[sign * zL, zR][order]
        Qb = np.zeros((size, size))
        Qb[:nl, :nl] = QL
        Qb[nl:, nl:] = QR
        X = Qb[:, order]
        act, defl = _walk(D, Z, X, tol)
        K = len(act)
        dA, zA = D[act].copy(), Z[act].copy()
        recs.append((level, off, size, K, rho, dA, zA))
        org = np.zeros(K, dtype=np.int32)
        tau = np.zeros(K)
        for j in range(K):
            org[j], tau[j], _ = solve_root(dA, zA, rho, j)
        lam_roots = dA[org] + tau
        Dd = D[defl]
        par = np.argsort(np.r_[Dd, lam_roots], kind="stable")  # deflated first on ties
        lam = np.r_[Dd, lam_roots][par]
        if root:
            return lam, None, level
        zh = refreshed_weights(dA, zA, org, tau) if (zhat and K > 1) else zA
        U = np.empty((K, K))
        for j in range(K):
            y = zh / ((dA - dA[org[j]]) - tau[j])
            U[:, j] = y / np.sqrt(np.sum(y * y))
        Qp = np.concatenate([X[:, defl], X[:, act] @ U], axis=1)[:, par]
        return lam, Qp, level

    lam, _, _ = rec(0, n, d.copy(), True) if n > cutoff else (leaf_full(d, e)[0], None, 0)
    recs.sort(key=lambda r: (r[0], r[1]))
    return lam * sc, recs
