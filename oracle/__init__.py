"""ctypes bindings of the TEST-ONLY checkers.

* ``oracle/build/libbro.so`` -- the C restatement (br_oracle.c), two arithmetic
  modes (see br_oracle.h).
* ``oracle/_ref/libbrref.so`` -- the unmodified reference sources from
  /root/reference/proj/src composed into the SPEC.md:312-380 driver
  (ref_compose.cpp).  Built in the container, travels to the GPU box prebuilt.

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline legs may use
this package; the product (paper_2605_26599_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIBBRO = HERE / "build" / "libbro.so"
LIBREF = HERE / "_ref" / "libbrref.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class BroOpts(C.Structure):
    _fields_ = [("leaf_cutoff", C.c_int), ("zhat", C.c_int), ("patched_stop", C.c_int),
                ("ref_arith", C.c_int), ("threads", C.c_int), ("tol_scale", C.c_double)]


class BroStats(C.Structure):
    _fields_ = [("merges", C.c_int64), ("sum_k", C.c_int64), ("sum_k2", C.c_double),
                ("sum_nn", C.c_int64), ("rotations", C.c_int64), ("evals", C.c_int64),
                ("pole_terms", C.c_double), ("zhat_terms", C.c_double), ("row_terms", C.c_double),
                ("max_k", C.c_int64), ("height", C.c_int32), ("blocks", C.c_int32)]


class BroTrace(C.Structure):
    _fields_ = [("level", C.c_int32), ("is_root", C.c_int32), ("offset", C.c_int64),
                ("size", C.c_int64), ("nn", C.c_int64), ("k", C.c_int64), ("tol", C.c_double),
                ("rho", C.c_double)]


_bro = None
_ref = None


def _ensure_built() -> None:
    if not LIBBRO.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def bro() -> C.CDLL:
    global _bro
    if _bro is None:
        _ensure_built()
        lib = C.CDLL(str(LIBBRO))
        lib.bro_eigvals.argtypes = [C.c_int64, _dp, _dp, _dp, C.POINTER(BroOpts), C.POINTER(BroStats),
                                    C.POINTER(BroTrace), C.c_int64, C.POINTER(C.c_int64)]
        lib.bro_eigvals_batched.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp, C.POINTER(BroOpts),
                                            C.POINTER(BroStats)]
        lib.bro_qrql_values.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int]
        lib.bro_leaf.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int]
        lib.bro_solve_root.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_int, C.c_int, C.c_int, _ip,
                                       _dp, _ip]
        lib.bro_deflate.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_int, _dp, _dp, _dp, _ip, _ip, _dp]
        lib.bro_refreshed_weights.argtypes = [C.c_int, _dp, _dp, _ip, _dp, C.c_int, _dp]
        lib.bro_eigvals_rows.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int64, C.POINTER(C.c_int64), _dp,
                                         C.POINTER(BroOpts)]
        lib.bro_sturm_count.argtypes = [C.c_int64, _dp, _dp, C.c_double]
        lib.bro_sturm_count.restype = C.c_int64
        lib.bro_set_merge_dump.argtypes = [_dp, C.c_int64]
        lib.bro_merge_dump_used.restype = C.c_int64
        _bro = lib
    return _bro


def ref_available() -> bool:
    return LIBREF.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not LIBREF.exists():
            raise FileNotFoundError(f"{LIBREF} not built (needs /root/reference at build time)")
        lib = C.CDLL(str(LIBREF))
        lib.brref_eigvals.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int]
        lib.brref_eigenvalues_qrql.argtypes = [C.c_int64, _dp, _dp, _dp]
        lib.brref_dense_eig.argtypes = [C.c_int64, _dp, _dp, _dp]
        lib.brref_leaf_eig.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp]
        lib.brref_solve_root.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_int, _ip, _dp]
        lib.brref_deflate.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp, _dp, _dp, _ip, _ip, _dp]
        lib.brref_refreshed_weights.argtypes = [C.c_int, _dp, _dp, C.c_double, _ip, _dp, _dp]
        _ref = lib
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


@dataclass
class Result:
    w: np.ndarray
    stats: dict
    trace: list


def eigvals(d, e, *, leaf_cutoff=25, zhat=True, patched=True, ref_arith=False, threads=0,
            tol_scale=1.0, trace=False) -> Result:
    """BR eigenvalues by the C restatement (ascending)."""
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    n = len(d)
    w = np.empty(n)
    o = BroOpts(leaf_cutoff, int(zhat), int(patched), int(ref_arith), int(threads), float(tol_scale))
    st = BroStats()
    cap = 0
    tr = None
    tl = C.c_int64(0)
    if trace:
        cap = max(16, 2 * n // 8 + 16)
        tr = (BroTrace * cap)()
    rc = bro().bro_eigvals(n, _p(d), _p(e), _p(w), C.byref(o), C.byref(st),
                           tr if trace else None, cap, C.byref(tl))
    if rc:
        raise OracleError(rc)
    stats = {f: getattr(st, f) for f, _ in BroStats._fields_}
    recs = []
    if trace:
        for i in range(min(tl.value, cap)):
            t = tr[i]
            recs.append((t.level, t.is_root, t.offset, t.size, t.nn, t.k))
    return Result(w, stats, recs)


def eigvals_rows(d, e, rows, *, leaf_cutoff=25, zhat=True, patched=True, ref_arith=False, threads=0):
    """Eigenvalues and the requested eigenvector rows (Algorithm 1's sigma,
    SPEC.md:317-337): returns (w, R) with R[r, j] = Q[rows[r], j], the columns in
    the order of w.  0-based row indices; duplicates and any order allowed."""
    d = _f64(d)
    n = len(d)
    e = _f64(e) if n > 1 else np.zeros(1)
    sel = np.ascontiguousarray(rows, dtype=np.int64).reshape(-1)
    w = np.empty(n)
    R = np.empty((len(sel), n))
    o = BroOpts(leaf_cutoff, int(zhat), int(patched), int(ref_arith), int(threads), 1.0)
    rc = bro().bro_eigvals_rows(n, _p(d), _p(e), _p(w), len(sel),
                                sel.ctypes.data_as(C.POINTER(C.c_int64)), _p(R), C.byref(o))
    if rc:
        raise OracleError(rc)
    return w, R


def eigvals_batched(d, e, batch: int, n: int, **kw) -> np.ndarray:
    d = _f64(d)
    e = _f64(e) if n > 1 else np.zeros(1)
    w = np.empty(batch * n)
    o = BroOpts(kw.get("leaf_cutoff", 25), int(kw.get("zhat", True)), int(kw.get("patched", True)),
                int(kw.get("ref_arith", False)), int(kw.get("threads", 0)), 1.0)
    st = BroStats()
    rc = bro().bro_eigvals_batched(batch, n, _p(d), _p(e), _p(w), C.byref(o), C.byref(st))
    if rc:
        raise OracleError(rc)
    return w


def qrql(d, e, ref_arith=False) -> np.ndarray:
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    w = np.empty(len(d))
    rc = bro().bro_qrql_values(len(d), _p(d), _p(e), _p(w), int(ref_arith))
    if rc:
        raise OracleError(rc)
    return w


def leaf(d, e, ref_arith=False):
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    m = len(d)
    lam, blo, bhi = np.empty(m), np.empty(m), np.empty(m)
    rc = bro().bro_leaf(m, _p(d), _p(e), _p(lam), _p(blo), _p(bhi), int(ref_arith))
    if rc:
        raise OracleError(rc)
    return lam, blo, bhi


def leaf_full(d, e, ref_arith=False):
    """(lam, Q) of a leaf by the leaf QL/QR sweeps, every row tracked (Q[i, k] =
    row i of eigenvector k) -- test infrastructure for the Theorem 1 check."""
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    m = len(d)
    lam, Q = np.empty(m), np.empty((m, m))
    rc = bro().bro_leaf_full(m, _p(d), _p(e), _p(lam), _p(Q), int(ref_arith))
    if rc:
        raise OracleError(rc)
    return lam, Q


def solve_root(d, z, rho, j, patched=True, ref_arith=False):
    d, z = _f64(d), _f64(z)
    org, tau, ne = C.c_int(0), C.c_double(0.0), C.c_int(0)
    rc = bro().bro_solve_root(len(d), _p(d), _p(z), float(rho), int(j), int(patched), int(ref_arith),
                              C.byref(org), C.byref(tau), C.byref(ne))
    if rc:
        raise OracleError(rc)
    return org.value, tau.value, ne.value


def deflate(d, z, tol_scale=1.0, ref_arith=False):
    d, z = _f64(d), _f64(z)
    n = len(d)
    da, za, df = np.empty(n), np.empty(n), np.empty(n)
    k, nrot, tol = C.c_int(0), C.c_int(0), C.c_double(0)
    rc = bro().bro_deflate(n, _p(d), _p(z), float(tol_scale), int(ref_arith), _p(da), _p(za), _p(df),
                           C.byref(k), C.byref(nrot), C.byref(tol))
    if rc:
        raise OracleError(rc)
    K = k.value
    return da[:K].copy(), za[:K].copy(), df[: n - K].copy(), nrot.value, tol.value


def refreshed_weights(d, z, origin, tau, ref_arith=False):
    d, z, tau = _f64(d), _f64(z), _f64(tau)
    org = np.ascontiguousarray(origin, dtype=np.int32)
    out = np.empty(len(d))
    bro().bro_refreshed_weights(len(d), _p(d), _p(z), org.ctypes.data_as(_ip), _p(tau),
                                int(ref_arith), _p(out))
    return out


def sturm_count(d, e, x: float) -> int:
    d, e = _f64(d), _f64(e)
    return int(bro().bro_sturm_count(len(d), _p(d), _p(e), float(x)))


# ---------------------------------------------------------------- reference
def ref_eigvals(d, e, *, threads=0, zhat=True, leaf_cutoff=25) -> np.ndarray:
    """SPEC driver composed from the UNMODIFIED reference blocks (oracle/_ref)."""
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    w = np.empty(len(d))
    rc = ref().brref_eigvals(len(d), _p(d), _p(e), _p(w), int(threads), int(zhat), int(leaf_cutoff))
    if rc:
        raise OracleError(rc, "reference")
    return w


def ref_qrql(d, e) -> np.ndarray:
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    w = np.empty(len(d))
    rc = ref().brref_eigenvalues_qrql(len(d), _p(d), _p(e), _p(w))
    if rc:
        raise OracleError(rc, "reference qrql")
    return w


def ref_dense(d, e) -> np.ndarray:
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    w = np.empty(len(d))
    rc = ref().brref_dense_eig(len(d), _p(d), _p(e), _p(w))
    if rc:
        raise OracleError(rc, "reference dense")
    return w


def ref_leaf(d, e):
    d = _f64(d)
    e = _f64(e) if len(d) > 1 else np.zeros(1)
    m = len(d)
    lam, blo, bhi = np.empty(m), np.empty(m), np.empty(m)
    rc = ref().brref_leaf_eig(m, _p(d), _p(e), _p(lam), _p(blo), _p(bhi))
    if rc:
        raise OracleError(rc, "reference leaf")
    return lam, blo, bhi


def ref_solve_root(d, z, rho, j):
    d, z = _f64(d), _f64(z)
    org, tau = C.c_int(0), C.c_double(0.0)
    rc = ref().brref_solve_root(len(d), _p(d), _p(z), float(rho), int(j), C.byref(org), C.byref(tau))
    if rc:
        raise OracleError(rc, "reference solve_root")
    return org.value, tau.value


def ref_deflate(d, z, rho=1.0):
    d, z = _f64(d), _f64(z)
    n = len(d)
    da, za, df = np.empty(n), np.empty(n), np.empty(n)
    k, nrot, tol = C.c_int(0), C.c_int(0), C.c_double(0)
    rc = ref().brref_deflate(n, _p(d), _p(z), float(rho), _p(da), _p(za), _p(df), C.byref(k),
                             C.byref(nrot), C.byref(tol))
    if rc:
        raise OracleError(rc, "reference deflate")
    K = k.value
    return da[:K].copy(), za[:K].copy(), df[: n - K].copy(), nrot.value, tol.value


def ref_refreshed_weights(d, z, rho, origin, tau):
    d, z, tau = _f64(d), _f64(z), _f64(tau)
    org = np.ascontiguousarray(origin, dtype=np.int32)
    out = np.empty(len(d))
    rc = ref().brref_refreshed_weights(len(d), _p(d), _p(z), float(rho), org.ctypes.data_as(_ip),
                                       _p(tau), _p(out))
    if rc:
        raise OracleError(rc, "reference refreshed_weights")
    return out


def tolerance(d, e) -> float:
    """BASELINE tolerance 8 n eps ||T||_inf with eps = 2^-52."""
    d = np.abs(_f64(d))
    e = np.abs(_f64(e)) if len(d) > 1 else np.zeros(0)
    row = d.copy()
    if len(d) > 1:
        row[:-1] += e
        row[1:] += e
    return 8.0 * len(d) * 2.0 ** -52 * float(row.max())


def merge_inputs(d, e, **kw) -> list[tuple[int, int, int, np.ndarray, np.ndarray]]:
    """Per merge (offset, size, n_left, D, z): the merged child eigenvalues and
    z = (sign*bhi_L, blo_R) that each BR merge hands to deflation (Theorem 1
    check; single-threaded so the records come in tree order per level)."""
    d = _f64(d)
    n = len(d)
    cap = 64 * n + 1024
    for _ in range(2):
        buf = np.zeros(cap)
        bro().bro_set_merge_dump(_p(buf), cap)
        try:
            eigvals(d, e, threads=1, **kw)
        finally:
            used = bro().bro_merge_dump_used()
            bro().bro_set_merge_dump(None, 0)
        if used <= cap:
            break
        cap = used
    out, at = [], 0
    while at < used:
        off, size, nl = int(buf[at]), int(buf[at + 1]), int(buf[at + 2])
        out.append((off, size, nl, buf[at + 3:at + 3 + size].copy(), buf[at + 3 + size:at + 3 + 2 * size].copy()))
        at += 3 + 2 * size
    return out


# ---------------------------------------------------------------- GPU certificate
LIBSTURM = HERE / "build" / "libbrsturm.so"
_sturm = None


def sturm_counts_gpu(d, e, x) -> np.ndarray:
    """Sturm counts #{eigenvalues < x_j} for many shifts at once on the GPU
    (oracle/sturm_gpu.cu, test-only; arithmetic identical to sturm_count)."""
    global _sturm
    if _sturm is None:
        _ensure_built()
        lib = C.CDLL(str(LIBSTURM))
        lib.brsturm_counts.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int64, C.POINTER(C.c_int64)]
        _sturm = lib
    d, e, x = _f64(d), _f64(e), _f64(x)
    out = np.empty(len(x), dtype=np.int64)
    rc = _sturm.brsturm_counts(len(d), _p(d), _p(e) if len(d) > 1 else None, _p(x), len(x),
                               out.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc:
        raise OracleError(rc, "GPU Sturm counts")
    return out


def sturm_certificate(d, e, w, tol) -> tuple[int, int]:
    """Certify EVERY index: count(w_i - tol) <= i < count(w_i + tol), so the exact
    i-th eigenvalue lies within tol of w_i.  Returns (#violations, first bad i or -1)."""
    w = _f64(w)
    n = len(w)
    lo = sturm_counts_gpu(d, e, w - tol)
    hi = sturm_counts_gpu(d, e, w + tol)
    idx = np.arange(n)
    bad = np.nonzero((lo > idx) | (hi < idx + 1))[0]
    return len(bad), int(bad[0]) if len(bad) else -1
