"""Benchmark / solve CLI of the SPEC's bench module, on the GPU solver.

    python -m paper_2605_26599_b200 --family uniform --n 16384 --repeat 5 --format json
    python -m paper_2605_26599_b200 --family file --input T.txt --out lam.txt

Families: the paper's uniform / normal / toeplitz (d=2, e=0.25) / clustered (SPEC.md:562,
PAPER.md:1916) plus BASELINE's sym-uniform / toeplitz121 / wilkinson, `reduced` (a dense
symmetric Gaussian matrix reduced on the GPU by cuSOLVER dsytrd, the paper's reduced-dense
family) and `file` (the reference's text format, src/tridiagonal.cpp:60-91).  The solver is this repository's
sm_100a BR solver (`--solver br`); the SPEC's `qrql` / `reference` CPU solvers are not part of
the product and are refused.  Accuracy: e_fwd = |lam - lam_ref|_inf /
max(1, |lam_ref|_inf), e_bwd = |lam - lam_ref|_inf / max(1, |T|_inf) against LAPACK
(scipy eigvalsh_tridiagonal) or the analytic spectrum of a Toeplitz family.  One record per
run with the SPEC's schema {family, n, solver, threads, time_ms, e_fwd, e_bwd,
ws_doubles_peak, ws_ints_peak, checksum_sum, checksum_l2, status}; exit code 0 iff every
record has status ok.
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import sys
import time

import numpy as np

COLUMNS = ["family", "n", "solver", "threads", "time_ms", "e_fwd", "e_bwd", "ws_doubles_peak",
           "ws_ints_peak", "checksum_sum", "checksum_l2", "status"]


def accuracy(lam: np.ndarray, ref: np.ndarray, tnorm: float) -> tuple[float, float]:
    """SPEC.md:571-578 (equal lengths, both ascending)."""
    if len(lam) != len(ref):
        raise ValueError("accuracy: length mismatch")
    diff = float(np.max(np.abs(lam - ref))) if len(lam) else 0.0
    return diff / max(1.0, float(np.max(np.abs(ref)))), diff / max(1.0, tnorm)


def toeplitz_exact(n: int, a: float, b: float) -> np.ndarray:
    k = np.arange(1, n + 1, dtype=np.float64)
    return np.sort(a + 2.0 * b * np.cos(k * np.pi / (n + 1)))


def reference_spectrum(kind: str, family: str, d: np.ndarray, e: np.ndarray):
    if kind == "none":
        return None, "none"
    if family in ("toeplitz", "toeplitz121") and kind in ("auto", "analytic"):
        b = 0.25 if family == "toeplitz" else 1.0
        return toeplitz_exact(len(d), 2.0, b), "analytic"
    if kind == "analytic":
        raise ValueError("analytic reference only for the Toeplitz families")
    if kind in ("auto", "lapack") and (kind == "lapack" or len(d) <= 65536):
        from scipy.linalg import eigvalsh_tridiagonal
        return np.sort(eigvalsh_tridiagonal(d, e)), "lapack"
    return None, "none"


def main(argv=None) -> int:
    import paper_2605_26599_b200 as br
    from paper_2605_26599_b200 import generators as G
    from paper_2605_26599_b200.tridiag_io import read_tridiagonal

    ap = argparse.ArgumentParser(prog="python -m paper_2605_26599_b200", description=__doc__.split("\n")[0])
    ap.add_argument("--family", default="uniform",
                    choices=["uniform", "normal", "toeplitz", "clustered", "sym-uniform", "toeplitz121",
                             "wilkinson", "reduced", "file"])
    ap.add_argument("--n", type=int, nargs="+", default=[4096])
    ap.add_argument("--solver", default="br", choices=["br", "qrql", "reference"])
    ap.add_argument("--threads", type=int, default=1, help="recorded only (one GPU)")
    ap.add_argument("--repeat", type=int, default=0, help="best-of-R; 0: 5 for n <= 8192, else 1")
    ap.add_argument("--warmup", type=int, default=1, help="untimed solves first (plan + CUDA graph capture)")
    ap.add_argument("--reference", default="auto", choices=["auto", "lapack", "analytic", "none"])
    ap.add_argument("--format", default="json", choices=["json", "csv"])
    ap.add_argument("--input", default=None)
    ap.add_argument("--out", default=None, help="write the eigenvalues (one per line, %%.17g)")
    ap.add_argument("--trace-merges", action="store_true", help="emit the per-merge trace (level, offset, size, NN, K)")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)

    if a.solver != "br":
        print(f"solver {a.solver!r}: CPU solvers are not part of this product (use --solver br)", file=sys.stderr)
        return 2
    if a.family == "file" and not a.input:
        print("--family file needs --input", file=sys.stderr)
        return 2

    records, ok_all = [], True
    sizes = [None] if a.family == "file" else a.n
    with br.Solver(a.device) as s:
        for n in sizes:
            rec = dict(family=a.family, n=n, solver="br", threads=a.threads)
            try:
                A = None
                if a.family == "file":
                    T = read_tridiagonal(a.input)
                    d, e = T.d, T.e
                elif a.family == "reduced":  # dense symmetric -> cuSOLVER dsytrd -> BR
                    import torch
                    M = np.random.default_rng(G.seed_for("normal", n)).standard_normal((n, n))
                    A = (M + M.T) / 2
                    d = np.zeros(n)
                    e = np.zeros(n - 1)
                else:
                    d, e = G.generate(a.family, n)
                rec["n"] = len(d)
                R = a.repeat or (5 if len(d) <= 8192 else 1)
                best, lam = math.inf, None
                def run_once():
                    if A is None:
                        return s.eigvals(d, e)
                    At = torch.tensor(A, device=f"cuda:{a.device}")  # overwritten by the reduction
                    torch.cuda.synchronize()
                    t = time.perf_counter()
                    out = s.eigvals_dense_device(At).cpu().numpy()
                    return out, time.perf_counter() - t

                for _ in range(a.warmup):
                    run_once()
                if a.trace_merges:
                    s.set_trace(True)
                for _ in range(R):
                    t0 = time.perf_counter()
                    lam = run_once()
                    dt = time.perf_counter() - t0
                    if A is not None:
                        lam, dt = lam  # reduction + solve, excluding the host-to-device copy of A
                    best = min(best, dt)
                led = s.ledger()
                if A is not None:
                    ref = np.linalg.eigvalsh(A) if (a.reference != "none" and n <= 8192) else None
                    tn = float(np.max(np.sum(np.abs(A), axis=1)))
                else:
                    ref, kind = reference_spectrum(a.reference, a.family, d, e)
                    tn = float(np.max(np.abs(d) + np.r_[np.abs(e), 0] + np.r_[0, np.abs(e)]))
                ef, eb = accuracy(lam, ref, tn) if ref is not None else (None, None)
                rec.update(time_ms=best * 1e3, e_fwd=ef, e_bwd=eb, ws_doubles_peak=led.peak_doubles,
                           ws_ints_peak=led.peak_ints, checksum_sum=float(np.sum(lam)),
                           checksum_l2=float(np.sqrt(np.sum(lam * lam))), status="ok")
                if a.trace_merges:
                    rec["trace"] = [list(map(int, t)) for t in s.trace()]
                    s.set_trace(False)
                if a.out:
                    with open(a.out, "w") as f:
                        f.writelines(f"{v:.17g}\n" for v in lam)
            except br.Error as ex:
                rec.update(time_ms=None, e_fwd=None, e_bwd=None, ws_doubles_peak=None, ws_ints_peak=None,
                           checksum_sum=None, checksum_l2=None, status=f"{type(ex).__name__}: {ex}")
                ok_all = False
            records.append(rec)
    if a.format == "json":
        for r in records:
            print(json.dumps(r))
    else:
        w = csv.writer(sys.stdout)
        w.writerow(COLUMNS)
        for r in records:
            w.writerow([r.get(c) for c in COLUMNS])
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
