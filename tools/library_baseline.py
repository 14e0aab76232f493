"""Library baselines for the values-only tridiagonal eigenproblem (SURVEY.md §8(f)-4,
PAPER.md:2031-2055) next to this repo's BR solver, on the same inputs.

* cuSOLVER ``cusolverDnXstedc`` (compz=N) -- the paper's GPU baseline -- does not
  exist in this image's cuSOLVER 11.7 (CUDA 12.9; the paper used CUDA 13.2), so
  the GPU library baseline here is cuSOLVER's dense symmetric eigensolver
  (``syevd``, values only, via torch.linalg.eigvalsh on a float64 CUDA matrix)
  applied to the tridiagonal stored densely: O(n^2) memory and O(n^3) work.
* LAPACK ``dsterf`` (scipy, host): the paper's CPU values-only baseline.

Families: the paper's four (uniform, normal, Toeplitz (2, 0.25), clustered;
PAPER.md:1916) plus BASELINE's random sym-uniform, at N = 4096, 16384 and the
largest N whose syevd workspace fits the 32-bit cuSOLVER dense API (24576; the paper used 49,152); dsterf only to
16384).  Writes one JSON document (stdout and --out).

    python tools/library_baseline.py --out profiles/r02/library_baseline.json
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def gpu_dense_values(d, e, reps: int = 2) -> tuple[float, np.ndarray]:
    import torch
    n = len(d)
    A = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    idx = torch.arange(n, device="cuda")
    A[idx, idx] = torch.tensor(d, device="cuda")
    if n > 1:
        te = torch.tensor(e, device="cuda")
        A[idx[:-1], idx[1:]] = te
        A[idx[1:], idx[:-1]] = te
    w = torch.linalg.eigvalsh(A)  # warm-up (workspace, handles)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        w = torch.linalg.eigvalsh(A)
        t.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(t) * 1e-3)
    out = w.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    return best, out


def br_values(solver, d, e, reps: int = 5) -> tuple[float, np.ndarray]:
    import torch
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w = solver.eigvals_device(td, te)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        w = solver.eigvals_device(td, te)
        torch.cuda.synchronize()
        best = min(best, solver.timing()["device_ms"] * 1e-3)
    return best, w.cpu().numpy()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--sizes", default="4096,16384,24576")
    a = ap.parse_args()
    import scipy.linalg as sl
    import torch

    import paper_2605_26599_b200 as br
    from paper_2605_26599_b200 import generators as G

    props = torch.cuda.get_device_properties(0)
    res = {"device": props.name, "gpu_library": "cuSOLVER syevd (values only) via torch.linalg.eigvalsh, "
                                                 "dense storage of the tridiagonal",
           "cusolverDnXstedc": "absent from cuSOLVER 11.7 / CUDA 12.9 in this image",
           "cpu_library": "LAPACK dsterf (scipy.linalg.eigvalsh_tridiagonal, lapack_driver='sterf'), 1 call",
           "rows": []}
    with br.Solver(0) as s:
        for n in [int(x) for x in a.sizes.split(",")]:
            for fam in ["uniform", "normal", "toeplitz", "clustered", "sym-uniform"]:
                d, e = G.generate(fam, n)
                tol = G.tolerance(d, e)
                row = {"family": fam, "n": n}
                tb, wb = br_values(s, d, e)
                row["br_gpu_s"] = tb
                dense_bytes = 8 * n * n * 3
                if dense_bytes < 0.6 * props.total_memory:
                    tg, wg = gpu_dense_values(d, e)
                    row["cusolver_syevd_s"] = tg
                    row["syevd_over_br"] = tg / tb
                    row["max_abs_diff_vs_syevd"] = float(np.max(np.abs(wb - wg)))
                    row["within_tol"] = bool(row["max_abs_diff_vs_syevd"] <= tol)
                    row["syevd_workspace_bytes"] = 8 * n * n
                if n <= 16384:
                    t0 = time.perf_counter()
                    wl = sl.eigvalsh_tridiagonal(d, e, lapack_driver="sterf")
                    row["lapack_dsterf_s"] = time.perf_counter() - t0
                    row["max_abs_diff_vs_dsterf"] = float(np.max(np.abs(wb - wl)))
                led = s.ledger()
                row["br_workspace_bytes"] = 8 * led.peak_doubles + 4 * led.peak_ints
                res["rows"].append(row)
                print(json.dumps(row), flush=True)
    txt = json.dumps(res, indent=1)
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(txt)


if __name__ == "__main__":
    main()
