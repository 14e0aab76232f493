"""Tridiagonal text format of the reference (src/tridiagonal.cpp:60-91):

    n
    d_0 ... d_{n-1}      (one value per line, %.17g)
    e_0 ... e_{n-2}

`read_tridiagonal` raises InvalidArgument with the reference's messages for an
unreadable file, a bad order line, or a missing diagonal / off-diagonal entry;
values are validated by TridiagonalMatrix (src/tridiagonal.cpp:17-30).
"""
from __future__ import annotations

import numpy as np

from . import InvalidArgument, TridiagonalMatrix


def read_tridiagonal(path: str) -> TridiagonalMatrix:
    try:
        with open(path, "r") as f:
            toks = f.read().split()
    except OSError:
        raise InvalidArgument(f"cannot open tridiagonal file: {path}") from None
    try:
        n = int(toks[0])
    except (IndexError, ValueError):
        n = 0
    if n <= 0:
        raise InvalidArgument(f"tridiagonal file: bad order line in {path}")
    vals = []
    for t in toks[1:2 * n]:
        try:
            vals.append(float(t))
        except ValueError:
            break
    if len(vals) < n:
        raise InvalidArgument(f"tridiagonal file: missing diagonal entry in {path}")
    if len(vals) < 2 * n - 1:
        raise InvalidArgument(f"tridiagonal file: missing off-diagonal entry in {path}")
    return TridiagonalMatrix(np.array(vals[:n]), np.array(vals[n:2 * n - 1]))


def write_tridiagonal(T: TridiagonalMatrix, path: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(f"{T.n}\n")
            f.writelines(f"{v:.17g}\n" for v in T.d)
            f.writelines(f"{v:.17g}\n" for v in T.e)
    except OSError:
        raise InvalidArgument(f"cannot write tridiagonal file: {path}") from None
