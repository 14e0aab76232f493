"""The product library loads on a CPU-only box and exports every symbol that
include/brgpu.h declares (no compute calls without a GPU)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

from conftest import has_gpu
from paper_2605_26599_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> list[str]:
    txt = (ROOT / "include" / "brgpu.h").read_text()
    return sorted(set(re.findall(r"BRGPU_API\s+[\w\s\*]+?\b(brgpu_\w+)\s*\(", txt)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for s in ["brgpu_create", "brgpu_eigvals", "brgpu_eigvals_device", "brgpu_eigvals_batched",
              "brgpu_workspace_query", "brgpu_get_ledger", "brgpu_last_error_message"]:
        assert s in syms
    assert set(syms) == set(_native.EXPORTS)


def test_library_loads_and_exports_all_declared_symbols():
    lib = _native.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.brgpu_version()


def test_workspace_query_contract():
    # PAPER.md:1413 / SPEC.md:83: 16N doubles + 7N ints; 9.75 MiB at N = 65536
    lib = _native.lib()
    dd, ii = C.c_int64(), C.c_int64()
    assert lib.brgpu_workspace_query(65536, C.byref(dd), C.byref(ii)) == 0
    assert dd.value == 16 * 65536 and ii.value == 7 * 65536
    assert (dd.value * 8 + ii.value * 4) / 2**20 == 9.75
    assert lib.brgpu_workspace_query(0, C.byref(dd), C.byref(ii)) == 1


def test_status_strings_mirror_reference_errors():
    lib = _native.lib()
    names = [lib.brgpu_status_string(i).decode() for i in range(1, 9)]
    assert names == ["InvalidArgument", "NoConvergence", "BudgetExceeded", "PoleHit", "ZeroDenominator",
                     "MalformedCompactRoot", "DimensionMismatch", "DomainError"]


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_create_without_device_fails_loudly():
    import paper_2605_26599_b200 as br
    with pytest.raises(br.DeviceError):
        br.Solver(0)


def test_python_mirror_validation():
    import numpy as np
    import paper_2605_26599_b200 as br
    with pytest.raises(br.InvalidArgument):
        br.TridiagonalMatrix([], [])
    with pytest.raises(br.InvalidArgument):
        br.TridiagonalMatrix([1.0, np.nan], [0.5])
    with pytest.raises(br.InvalidArgument):
        br.TridiagonalMatrix([1.0, 2.0], [0.5, 0.1])
    T = br.TridiagonalMatrix([1.0, 2.0, 2.0], [0.0, 0.25])
    assert br.find_irreducible_blocks(T, 2.0**-52) == [br.Block(0, 1), br.Block(1, 2)]
    # SPEC.md:54-56
    assert br.find_irreducible_blocks(br.TridiagonalMatrix([1.0, 1.0], [1e-20]), 2.0**-52) == \
        [br.Block(0, 1), br.Block(1, 1)]
