"""The C++ drop-in a reference maintainer adds (integration/br_gpu.cpp, INTEGRATION.md
§2), compiled with the reference's own src/tridiagonal.cpp + src/qrql.cpp and linked
against libbrgpu.so (oracle/Makefile -> oracle/_ref/cpp_dropin, built where
/root/reference exists and shipped prebuilt), run on the GPU: br::eigenvalues_br_gpu
must agree with the reference's br::eigenvalues_qrql within 8 n eps ||T|| and map
errors to the reference's br::Error classes."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "oracle" / "_ref" / "cpp_dropin"


def _run() -> str:
    if not EXE.exists():
        pytest.fail(f"{EXE} not built (oracle/Makefile builds it where /root/reference exists)")
    res = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    return res.stdout + f"\nrc {res.returncode}\n" + res.stderr


@pytest.mark.gpu
def test_cpp_dropin_matches_reference_qrql():
    out = _run()
    cases = [ln.split() for ln in out.splitlines() if ln.startswith("case ")]
    assert len(cases) == 9, out
    for c in cases:
        name, n, md, tol, srt = c[1], int(c[3]), float(c[5]), float(c[7]), int(c[9])
        assert md <= tol, f"{name}: {md} > {tol}"
        assert srt == 1, name
    assert "ctor-invalid-argument" in out
    assert "gpu-invalid-argument" in out
    assert "br_eigenvalues lambda 3 rows 6 ledger_ok 1" in out
    assert "done" in out and "rc 0" in out


def test_cpp_dropin_fails_loudly_without_gpu():
    """No CPU fallback: on a box without a device the drop-in raises DeviceError."""
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    if not EXE.exists():
        pytest.skip("cpp_dropin not built here")
    out = _run()
    assert "device-error" in out and "rc 3" in out
