"""The C++ wrapper (include/brgpu.hpp) compiles, links against libbrgpu.so and maps
status codes to the reference's exception names; with BRGPU_USE_BR_ERRORS it compiles
against the reference's own br/errors.hpp (the INTEGRATION.md binding)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2605_26599_b200" / "libbrgpu.so"
REF_INC = Path("/root/reference/proj/include")

PROG = r'''
#include <cstdio>
#include "brgpu.hpp"
int main() {
    try {
        brgpu::Solver s(0);
        std::vector<double> d{2.0, 2.0}, e{0.25};
        auto w = s.eigenvalues(d, e);
        std::printf("ok %.17g %.17g\n", w[0], w[1]);
        try { s.eigenvalues(std::vector<double>{1.0, 0.0 / 0.0}, std::vector<double>{1.0}); }
        catch (const brgpu::InvalidArgument&) { std::printf("invalid-argument\n"); }
    } catch (const brgpu::DeviceError& ex) {
        std::printf("device-error %s\n", ex.what());
    }
    return 0;
}
'''


def _build(tmp_path, src, extra=()):
    c = tmp_path / "t.cpp"
    c.write_text(src)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", *extra, str(c), str(LIB),
                    f"-Wl,-rpath,{LIB.parent}", "-o", str(exe)], check=True)
    return exe


@pytest.mark.gpu
def test_cpp_wrapper_builds_and_runs_on_gpu(tmp_path):
    exe = _build(tmp_path, PROG)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout
    assert out.startswith("ok 1.75 2.25") and "invalid-argument" in out


def test_cpp_wrapper_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = _build(tmp_path, PROG)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout
    if has_gpu():
        pytest.skip("GPU present: covered by the gpu-marked test")
    assert out.startswith("device-error")


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present")
def test_reference_side_binding_compiles(tmp_path):
    src = r'''
#include "br/errors.hpp"
#include "br/tridiagonal.hpp"
#define BRGPU_USE_BR_ERRORS
#include "brgpu.hpp"
namespace br {
std::vector<double> eigenvalues_br_gpu(const TridiagonalMatrix& t) {
    static thread_local brgpu::Solver solver(0);
    return solver.eigenvalues(t);
}
}
int main() { return 0; }
'''
    (tmp_path / "t.cpp").write_text(src)
    subprocess.run(["g++", "-std=c++20", "-c", f"-I{REF_INC}", f"-I{ROOT / 'include'}",
                    str(tmp_path / "t.cpp"), "-o", str(tmp_path / "t.o")], check=True)
