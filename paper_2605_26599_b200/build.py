"""Build recipe for the product library (libbrgpu.so) and the test-only checkers.

    python -m paper_2605_26599_b200.build          # product + oracle
    python -m paper_2605_26599_b200.build --product

The product is compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``),
with ``--fmad=false`` so that every FP64 expression rounds exactly as written
(the arithmetic contract shared with oracle/br_oracle.c), ``-lineinfo`` for
ncu source correlation, and static cudart so the .so is self-contained.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libbrgpu.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
CXX = "g++"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}",
]
CXX_FLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", f"-I{CUDA_HOME / 'include'}",
             f"-I{ROOT / 'include'}"]

CU_SOURCES = ["kernels.cu", "fused.cu", "tiled.cu", "warp.cu", "sigma.cu", "sparse.cu", "live.cu"]
CPP_SOURCES = ["api.cpp"]


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build_product(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [ROOT / "include" / "brgpu.h"]
    objs: list[Path] = []
    for src in CU_SOURCES:
        s = CSRC / src
        if not s.exists():
            continue
        o = BUILD / (s.stem + ".o")
        if force or _stale(o, [s, *headers]):
            _run([NVCC, *NVCC_FLAGS, "-c", str(s), "-o", str(o)], BUILD / (s.stem + ".ptxas.log"))
        objs.append(o)
    for src in CPP_SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        if force or _stale(o, [s, *headers]):
            _run([CXX, *CXX_FLAGS, "-c", str(s), "-o", str(o)])
        objs.append(o)
    if force or _stale(LIB, objs):
        _run([CXX, "-shared", "-o", str(LIB), *map(str, objs),
              f"-L{CUDA_HOME / 'lib64'}", "-lcudart_static", "-ldl", "-lrt", "-lpthread",
              "-Wl,--exclude-libs,ALL"])
    return LIB


PROBE = PKG / "libbrprobe.so"


def build_probe(force: bool = False) -> Path:
    """FP64 peak microbenchmark (tooling for the roofline denominator)."""
    BUILD.mkdir(exist_ok=True)
    s = CSRC / "probe_fp64.cu"
    if force or _stale(PROBE, [s]):
        _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
              "-shared", str(s), "-o", str(PROBE), "-cudart", "static"])
    return PROBE


def build_oracle() -> None:
    """Test-only checkers: oracle/build/libbro.so and (where /root/reference
    exists) oracle/_ref/libbrref.so.  Never linked into the product."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--product", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build_product(force=a.force))
    build_probe(force=a.force)
    if not a.product:
        build_oracle()


if __name__ == "__main__":
    main()
