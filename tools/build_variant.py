"""Build an A/B variant of libbrgpu.so with extra nvcc defines:
    python tools/build_variant.py NAME -DBRGPU_LEAF_SM=0 ...   -> tools/libNAME.so
Run a variant with BRGPU_LIB=tools/libNAME.so (tools/ab_bench.py)."""
import sys
from pathlib import Path
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_26599_b200 import build as B

name, defs = sys.argv[1], sys.argv[2:]
out = B.ROOT / "tools" / f"lib{name}.so"
bdir = Path("/tmp/brgpu_variant_" + name)
bdir.mkdir(exist_ok=True)

def cu(src):
    o = bdir / (Path(src).stem + ".o")
    B._run([B.NVCC, *B.NVCC_FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(o)])
    return o

with ThreadPoolExecutor(4) as ex:
    objs = list(ex.map(cu, B.CU_SOURCES))
o = bdir / "api.o"
B._run([B.CXX, *B.CXX_FLAGS, *[d for d in defs if d.startswith("-D")], "-c", str(B.CSRC / "api.cpp"), "-o", str(o)])
B._run([B.CXX, "-shared", "-o", str(out), *map(str, objs), str(o), f"-L{B.CUDA_HOME / 'lib64'}",
        "-lcudart_static", "-ldl", "-lrt", "-lpthread", "-Wl,--exclude-libs,ALL"])
print(out)
