"""Build libbrgpu.so from a git revision into tools/lib<name>.so (A/B timing):
    python tools/build_head.py [REV] [NAME]"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_26599_b200 import build as B  # noqa: E402

rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
name = sys.argv[2] if len(sys.argv) > 2 else "head"
src = Path(f"/tmp/src_{name}")
subprocess.run(f"rm -rf {src} && mkdir -p {src} && git -C {B.ROOT} archive {rev} paper_2605_26599_b200/csrc include "
               f"| tar -x -C {src}", shell=True, check=True)
csrc = src / "paper_2605_26599_b200" / "csrc"
bd = Path(f"/tmp/build_{name}")
bd.mkdir(exist_ok=True)
inc = str(B.ROOT / "include")
nv = [f.replace(inc, str(src / "include")) for f in B.NVCC_FLAGS]
cx = [f.replace(inc, str(src / "include")) for f in B.CXX_FLAGS]


def cu(s):
    o = bd / (Path(s).stem + ".o")
    B._run([B.NVCC, *nv, "-c", str(csrc / s), "-o", str(o)])
    return o


with ThreadPoolExecutor(4) as ex:
    objs = list(ex.map(cu, B.CU_SOURCES))
o = bd / "api.o"
B._run([B.CXX, *cx, "-c", str(csrc / "api.cpp"), "-o", str(o)])
out = B.ROOT / "tools" / f"lib{name}.so"
B._run([B.CXX, "-shared", "-o", str(out), *map(str, objs), str(o), f"-L{B.CUDA_HOME / 'lib64'}",
        "-lcudart_static", "-ldl", "-lrt", "-lpthread", "-Wl,--exclude-libs,ALL"])
print(out)
