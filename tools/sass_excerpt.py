"""SASS evidence of the hot kernels (cuobjdump of the in-tree build objects):
opcode mix per kernel and the unrolled pole loop of the lane-tier evaluation.
python tools/sass_excerpt.py > profiles/r02/sass_hot_kernels.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
BUILD = ROOT / "paper_2605_26599_b200" / "_build"
KERNELS = [("fused.o", "k_levels_fused"), ("live.o", "k_live_level"), ("kernels.o", "k_secular"),
           ("warp.o", "k_secular_warp"), ("kernels.o", "k_leaf")]
KEY = ["DFMA", "DADD", "DMUL", "MUFU.RCP64H", "MUFU.RSQ64H", "LDS", "STS", "LDG", "STG", "SHFL", "BAR",
       "ATOMS", "ATOMG", "RED", "LDGSTS", "UBLKCP", "UTMALDG", "BRA"]


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", str(BUILD / obj)], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
        elif name:
            cur.append(line)
    if name:
        funcs[name] = cur
    return funcs


for obj, kname in KERNELS:
    fs = functions(obj)
    for name, lines in fs.items():
        if kname not in name or (kname == "k_secular" and "warp" in name) or "tiled" in name:
            continue
        ops = collections.Counter()
        for l in lines:
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
            if m:
                op = m.group(1)
                for k in KEY:
                    if op == k or op.startswith(k + "."):
                        ops[k] += 1
        print(f"== {name}  ({obj})")
        print("   " + "  ".join(f"{k}:{ops[k]}" for k in KEY if ops[k]))
        if kname in ("k_live_level", "k_secular"):
            idx = [i for i, l in enumerate(lines) if "MUFU.RCP64H" in l]
            # the 4-term unrolled pole loop: the first run of 4 reciprocal seeds within 120 lines
            for a in range(len(idx) - 3):
                if idx[a + 3] - idx[a] < 120:
                    lo, hi = max(0, idx[a] - 20), min(len(lines), idx[a + 3] + 60)
                    print("   -- unrolled pole loop (4 terms per iteration) --")
                    for l in lines[lo:hi]:
                        s = re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).rstrip()
                        if s.strip():
                            print("   " + s.strip())
                    break
        print()
