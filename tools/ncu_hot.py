"""Hot source lines of an ncu --set full report (mixed cuda,sass source page):
per CUDA source line: stall samples, executed warp instructions, top stall reasons.
python tools/ncu_hot.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main(path, top=40):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = txt.splitlines()
    agg = defaultdict(lambda: defaultdict(float))
    src = {}
    fname = None
    hdr = None
    cur = None
    for row in csv.reader(lines):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) != len(hdr):
            continue
        if row[0]:
            cur = (fname, int(row[0]))
            src[cur] = row[1].strip()
            continue
        d = dict(zip(hdr[2:], row[2:]))
        a = agg[cur]
        for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                a[k] += float(d.get(k, 0) or 0)
            except ValueError:
                pass
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    a[k] += float(v or 0)
                except ValueError:
                    pass
    tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
    print(f"total samples {tot:.0f}")
    for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
        s = a["Warp Stall Sampling (All Samples)"]
        st = sorted(((k[6:], v) for k, v in a.items() if k.startswith("stall_")), key=lambda x: -x[1])[:3]
        sts = " ".join(f"{k}:{100*v/max(s,1):.0f}%" for k, v in st if v)
        print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]:<5d} inst {a['Instructions Executed']:10.0f}  {sts:40s} | {src.get(key,'')[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
