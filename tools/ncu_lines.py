"""Per CUDA source line of an ncu --set full report: warp instructions, average
active threads, shared wavefronts vs ideal, stall samples.
python tools/ncu_lines.py report.ncu-rep [file-substring] [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main(path, fsub="", top=40):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: defaultdict(float))
    fname, hdr, cur = None, None, None
    srcs = {}
    for row in csv.reader(txt.splitlines()):
        if not row:
            continue
        if row[0] == "File Name" or row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) != len(hdr):
            continue
        if row[0]:
            cur = (fname, int(row[0]))
            srcs[cur] = row[1][:70]
            continue
        d = dict(zip(hdr[2:], row[2:]))
        def num(k):
            try:
                return float(d.get(k, "0").replace(",", "") or 0)
            except ValueError:
                return 0.0
        a = agg[cur]
        a["inst"] += num("Instructions Executed")
        a["tinst"] += num("Thread Instructions Executed")
        a["samp"] += num("Warp Stall Sampling (All Samples)")
        a["wf"] += num("L1 Wavefronts Shared")
        a["wfi"] += num("L1 Wavefronts Shared Ideal")
    tot_s = sum(a["samp"] for a in agg.values()) or 1
    tot_i = sum(a["inst"] for a in agg.values()) or 1
    tot_t = sum(a["tinst"] for a in agg.values()) or 1
    print(f"overall avg threads/inst {tot_t / tot_i:.2f}")
    rows = [(k, a) for k, a in agg.items() if fsub in k[0]]
    rows.sort(key=lambda x: -x[1]["samp"])
    for (f, ln), a in rows[:top]:
        thr = a["tinst"] / a["inst"] if a["inst"] else 0
        wf = f"{a['wf']/a['wfi']:.2f}" if a["wfi"] else "-"
        print(f"{100*a['samp']/tot_s:5.1f}% {f}:{ln:<5d} inst {100*a['inst']/tot_i:5.1f}% thr {thr:5.1f} smem x{wf:5s} | {srcs.get((f, ln), '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 40)
