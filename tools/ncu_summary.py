"""Summarise an ncu report: key throughput / occupancy / divergence metrics per kernel."""
import csv
import subprocess
import sys

WANT = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Branch Efficiency", "L1/TEX Hit Rate", "Grid Size", "Block Size"]
RAW = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(det.splitlines()))
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ["Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"])
    out = {}
    for x in r[1:]:
        if x[mi] in WANT:
            out.setdefault((x[ii], x[ki].split("(")[0]), {})[x[mi]] = f"{x[vi]} {x[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    for row in rr[2:]:
        key = (row[hh.index("ID")], row[hh.index("Kernel Name")].split("(")[0])
        for m in RAW:
            if m in hh:
                out.setdefault(key, {})[m] = f"{row[hh.index(m)]} {rr[1][hh.index(m)]}".strip()
    for (i, k), v in out.items():
        print(f"== [{i}] {k}")
        for a, b in v.items():
            print(f"   {a:70s} {b}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
