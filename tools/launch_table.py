"""Per-kernel table of an ncu launch list (last solve of the capture):
python tools/launch_table.py gpurun_out/ncu_X/launches_c5.csv"""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    out = OrderedDict()
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        key = int(d["ID"])
        out.setdefault(key, {"name": d["Kernel Name"].split("(")[0].replace("void ", ""),
                             "grid": d["Grid Size"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(out.values())


def main(path, solve=-1):
    ks = load(path)
    starts = [i for i, k in enumerate(ks) if k["name"].startswith("k_copy_input")] + [len(ks)]
    if len(starts) > 2:
        a, b = starts[solve - 1], starts[solve]
    else:
        a, b = 0, len(ks)
    tot = 0.0
    by = OrderedDict()
    for k in ks[a:b]:
        t = k.get("gpu__time_duration.sum", 0) / 1e3
        tot += t
        by[k["name"]] = by.get(k["name"], 0) + t
        extra = ""
        if "dram__bytes_read.sum" in k:
            extra = f"  dram r {k['dram__bytes_read.sum']/1e6:8.2f} MB w {k.get('dram__bytes_write.sum',0)/1e6:8.2f} MB"
        print(f"{k['name']:28s} {k['grid']:>16s} {t:9.2f} us{extra}")
    print(f"total {tot:.1f} us over {b - a} launches")
    for n, t in sorted(by.items(), key=lambda x: -x[1]):
        print(f"  {n:28s} {t:9.1f} us  {100*t/tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
