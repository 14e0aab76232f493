"""profiles/<round>/traffic.json from ncu launch lists (tools/ncu_round.sh): per
kernel class of bench.py, DRAM bytes (read + write) per launch and the summed
ncu durations of the last solve in each capture.
python tools/traffic_json.py profiles/r01 c3=launches_c3.csv c4=launches_c4.csv c5=launches_c5.csv"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from launch_table import load  # noqa: E402

CLASSES = {
    "leaf": ["k_leaf"], "fused_level": ["k_levels_fused", "k_level_fused"],
    "merge_scatter": ["k_merge_prep", "k_merge_nn"], "segment_walk": ["k_segment_walk"],
    "surv_write": ["k_surv_scan"], "secular": ["k_secular", "k_secular_tiled", "k_secular_warp"],
    "zhat": ["k_zhat", "k_zhat_warp"], "rows": ["k_rows", "k_rows_warp"], "deflated_out": ["k_deflated_out"],
    "live_level": ["k_live_init", "k_live_level", "k_live_top", "k_live_cluster", "k_live_flow"],
    "live_sort": ["k_live_bounds", "k_live_hist", "k_live_scan", "k_live_scatter", "k_live_bucket"],
}


def base(name):
    n = name.replace("brgpu::", "").replace("(anonymous namespace)::", "").strip()
    return n.split("<")[0].strip()


def classes(path):
    ks = load(path)
    starts = [i for i, k in enumerate(ks) if k["name"].startswith("k_copy_input")] + [len(ks)]
    a, b = (starts[-2], starts[-1]) if len(starts) > 2 else (0, len(ks))
    out = {}
    for k in ks[a:b]:
        nm = base(k["name"])
        cls = next((c for c, names in CLASSES.items() if nm in names), None)
        if cls is None:
            continue
        e = out.setdefault(cls, {"launches": 0, "bytes": 0.0, "us": 0.0})
        e["launches"] += 1
        e["bytes"] += k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        e["us"] += k.get("gpu__time_duration.sum", 0.0) / 1e3
    return {c: {"launches": e["launches"], "dram_bytes_per_launch": e["bytes"] / e["launches"],
                "ncu_us_total": e["us"]} for c, e in out.items()}


def main(root, *specs):
    res = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     "(tools/ncu_round.sh), last solve of the capture, graph off, cold caches",
           "unit": "bytes per launch (dram read + write)", "configs": {}}
    for sp in specs:
        cfg, f = sp.split("=")
        res["configs"][cfg] = classes(str(Path(root) / f))
    (Path(root) / "traffic.json").write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res["configs"], indent=1)[:1500])


if __name__ == "__main__":
    main(*sys.argv[1:])
