#!/usr/bin/env python
"""Benchmark: seconds for all FP64 eigenvalues of a random n = 2^20 symmetric
tridiagonal (BASELINE.json config 5), plus FP64-pipe fraction of the dominant
kernel.  One JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

ours       : the sm_100a BR solver through the C ABI.  ``value`` = mean device
             seconds per solve (CUDA events on the solver's stream, inputs resident
             in HBM, L2 flushed with a 256 MiB write before every timed step);
             ``e2e`` = the same solve through the host-buffer C-ABI call
             (pinned H2D of d, e + solve + D2H of the eigenvalues, wall clock).
reference  : the reference's own CPU implementation of the path -- the unmodified
             reference building blocks (/root/reference/proj/src, built into
             oracle/_ref) composed into the SPEC.md:312-380 driver with OpenMP over
             merges and roots -- on all host cores, same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "seconds for all fp64 eigenvalues, n=2^20 tridiagonal; FP64-pipe % of peak"

CONFIGS = {
    "c1": dict(family="sym-uniform", n=4096, batch=0,
               workload="random symmetric tridiagonal n=4096, d,e~U(-1,1) (config 1)"),
    "c2": dict(family="sym-uniform", n=1024, batch=4096,
               workload="batch of 4096 random tridiagonals n=1024, d,e~U(-1,1) (config 2)"),
    "c3": dict(family="toeplitz121", n=1 << 16, batch=0,
               workload="(1,2,1) Toeplitz n=2^16 (config 3)"),
    "c4": dict(family="wilkinson", n=1 << 18, batch=0,
               workload="glued Wilkinson W21+ n=2^18, glue 1e-10 (config 4)"),
    "c5": dict(family="sym-uniform", n=1 << 20, batch=0,
               workload="random symmetric tridiagonal n=2^20, d,e~U(-1,1) (config 5)"),
}

# FP64 pipe operations per algorithmic unit (verified in SASS of this
# build): secular pole term 2 DADD (delta) + 5 DFMA (reciprocal) + 2 DMUL + 2 DADD
# (sum, derivative; psi' and sum_{i<=j} t are prefix snapshots, sum|t| follows from the
# bracket's sign split) = 11; refreshed-weight term 3 DADD + 5 DFMA + 2 DMUL = 10;
# boundary-row term 2 DADD + 5 DFMA + 1 DMUL + 3 DFMA = 11.
OPS_PER_TERM = {"secular": 11, "zhat": 10, "rows": 11}
# algorithmic bytes per element per grid-tier level of the memory-bound classes
# (kernel class names of brgpu_kernel_class_name):
#   merge_scatter = k_merge_prep: read lam + the z source            16 B
#   nn_flag       = k_merge_nn: read lam, blo, bhi (24), write D, Z,
#                   R0, R1 (32), flag (1), prefix (4)                  61 B
#   deflated_out  : read D, R0, R1 (24), flag + prefix (5), survivor
#                   flag + prefix (5), write lam, blo, bhi (24)        58 B
#   surv_write    = k_surv_scan over the NN list (counted per element: 1 B)
BYTES_PER_ELEM = {"merge_scatter": 16, "nn_flag": 61, "deflated_out": 58, "surv_write": 1,
                  "segment_walk": 0}


def traffic_bytes(config: str, kernel: str):
    """DRAM bytes per launch (read + write) of a kernel class, from the committed
    ncu launch list of this config (profiles/r01/traffic.json), else None."""
    try:
        t = json.loads((ROOT / "profiles" / "r01" / "traffic.json").read_text())
        return t["configs"][config][kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows: list[list[str]] = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        def rd():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        self.t = threading.Thread(target=rd, daemon=True)
        self.t.start()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak(device: int) -> dict:
    import ctypes as C
    lib = C.CDLL(str(ROOT / "paper_2605_26599_b200" / "libbrprobe.so"))
    lib.brprobe_fp64_peak.restype = C.c_double
    lib.brprobe_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    ms = C.c_double()
    ops = lib.brprobe_fp64_peak(device, C.byref(ms))
    return {"lane_ops_per_s": ops, "probe_ms": ms.value}


def cpu_reference(d, e, threads: int, batch: int, n: int) -> float:
    """One solve by the reference composition (oracle/_ref), seconds.  A batch runs
    its matrices concurrently, one single-threaded solve per host core (ctypes
    releases the GIL), which is the fastest way to use the cores for many small
    problems."""
    import oracle as O
    t0 = time.perf_counter()
    if batch:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda b: O.ref_eigvals(d[b], e[b], threads=1), range(batch)))
    else:
        O.ref_eigvals(d, e, threads=threads)
    return time.perf_counter() - t0


def make_input(cfg):
    from paper_2605_26599_b200 import generators as G
    if cfg["batch"]:
        return G.generate_batch(cfg["family"], cfg["batch"], cfg["n"])
    return G.generate(cfg["family"], cfg["n"])


def run_reference(args, cfg, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle as O
    cores = os.cpu_count() or 1
    d, e = make_input(cfg)
    batch, n = cfg["batch"], cfg["n"]
    if batch:  # bounded sample: 256 of the 4096 matrices, scaled to the whole batch
        sample = 256
        d, e = d[:sample], e[:sample]
    else:
        sample = 0
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbrref.so not built"}))
        return
    for _ in range(args.warmup):
        cpu_reference(d, e, cores, sample, n)
    ts = [cpu_reference(d, e, cores, sample, n) for _ in range(args.steps)]
    v = statistics.mean(ts)
    if batch:
        v *= batch / sample
    samp = (f"{sample} of {batch} matrices per step, scaled x{batch // sample}" if batch
            else f"1 full solve per step ({cfg['workload']})")
    line = {
        "metric": METRIC, "value": v, "unit": "s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (xorshift64*, SPEC.md:595)",
        "config": {"workload": cfg["workload"], "n": n, "batch": batch or 1,
                   "solver": "reference blocks composed per SPEC.md:312-380, OpenMP"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "reference", "sample": samp},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_2605_26599_b200 as br

    dev = local_rank
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    d, e = make_input(cfg)
    batch, n = cfg["batch"], cfg["n"]
    N = (batch or 1) * n
    td = torch.tensor(d, device="cuda")
    te = torch.tensor(e, device="cuda")
    tw = torch.empty_like(td)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # one process per GPU: rank r solves its subtree(s), one NCCL exchange, shared top merges
    parallelism = "single-gpu"
    if world > 1:
        try:
            s = br.distributed_solver(dev)
            parallelism = (f"subtree-split over {world} GPUs (NCCL broadcast exchange, "
                           "shared top merges)")
        except Exception as ex:  # stated in the JSON line, never silent
            print(f"[bench] distributed init failed on rank {rank}: {ex!r}", file=sys.stderr)
            s = br.Solver(dev)
            parallelism = f"replica{world} (distributed init failed: {type(ex).__name__})"
    else:
        s = br.Solver(dev)
    s.reserve(N)

    def solve():
        if batch:
            s.eigvals_batched_device(td, te, tw)
        else:
            s.eigvals_device(td, te, tw)

    for _ in range(max(args.warmup, 0)):
        solve()
    torch.cuda.synchronize()

    # --- untimed: work counts (trace) and per-kernel profile (events between launches)
    s.set_trace(True)
    solve()
    stats = s.stats()
    s.set_trace(False)
    solve()
    launches = s.stats()["kernel_launches"]
    prof = s.profile_kernels(td, te, batch) if world == 1 else {}

    # --- timed region: K steps, L2 flushed before each, device time per step
    sampler = ClockSampler(dev)
    sampler.start()
    step_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        solve()
        step_ms.append(s.timing()["device_ms"])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    mean_ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([mean_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms = float(t.item())
    out = s.eigvals_batched_device(td, te) if batch else s.eigvals_device(td, te)
    torch.cuda.synchronize()

    # --- end to end through the host-buffer C-ABI call (pinned buffers)
    hd = torch.from_numpy(np.ascontiguousarray(d).reshape(-1)).pin_memory()
    he = torch.from_numpy(np.ascontiguousarray(e).reshape(-1)).pin_memory()
    hw = torch.empty(N, dtype=torch.float64).pin_memory()
    def e2e_call():
        if batch:
            s._lib.brgpu_eigvals_batched(s._h, batch, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr())
        else:
            s._lib.brgpu_eigvals(s._h, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr())

    for _ in range(max(args.warmup, 1)):  # the host-buffer path's staging buffers and graph
        e2e_call()
    e2e = []
    for _ in range(max(1, min(args.steps, 10))):
        t0 = time.perf_counter()
        e2e_call()
        e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e)
    if os.environ.get("BENCH_DEBUG"):
        print("e2e samples ms:", " ".join(f"{x * 1e3:.3f}" for x in e2e), file=sys.stderr)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    if rank == 0:
        # --- roofline of the dominant kernel class (live profile)
        peak = fp64_peak(dev)
        roof = None
        if prof:
            # FP64 work per kernel class (algorithmic lane-ops, see OPS_PER_TERM)
            grid_terms = stats["pole_terms"] - stats["pole_terms_fused"]
            work = {
                "secular": OPS_PER_TERM["secular"] * grid_terms,
                "zhat": OPS_PER_TERM["zhat"] * stats["k2_nonroot_grid"],
                "rows": OPS_PER_TERM["rows"] * stats["k2_nonroot_grid"],
                "fused_level": (OPS_PER_TERM["secular"] * stats["pole_terms_fused"]
                                + (OPS_PER_TERM["zhat"] + OPS_PER_TERM["rows"]) * stats["k2_nonroot_fused"]),
            }
            pk = peak["lane_ops_per_s"] / 1e12
            fp64 = {}
            for k, ops in work.items():
                if k in prof and ops > 0:
                    t = prof[k][0] * 1e-3
                    fp64[k] = {"ms": prof[k][0], "tops": ops / t / 1e12, "frac_of_peak": ops / t / 1e12 / pk}
            dom = max(prof, key=lambda k: prof[k][0])
            dom_ms, dom_launch = prof[dom]
            if dom in work:
                ach = work[dom] / (dom_ms * 1e-3) / 1e12
                roof = {"bound": "fp64", "kernel": dom, "achieved": ach, "peak": pk,
                        "unit": "TFLOP/s (FP64 pipe lane-ops: DADD/DMUL/DFMA = 1)", "frac": ach / pk,
                        "traffic": traffic_bytes(args.config, dom), "launches": dom_launch,
                        "avg_launch_ms": dom_ms / dom_launch,
                        "traffic_note": "DRAM bytes per launch from the committed ncu launch list "
                                        "(profiles/r01/traffic.json); a bound=fp64 kernel, reported as context",
                        "peak_source": "measured DFMA probe (libbrprobe.so), burst",
                        "work_note": "fused_level = secular + zhat + rows FP64 work of the SMEM levels"}
            else:
                levels = stats["height"]
                byts = BYTES_PER_ELEM.get(dom, 0) * N * levels
                ach = byts / (dom_ms * 1e-3) / 1e9
                hb = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
                    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
                roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hb, "unit": "GB/s",
                        "frac": ach / hb, "traffic": traffic_bytes(args.config, dom), "launches": dom_launch,
                        "avg_launch_ms": dom_ms / dom_launch}
        # --- memory-bound grid-tier kernels: achieved GB/s on algorithmic bytes
        hbm = {}
        if prof:
            hb = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
                if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
            glev = prof.get("nn_flag", (0.0, 0))[1]  # one k_merge_nn launch per grid-tier level
            for k in ("merge_scatter", "nn_flag", "deflated_out"):
                if k in prof and prof[k][0] > 0 and glev:
                    gbs = BYTES_PER_ELEM[k] * N * glev / (prof[k][0] * 1e-3) / 1e9
                    hbm[k] = {"ms": prof[k][0], "levels": glev, "gbs": gbs, "frac_of_hbm": gbs / hb,
                              "note": "per-level working set is L2-resident at n <= 2^20"}
        # --- CPU baseline: the reference composition on this box's host cores
        import oracle as O
        cores = os.cpu_count() or 1
        cpu = None
        if O.ref_available():
            if batch:
                smp = 256
                v = cpu_reference(d[:smp], e[:smp], cores, smp, n) * batch / smp
                samp = f"{smp} of {batch} matrices, scaled x{batch // smp}"
            else:
                v = cpu_reference(d, e, cores, 0, n)
                samp = f"1 full solve ({cfg['workload']})"
            cpu = {"value": v, "unit": "s", "cores": cores, "kind": "reference", "sample": samp}
        ok = bool(np.all(np.diff(out.cpu().numpy().reshape(batch or 1, n), axis=1) >= 0))
        line = {
            "metric": METRIC, "value": mean_ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (xorshift64*, SPEC.md:595); inputs resident in HBM",
            "config": {"workload": cfg["workload"], "n": n, "batch": batch or 1,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": parallelism,
                       "leaf_cutoff": 25, "zhat": True, "stop": "tau-relative"},
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * N + 8 * (batch or 1) * (n - 1),
                    "d2h_bytes_per_step": 8 * N},
            "roofline": roof,
            "fp64_kernels": fp64 if prof else None,
            "hbm_kernels": hbm if prof else None,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
            "kernel_profile_ms": {k: round(v[0], 4) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])},
            "work": {"sum_k": stats["sum_k"], "sum_k2": stats["sum_k2"], "max_k": stats["max_k"],
                     "pole_terms": stats["pole_terms"], "pole_terms_fused": stats["pole_terms_fused"],
                     "evals": stats["evals"], "merges": stats["merges"], "height": stats["height"],
                     "k2_nonroot_fused": stats["k2_nonroot_fused"],
                     "k2_nonroot_grid": stats["k2_nonroot_grid"]},
            "fp64_peak_probe": peak,
            "sorted_output": ok,
            "ledger": vars(s.ledger()),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
