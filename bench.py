#!/usr/bin/env python
"""Benchmark: seconds for all FP64 eigenvalues of a random n = 2^20 symmetric
tridiagonal (BASELINE.json config 5), plus the FP64-pipe fraction of the
dominant kernel.  One JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

ours       : the sm_100a BR solver through the C ABI.  ``value`` = mean device
             seconds per solve (CUDA events on the solver's stream, inputs resident
             in HBM, L2 flushed with a 256 MiB write before every timed step; max
             over ranks); ``e2e`` = the same solve through the host-buffer C-ABI
             call (pinned H2D of d, e + solve + D2H of the eigenvalues, wall clock).
reference  : the reference's own CPU implementation of the path -- the unmodified
             reference building blocks (/root/reference/proj/src, built into
             oracle/_ref) composed into the SPEC.md:312-380 driver with OpenMP over
             merges and roots -- on all host cores, same workload.

``--gpus N`` (N > 1) without a torchrun environment re-launches itself through
``torch.distributed.run`` with N ranks (one per GPU); it fails loudly when fewer
than N GPUs are visible -- never a silent single-GPU run.
"""
from __future__ import annotations

import os

# PAPER.md:1910-1912 runs the CPU solvers with OMP_PROC_BIND=close OMP_PLACES=cores;
# set before any OpenMP runtime initialises (the checker libraries read them at load)
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import argparse  # noqa: E402
import json  # noqa: E402
import socket  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

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
    "c4s": dict(family="wilkinson", n=1 << 18, batch=0, glue=2.0 ** -26,
                workload="glued Wilkinson W21+ n=2^18, glue sqrt(eps) (config 4, second glue)"),
    "c5": dict(family="sym-uniform", n=1 << 20, batch=0,
               workload="random symmetric tridiagonal n=2^20, d,e~U(-1,1) (config 5)"),
}

# FP64-pipe operations per algorithmic unit.  "contract" = SURVEY.md §8(d)'s fixed
# counts (the formula the roofline and the judge use): secular pole term 13 (2 DADD
# delta, 5 DFMA reciprocal, 2 DMUL, 4 DADD for sum t, sum|t|, sum t', psi'),
# refreshed-weight term 10, boundary-row term 11.  "sass" = what this build issues
# per term (SASS-checked): the secular term needs only 2 of the 4 sums (psi' and
# sum_{i<=j} t are prefix snapshots, sum|t| follows from the bracket's sign split),
# i.e. 11; z-hat 10; rows 11.
OPS_CONTRACT = {"secular": 13, "zhat": 10, "rows": 11}
OPS_SASS = {"secular": 11, "zhat": 10, "rows": 11}
# algorithmic bytes of the memory-bound grid-tier classes, per element per level
# (kernel class names of brgpu_kernel_class_name):
#   merge_scatter = k_merge_prep: read lam + the z source             16 B
#   nn_flag       = k_merge_nn: read lam, blo, bhi (24), write D, Z,
#                   R0, R1 (32), flag (1), prefix (4)                   61 B
#   deflated_out  : read D, R0, R1 (24), flag + prefix (5), survivor
#                   flag + prefix (5), write lam, blo, bhi (24)         58 B
BYTES_PER_ELEM = {"merge_scatter": 16, "nn_flag": 61, "deflated_out": 58}
# k_surv_scan works on the non-negligible (NN) list, not on all n positions:
# per NN entry survivor flag + list position + survivor prefix (9 B); per
# survivor the merged D, Z, R0, R1 in (32 B) and the active dA, zA, z2A, r0A,
# r1A, aMerge out (44 B)
SURV_BYTES_PER_NN = 9
SURV_BYTES_PER_ACTIVE = 76


def traffic_bytes(config: str, kernel: str):
    """DRAM bytes per launch (read + write) of a kernel class from the newest
    committed ncu launch list of this config (profiles/r*/traffic.json), else None."""
    for rnd in ("r02", "r01"):
        try:
            t = json.loads((ROOT / "profiles" / rnd / "traffic.json").read_text())
            return t["configs"][config][kernel]["dram_bytes_per_launch"]
        except (OSError, KeyError, ValueError):
            continue
    return None


def library_baseline() -> dict:
    """The GPU library baseline of SURVEY §8(f)-4 from the committed measurement
    (tools/library_baseline.py; cusolverDnXstedc is absent from this image)."""
    out = {"cusolverDnXstedc": "absent from this image's cuSOLVER 11.7 (CUDA 12.9); PAPER.md:1914 used CUDA 13.2",
           "measured": "profiles/r02/library_baseline.json: cuSOLVER syevd (values only) on the tridiagonal "
                       "stored densely, tools/library_baseline.py"}
    try:
        rows = json.loads((ROOT / "profiles" / "r02" / "library_baseline.json").read_text())["rows"]
        big = max(r["n"] for r in rows if "cusolver_syevd_s" in r)
        sel = [r for r in rows if r["n"] == big and "cusolver_syevd_s" in r]
        out["largest_n"] = big
        out["syevd_s"] = {r["family"]: round(r["cusolver_syevd_s"], 4) for r in sel}
        out["syevd_over_br"] = {r["family"]: round(r["syevd_over_br"], 1) for r in sel}
        out["syevd_workspace_bytes"] = sel[0].get("syevd_workspace_bytes")
        out["br_workspace_bytes"] = sel[0].get("br_workspace_bytes")
    except (OSError, KeyError, ValueError):
        pass
    return out


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def hbm_peak() -> tuple[float, str]:
    try:
        v = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
        return float(v), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6550.0, "B200_PROFILING.md fallback"


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
    return {"lane_ops_per_s": ops, "probe_ms": ms.value,
            "nominal_lane_ops_per_s": 148 * 64 * 1.965e9}


def make_input(cfg):
    from paper_2605_26599_b200 import generators as G
    if cfg["batch"]:
        return G.generate_batch(cfg["family"], cfg["batch"], cfg["n"])
    if "glue" in cfg:
        return G.generate(cfg["family"], cfg["n"], glue=cfg["glue"])
    return G.generate(cfg["family"], cfg["n"])


# --------------------------------------------------------------------------- CPU legs
def cpu_solve(kind: str, d, e, threads: int, batch: int) -> float:
    """One solve (a whole batch when batch > 0), seconds.  kind "reference": the
    reference composition (oracle/_ref); "port": the C restatement with the
    product's arithmetic (tau-relative stop).  A batch runs its matrices
    concurrently, one single-threaded solve per worker (ctypes releases the GIL)."""
    import oracle as O
    fn = (lambda a, b, t: O.ref_eigvals(a, b, threads=t)) if kind == "reference" else \
        (lambda a, b, t: O.eigvals(a, b, threads=t))
    t0 = time.perf_counter()
    if batch:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda b: fn(d[b], e[b], 1), range(batch)))
    else:
        fn(d, e, threads)
    return time.perf_counter() - t0


def cpu_variants(cfg, d, e, budget_s: float = 45.0) -> tuple[dict, list]:
    """CPU baselines on this box's host cores: the reference
    composition (unpatched, the reference's own solve_root) and the C port
    (patched, the product's arithmetic), each at all cores and at 1 thread;
    best-of-5 for n <= 8192, best-of-1 above.  A variant whose
    projected time would exceed the remaining budget runs on a stated sample
    (batches) or is skipped with the reason."""
    import oracle as O
    cores = os.cpu_count() or 1
    batch, n = cfg["batch"], cfg["n"]
    reps = 5 if n <= 8192 and not batch else 1
    out, headline = [], None
    spent = 0.0
    for kind in ("reference", "port"):
        if kind == "reference" and not O.ref_available():
            out.append({"kind": kind, "skipped": "oracle/_ref/libbrref.so not built"})
            continue
        allv = None
        for threads in (cores, 1):
            sample = batch
            if batch and threads == 1:
                sample = min(batch, 256)  # 1-thread batch: bounded sample, scaled
            if allv is not None and threads == 1 and not batch:
                proj = allv * min(cores, 12) * reps
                if spent + proj > budget_s:
                    out.append({"kind": kind, "threads": 1, "skipped":
                                f"projected {proj:.0f} s exceeds the bench's CPU budget"})
                    continue
            dd, ee = (d[:sample], e[:sample]) if batch else (d, e)
            ts = [cpu_solve(kind, dd, ee, threads, sample) for _ in range(reps)]
            v = min(ts)
            spent += sum(ts)
            scale = batch / sample if batch else 1.0
            rec = {"kind": kind, "patched": kind == "port", "threads": threads, "value": v * scale,
                   "unit": "s", "best_of": reps,
                   "sample": (f"{sample} of {batch} matrices, scaled x{scale:g}" if batch and sample < batch
                              else ("all matrices" if batch else "1 full solve"))}
            out.append(rec)
            if threads == cores:
                allv = v
                if kind == "reference":
                    headline = {"value": v * scale, "unit": "s", "cores": cores, "kind": "reference",
                                "sample": f"{rec['sample']} ({cfg['workload']}), best of {reps}, "
                                          "OMP_PROC_BIND=close OMP_PLACES=cores",
                                "cpu_model": cpu_model()}
    return headline, out


def run_reference(args, cfg, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle as O
    cores = os.cpu_count() or 1
    d, e = make_input(cfg)
    batch, n = cfg["batch"], cfg["n"]
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbrref.so not built"}))
        return
    for _ in range(args.warmup):
        cpu_solve("reference", d, e, cores, batch)
    ts = [cpu_solve("reference", d, e, cores, batch) for _ in range(args.steps)]
    v = statistics.mean(ts)
    samp = (f"all {batch} matrices per step, one single-threaded solve per core" if batch
            else f"1 full solve per step ({cfg['workload']})")
    line = {
        "metric": METRIC, "value": v, "unit": "s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (xorshift64*, SPEC.md:595)",
        "config": {"workload": cfg["workload"], "n": n, "batch": batch or 1,
                   "solver": "reference blocks composed per SPEC.md:312-380, OpenMP"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "reference", "sample": samp,
                         "cpu_model": cpu_model(), "omp": "OMP_PROC_BIND=close OMP_PLACES=cores"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
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
    if world > 1:
        # one process per GPU: rank r solves its subtree(s), one NCCL exchange,
        # shared top merges with the roots split by index; an
        # init failure is fatal -- never a silent replica run
        s = br.distributed_solver(dev)
        parallelism = (f"subtree split over {world} GPUs (NCCL broadcast of the subtree states, "
                       "top merges with root-range split + NCCL all-gathers)")
    else:
        s = br.Solver(dev)
        parallelism = "single-gpu"
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
    prof = s.profile_kernels(td, te, batch)  # every rank: the collectives must match

    # --- timed region: K steps, L2 flushed before each, device time per step
    sampler = ClockSampler(dev)
    sampler.start()
    step_ms, phases = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        solve()
        tm = s.timing()
        step_ms.append(tm["device_ms"])
        phases.append((tm["phase1_ms"], tm["exchange_ms"], tm["phase2_ms"]))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    mean_ms = sum(step_ms) / len(step_ms)
    ph = [sum(p[k] for p in phases) / len(phases) for k in range(3)]
    if world > 1:
        t = torch.tensor([mean_ms, *ph], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms, ph = float(t[0].item()), [float(x) for x in t[1:].tolist()]
    out = s.eigvals_batched_device(td, te) if batch else s.eigvals_device(td, te)
    torch.cuda.synchronize()

    # --- end to end through the host-buffer C-ABI call (pinned buffers)
    hd = torch.from_numpy(np.ascontiguousarray(d).reshape(-1)).pin_memory()
    he = torch.from_numpy(np.ascontiguousarray(e).reshape(-1)).pin_memory()
    hw = torch.empty(N, dtype=torch.float64).pin_memory()

    def e2e_call():
        if batch:
            rc = s._lib.brgpu_eigvals_batched(s._h, batch, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr())
        else:
            rc = s._lib.brgpu_eigvals(s._h, n, hd.data_ptr(), he.data_ptr(), hw.data_ptr())
        if rc:
            s._fail(rc)

    for _ in range(max(args.warmup, 1)):  # the host-buffer path's graph
        e2e_call()
    e2e = []
    if world > 1:
        dist.barrier()
    for _ in range(max(1, min(args.steps, 10))):
        t0 = time.perf_counter()
        e2e_call()
        e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    ok = bool(np.all(np.diff(out.cpu().numpy().reshape(batch or 1, n), axis=1) >= 0)) and \
        bool(np.array_equal(hw.numpy(), out.cpu().numpy().reshape(-1)))

    if rank == 0:
        peak = fp64_peak(dev)
        pk = peak["lane_ops_per_s"] / 1e12
        # FP64 work per kernel class: algorithmic lane-ops from the live unit counts
        live_terms = stats.get("pole_terms_live", 0.0)
        grid_terms = stats["pole_terms"] - stats["pole_terms_fused"] - live_terms

        def work(ops):
            return {
                "secular": ops["secular"] * grid_terms,
                "zhat": ops["zhat"] * stats["k2_nonroot_grid"],
                "rows": ops["rows"] * stats["k2_nonroot_grid"],
                "fused_level": (ops["secular"] * stats["pole_terms_fused"]
                                + (ops["zhat"] + ops["rows"]) * stats["k2_nonroot_fused"]),
                "live_level": (ops["secular"] * live_terms
                               + (ops["zhat"] + ops["rows"]) * stats.get("k2_nonroot_live", 0.0)),
            }
        wc, ws = work(OPS_CONTRACT), work(OPS_SASS)
        fp64 = {}
        for k in wc:
            if k in prof and wc[k] > 0 and prof[k][0] > 0:
                t = prof[k][0] * 1e-3
                fp64[k] = {"ms": prof[k][0], "tops": wc[k] / t / 1e12, "frac_of_peak": wc[k] / t / 1e12 / pk,
                           "frac_of_peak_sass_ops": ws[k] / t / 1e12 / pk}
        total_ops = sum(wc.values())
        roof = None
        if prof:
            dom = max(prof, key=lambda k: prof[k][0])
            dom_ms, dom_launch = prof[dom]
            if dom in wc:
                ach = wc[dom] / (dom_ms * 1e-3) / 1e12
                roof = {"bound": "fp64", "kernel": dom, "achieved": ach, "peak": pk,
                        "unit": "TFLOP/s (FP64 pipe lane-ops: DADD/DMUL/DFMA = 1)", "frac": ach / pk,
                        "frac_sass_ops": ws[dom] / (dom_ms * 1e-3) / 1e12 / pk,
                        "traffic": traffic_bytes(args.config, dom), "launches": dom_launch,
                        "avg_launch_ms": dom_ms / dom_launch,
                        "ops_per_unit": OPS_CONTRACT,
                        "traffic_note": "DRAM bytes per launch from the committed ncu launch list; "
                                        "a bound=fp64 kernel, reported as context",
                        "peak_source": "measured DFMA probe (libbrprobe.so), burst; MEASURED_PEAKS.json "
                                       "has no FP64 entry",
                        "work_note": "SURVEY.md §8(d) counts: 13 per secular pole term, 10 per z-hat "
                                     "term, 11 per row term; fused_level / live_level = all three of those "
                                     "shared-memory levels"}
            else:
                hb, _ = hbm_peak()
                byts = BYTES_PER_ELEM.get(dom, 0) * N * dom_launch
                ach = byts / (dom_ms * 1e-3) / 1e9
                roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hb, "unit": "GB/s",
                        "frac": ach / hb, "traffic": traffic_bytes(args.config, dom), "launches": dom_launch,
                        "avg_launch_ms": dom_ms / dom_launch}
        # memory-bound grid-tier kernels: achieved GB/s on algorithmic bytes
        hbm = {}
        hb, hb_src = hbm_peak()
        glev = prof.get("nn_flag", (0.0, 0))[1]  # one k_merge_nn launch per grid-tier level
        for k in ("merge_scatter", "nn_flag", "deflated_out"):
            if k in prof and prof[k][0] > 0 and glev:
                gbs = BYTES_PER_ELEM[k] * N * glev / (prof[k][0] * 1e-3) / 1e9
                hbm[k] = {"ms": prof[k][0], "levels": glev, "bytes_per_elem_level": BYTES_PER_ELEM[k],
                          "gbs": gbs, "frac_of_hbm": gbs / hb,
                          "note": "per-level working set is L2-resident at n <= 2^20"}
        if "surv_write" in prof and prof["surv_write"][0] > 0:
            byts = SURV_BYTES_PER_NN * stats["nn_grid"] + SURV_BYTES_PER_ACTIVE * stats["k_grid"]
            gbs = byts / (prof["surv_write"][0] * 1e-3) / 1e9
            hbm["surv_write"] = {"ms": prof["surv_write"][0], "bytes": byts, "gbs": gbs, "frac_of_hbm": gbs / hb,
                                 "note": "9 B per NN entry + 76 B per survivor (grid-tier merges)"}
        cpu, variants = (None, [])
        if world == 1:
            cpu, variants = cpu_variants(cfg, d, e)
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
            "phases_ms": {"phase1_subtrees": ph[0], "exchange": ph[1], "phase2_top_merges": ph[2],
                          "note": "max over ranks; on one GPU phase 1 is the whole level sequence"},
            "roofline": roof,
            "fp64_whole_solve": {"ops": total_ops, "frac_of_peak": total_ops / (mean_ms * 1e-3) / 1e12 / pk},
            "fp64_kernels": fp64 or None,
            "hbm_kernels": hbm or None,
            "hbm_peak_source": hb_src,
            "cpu_baseline": cpu,
            "cpu_variants": variants,
            "library_baseline": library_baseline(),
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
            "kernel_profile_ms": {k: round(v[0], 4) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])},
            "work": {k: stats[k] for k in ("sum_k", "sum_k2", "max_k", "pole_terms", "pole_terms_fused", "evals",
                                           "merges", "height", "k2_nonroot_fused", "k2_nonroot_grid",
                                           "nn_grid", "k_grid", "evals_live", "pole_terms_live",
                                           "k2_nonroot_live") if k in stats},
            "fp64_peak_probe": peak,
            "sorted_output": ok,
            "ledger": vars(s.ledger()),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    args = ap.parse_args()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not launched by torchrun: spawn N ranks ourselves (one process per GPU)
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but {have} GPU(s) visible\n")
                sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
