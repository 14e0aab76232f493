"""ctypes binding of the product library libbrgpu.so (C ABI in include/brgpu.h).

There is no fallback: if the library is missing or no CUDA device is present the
calls raise.  The library is built in-tree by ``paper_2605_26599_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# BRGPU_LIB overrides the in-tree library (used for A/B builds in experiments).
LIB_PATH = Path(os.environ.get("BRGPU_LIB", Path(__file__).resolve().parent / "libbrgpu.so"))

_dp = C.c_void_p

OPT_LEAF_CUTOFF = 1
OPT_ZHAT = 2
OPT_PATCHED_STOP = 3
OPT_USE_GRAPH = 4
OPT_SUBTREE = 5
OPT_VIRTUAL_RANKS = 6
OPT_EXACT_PASSES = 7
OPT_ROOT_SPLIT = 8
OPT_SPARSE = 9
OPT_LIVE = 10
OPT_LIVE_CLUSTER = 11
OPT_LIVE_FLOW = 12


class Stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("blocks", C.c_int32), ("height", C.c_int32),
                ("merges", C.c_int64), ("sum_k", C.c_int64), ("sum_k2", C.c_double),
                ("sum_nn", C.c_int64), ("rotations", C.c_int64), ("evals", C.c_int64),
                ("pole_terms", C.c_double), ("zhat_terms", C.c_double), ("row_terms", C.c_double),
                ("max_k", C.c_int64), ("kernel_launches", C.c_int32), ("graph_replayed", C.c_int32),
                ("evals_fused", C.c_int64), ("pole_terms_fused", C.c_double),
                ("k2_nonroot_fused", C.c_double), ("k2_nonroot_grid", C.c_double),
                ("nn_grid", C.c_int64), ("k_grid", C.c_int64),
                ("evals_live", C.c_int64), ("pole_terms_live", C.c_double), ("k2_nonroot_live", C.c_double)]


class Ledger(C.Structure):
    _fields_ = [("live_doubles", C.c_int64), ("peak_doubles", C.c_int64), ("live_ints", C.c_int64),
                ("peak_ints", C.c_int64), ("limit_doubles", C.c_int64), ("limit_ints", C.c_int64),
                ("rows_doubles", C.c_int64), ("rows_ints", C.c_int64)]


class Trace(C.Structure):
    _fields_ = [("level", C.c_int32), ("is_root", C.c_int32), ("offset", C.c_int64),
                ("size", C.c_int64), ("nn", C.c_int64), ("k", C.c_int64)]


EXPORTS = [
    "brgpu_create", "brgpu_destroy", "brgpu_last_error_message", "brgpu_status_string",
    "brgpu_set_option", "brgpu_get_option", "brgpu_workspace_query", "brgpu_reserve",
    "brgpu_get_ledger", "brgpu_eigvals", "brgpu_eigvals_device", "brgpu_eigvals_batched",
    "brgpu_eigvals_batched_device", "brgpu_get_stats", "brgpu_set_trace", "brgpu_get_trace",
    "brgpu_get_timing", "brgpu_profile_kernels", "brgpu_profile_kernels_batched",
    "brgpu_kernel_class_name", "brgpu_selftest_rcp", "brgpu_set_secular_trace", "brgpu_get_secular_trace",
    "brgpu_nccl_unique_id", "brgpu_create_distributed", "brgpu_plan_owned", "brgpu_version",
    "brgpu_phase_cycles", "brgpu_eigvals_dense_device", "brgpu_eigvals_rows",
]

NCLASS = 22


class Timing(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("pre_ms", C.c_double), ("main_ms", C.c_double),
                ("phase1_ms", C.c_double), ("exchange_ms", C.c_double), ("phase2_ms", C.c_double)]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2605_26599_b200.build`")
    L = C.CDLL(str(LIB_PATH))
    hp = C.c_void_p
    L.brgpu_create.argtypes = [C.POINTER(hp), C.c_int]
    L.brgpu_destroy.argtypes = [hp]
    L.brgpu_last_error_message.argtypes = [hp]
    L.brgpu_last_error_message.restype = C.c_char_p
    L.brgpu_status_string.argtypes = [C.c_int]
    L.brgpu_status_string.restype = C.c_char_p
    L.brgpu_set_option.argtypes = [hp, C.c_int, C.c_int64]
    L.brgpu_get_option.argtypes = [hp, C.c_int, C.POINTER(C.c_int64)]
    L.brgpu_workspace_query.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.brgpu_reserve.argtypes = [hp, C.c_int64]
    L.brgpu_get_ledger.argtypes = [hp, C.POINTER(Ledger)]
    L.brgpu_eigvals.argtypes = [hp, C.c_int64, _dp, _dp, _dp]
    L.brgpu_eigvals_device.argtypes = [hp, C.c_int64, _dp, _dp, _dp, C.c_void_p]
    L.brgpu_eigvals_rows.argtypes = [hp, C.c_int64, _dp, _dp, C.c_int64, C.c_void_p, _dp, _dp]
    L.brgpu_eigvals_batched.argtypes = [hp, C.c_int64, C.c_int64, _dp, _dp, _dp]
    L.brgpu_eigvals_dense_device.argtypes = [hp, C.c_int64, _dp, C.c_int64, _dp, C.c_void_p]
    L.brgpu_phase_cycles.argtypes = [hp, C.c_void_p]
    L.brgpu_eigvals_batched_device.argtypes = [hp, C.c_int64, C.c_int64, _dp, _dp, _dp, C.c_void_p]
    L.brgpu_get_stats.argtypes = [hp, C.POINTER(Stats)]
    L.brgpu_set_trace.argtypes = [hp, C.c_int]
    L.brgpu_get_trace.argtypes = [hp, C.POINTER(Trace), C.c_int64, C.POINTER(C.c_int64)]
    if hasattr(L, "brgpu_set_secular_trace"):  # (older A/B builds lack the trace entry points)
        L.brgpu_set_secular_trace.argtypes = [hp, C.c_int]
        L.brgpu_get_secular_trace.argtypes = [hp, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int64)]
    L.brgpu_version.restype = C.c_char_p
    L.brgpu_get_timing.argtypes = [hp, C.POINTER(Timing)]
    L.brgpu_profile_kernels.argtypes = [hp, C.c_int64, _dp, _dp, C.POINTER(C.c_double),
                                        C.POINTER(C.c_int32)]
    L.brgpu_profile_kernels_batched.argtypes = [hp, C.c_int64, C.c_int64, _dp, _dp,
                                                C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    L.brgpu_kernel_class_name.argtypes = [C.c_int]
    L.brgpu_kernel_class_name.restype = C.c_char_p
    L.brgpu_selftest_rcp.argtypes = [hp, C.c_int64, C.c_uint64, C.POINTER(C.c_uint64)]
    L.brgpu_nccl_unique_id.argtypes = [C.c_void_p]
    L.brgpu_create_distributed.argtypes = [C.POINTER(hp), C.c_int, C.c_int, C.c_int, C.c_void_p]
    L.brgpu_plan_owned.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32]
    _lib = L
    return L
