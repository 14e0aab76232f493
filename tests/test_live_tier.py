"""The live-list tier (BRGPU_OPT_LIVE, csrc/live.cu): the top levels of a large
single-block solve keep only each node's live elements and bucket-sort the rest
at the root.  Checked against the checker (bit-exact), against the dense tiers
(bit-exact eigenvalues, identical per-merge (nn, K) traces), on non-power-of-two
trees, through the host-buffer path, and on inputs where the tier cannot prove a
solve exact (Toeplitz: every pole stays live; glued Wilkinson) -- those are redone
on the dense tiers with the same results."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dense_solver():
    s = br.Solver(0, br.BrOptions(live=False))
    yield s
    s.close()


def _live_ran(s, d, e) -> bool:
    import torch
    prof = s.profile_kernels(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"))
    return prof.get("live_level", (0.0, 0))[1] > 0


@pytest.fixture(scope="module")
def live_solver():
    # its own handle: a shared one may be backing off the tier at an order where an
    # earlier test's input fell back
    s = br.Solver(0)
    yield s
    s.close()


@pytest.mark.parametrize("fam,n", [("sym-uniform", 1 << 16), ("normal", 40000), ("uniform", 65537),
                                   ("sym-uniform", 131072)])
def test_live_bitwise_vs_checker(live_solver, fam, n):
    d, e = G.generate(fam, n)
    ref = O.eigvals(d, e).w
    for _ in range(2):  # the second solve replays the captured graph
        w = live_solver.eigvals(d, e)
        assert np.array_equal(w.view(np.int64), ref.view(np.int64)), f"max diff {np.max(np.abs(w - ref)):.3e}"
    assert _live_ran(live_solver, d, e)


@pytest.mark.parametrize("fam,n", [("sym-uniform", 1 << 20), ("sym-uniform", 100003), ("normal", 300001),
                                   ("uniform", 1 << 18)])
def test_live_matches_dense(live_solver, dense_solver, fam, n):
    d, e = G.generate(fam, n)
    live_solver.set_trace(True)
    dense_solver.set_trace(True)
    try:
        w1 = live_solver.eigvals(d, e)
        t1 = live_solver.trace()
        w0 = dense_solver.eigvals(d, e)
        t0 = dense_solver.trace()
    finally:
        live_solver.set_trace(False)
        dense_solver.set_trace(False)
    assert np.array_equal(w1.view(np.int64), w0.view(np.int64))
    assert t1 == t0
    assert np.all(np.diff(w1) >= 0)


@pytest.mark.parametrize("fam,n", [("toeplitz121", 1 << 16), ("wilkinson", 1 << 17), ("clustered", 40000)])
def test_live_fallback_is_exact(fam, n, dense_solver):
    # a fresh handle: its first solve of this order tries the live tier, falls back
    # and redoes the solve densely; later solves plan densely for this order
    d, e = G.generate(fam, n)
    s = br.Solver(0)
    try:
        w_first = s.eigvals(d, e)  # host-buffer path: the input is re-staged for the retry
        w_again = [s.eigvals(d, e) for _ in range(3)]  # the dense back-off
    finally:
        s.close()
    w0 = dense_solver.eigvals(d, e)
    assert np.array_equal(w_first, w0) and all(np.array_equal(w, w0) for w in w_again)


def test_live_device_path_and_option(live_solver):
    import torch
    d, e = G.generate("sym-uniform", 1 << 17)
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w = live_solver.eigvals_device(td, te).cpu().numpy()
    assert np.array_equal(w, O.eigvals(d, e).w)
    s = br.Solver(0, br.BrOptions(live=False))
    try:
        assert not _live_ran(s, d, e)
        assert np.array_equal(s.eigvals_device(td, te).cpu().numpy(), w)
    finally:
        s.close()


def test_live_scaled_and_shifted(live_solver):
    # block scaling (|T| >> 1) and a shifted spectrum: the final sort sees the
    # scaled values (the rescale follows it)
    d, e = G.generate("sym-uniform", 1 << 16)
    for sc, sh in ((2.0 ** 40, 0.0), (1.0, 1e3), (2.0 ** -30, -5.0)):
        dd, ee = d * sc + sh, e * sc
        assert np.array_equal(live_solver.eigvals(dd, ee), O.eigvals(dd, ee).w)


def _special(kind, n, rng):
    if kind == "graded":
        return np.exp(-np.linspace(0, 30, n)) * rng.uniform(-1, 1, n), rng.uniform(-1, 1, n - 1) * 1e-3
    if kind == "tiny-e":
        return rng.uniform(-1, 1, n), rng.uniform(-1, 1, n - 1) * 1e-9
    if kind == "repeated":
        return np.round(rng.uniform(-1, 1, n), 2), rng.uniform(-1, 1, n - 1) * 0.3
    if kind == "spikes":
        d = rng.uniform(-1, 1, n)
        d[::97] *= 1e6
        return d, rng.uniform(-1, 1, n - 1)
    return np.ones(n), rng.uniform(0.5, 1, n - 1)  # "ones": nothing deflates (fallback)


@pytest.mark.parametrize("kind", ["graded", "tiny-e", "repeated", "spikes", "ones"])
@pytest.mark.parametrize("n", [65536, 100001])
def test_live_special_inputs_vs_checker(kind, n):
    # graded / tiny-coupling / repeated / spiked / undeflatable inputs: whether the
    # tier holds or falls back, the result is the checker's bit for bit
    d, e = _special(kind, n, np.random.default_rng(11))
    s = br.Solver(0)
    try:
        w = s.eigvals(d, e)
    finally:
        s.close()
    assert np.array_equal(w.view(np.int64), O.eigvals(d, e).w.view(np.int64))


def test_live_batch_blocks_vs_checker():
    # a batch of 64 matrices of 4096: every block's three top levels are live and each
    # block is sorted by its own CTA at the end
    import torch
    rng = np.random.default_rng(3)
    batch, n = 64, 4096
    d = rng.uniform(-1, 1, (batch, n))
    e = rng.uniform(-1, 1, (batch, n - 1))
    s = br.Solver(0)
    try:
        w = s.eigvals_batched(d, e)
        prof = s.profile_kernels(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"), batch)
    finally:
        s.close()
    ref = O.eigvals_batched(d.reshape(-1), e.reshape(-1), batch, n)
    assert np.array_equal(np.asarray(w).reshape(-1).view(np.int64), np.asarray(ref).reshape(-1).view(np.int64))
    assert prof.get("live_level", (0.0, 0))[1] > 0


@pytest.mark.parametrize("big", [False, True])
def test_live_natural_blocks_vs_checker(big):
    # natural splits (zero couplings) into blocks of <= 4096, or with one block too large
    # for the per-block sort (the tier then stays off): the checker's result either way
    rng = np.random.default_rng(4)
    n = 1 << 17
    d, e = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n - 1)
    cuts = np.arange(4096, n, 4096) - 1
    if big:
        cuts = cuts[cuts > 3 * 4096]
    e[cuts] = 0.0
    s = br.Solver(0)
    try:
        w = s.eigvals(d, e)
    finally:
        s.close()
    assert np.array_equal(w.view(np.int64), O.eigvals(d, e).w.view(np.int64))


@pytest.mark.parametrize("fam,n", [("sym-uniform", 1 << 20), ("normal", 300001), ("uniform", 1 << 17),
                                   ("sym-uniform", 70001)])
def test_live_cluster_matches_single_cta(live_solver, fam, n):
    # split-rule live levels on thread-block clusters (one merge per cluster, roots /
    # weights / rows shared over DSMEM) against one merge per CTA with the dataflow
    # top run: bit-identical eigenvalues and per-merge (nn, K) traces
    d, e = G.generate(fam, n)
    s = br.Solver(0, br.BrOptions(live_cluster=False))
    live_solver.set_trace(True)
    s.set_trace(True)
    try:
        w1 = live_solver.eigvals(d, e)
        t1 = live_solver.trace()
        w0 = s.eigvals(d, e)
        t0 = s.trace()
        import ctypes
        v = ctypes.c_int64(-1)
        assert s._lib.brgpu_get_option(s._h, 11, ctypes.byref(v)) == 0 and v.value == 0
        assert live_solver._lib.brgpu_get_option(live_solver._h, 11, ctypes.byref(v)) == 0 and v.value == 1
    finally:
        live_solver.set_trace(False)
        s.close()
    assert np.array_equal(w1.view(np.int64), w0.view(np.int64))
    assert t1 == t0


def test_live_many_split_merges_vs_checker(live_solver):
    # n ~ 3M: the first split-rule live level has ~180 merges (> SMs), which run
    # on lane groups with G merges per CTA (k_live_level MODE 3), the few-merge
    # levels above it on clusters -- bit-identical to the checker
    n = 3_000_017
    d, e = G.generate("sym-uniform", n)
    ref = O.eigvals(d, e).w
    w = live_solver.eigvals(d, e)
    assert np.array_equal(w.view(np.int64), ref.view(np.int64)), f"max diff {np.max(np.abs(w - ref)):.3e}"
    assert _live_ran(live_solver, d, e)


@pytest.mark.parametrize("fam,n", [("sym-uniform", 1 << 20), ("uniform", 1 << 18), ("normal", 1 << 17)])
def test_live_flow_matches_per_level(live_solver, fam, n):
    # the lane-arithmetic live levels as one dataflow launch (k_live_flow: ticketed
    # work items, a batch starts when its children are done) against one launch per
    # level: bit-identical eigenvalues and per-merge (nn, K) traces
    d, e = G.generate(fam, n)
    s = br.Solver(0, br.BrOptions(live_flow=False))
    live_solver.set_trace(True)
    s.set_trace(True)
    try:
        w1 = live_solver.eigvals(d, e)
        t1 = live_solver.trace()
        w0 = s.eigvals(d, e)
        t0 = s.trace()
        import ctypes
        v = ctypes.c_int64(-1)
        assert s._lib.brgpu_get_option(s._h, 12, ctypes.byref(v)) == 0 and v.value == 0
    finally:
        live_solver.set_trace(False)
        s.close()
    assert np.array_equal(w1.view(np.int64), w0.view(np.int64))
    assert t1 == t0
    assert np.array_equal(w1, O.eigvals(d, e).w)
