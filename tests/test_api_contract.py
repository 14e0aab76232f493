"""API-contract tests of the Python mirror and the C ABI (argument checking,
per-call options, fresh-handle profiling, the workspace ledger)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G

pytestmark = pytest.mark.gpu


def test_br_eigenvalues_options_do_not_leak():
    """Options given to one br_eigenvalues call apply to that call only."""
    d, e = G.generate("sym-uniform", 3000)
    T = br.TridiagonalMatrix(d, e)
    r1 = br.br_eigenvalues(T, br.BrOptions(zhat=False, leaf_cutoff=8, virtual_ranks=2))
    assert np.array_equal(r1.lam, O.eigvals(d, e, zhat=False, leaf_cutoff=8).w)
    r2 = br.br_eigenvalues(T)
    assert np.array_equal(r2.lam, O.eigvals(d, e).w)
    assert br._solver().options == br.BrOptions()
    # a row request after a virtual-rank call must not trip 'single-device handles only'
    r3 = br.br_eigenvalues(T, sigma=br.RowRequest((1, 7)))
    assert r3.selected_rows.shape == (2, 3000)
    assert np.array_equal(br.eigenvalues(T), O.eigvals(d, e).w)


def test_profile_on_fresh_handle():
    import torch
    d, e = G.generate("sym-uniform", 50000)
    td, te = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    with br.Solver(0) as s:
        prof = s.profile_kernels(td, te)
        assert prof and all(v[0] >= 0 for v in prof.values())
    db, eb = G.generate_batch("sym-uniform", 8, 1024)
    with br.Solver(0) as s:
        prof = s.profile_kernels(torch.tensor(db, device="cuda"), torch.tensor(eb, device="cuda"), batch=8)
        assert prof


def test_batched_device_validation():
    import torch
    db, eb = G.generate_batch("sym-uniform", 4, 64)
    with br.Solver(0) as s:
        with pytest.raises(br.InvalidArgument):
            s.eigvals_batched_device(torch.tensor(db), torch.tensor(eb))  # host tensors
        with pytest.raises(br.InvalidArgument):
            s.eigvals_batched_device(torch.tensor(db, device="cuda", dtype=torch.float32),
                                     torch.tensor(eb, device="cuda", dtype=torch.float32))
        with pytest.raises(br.InvalidArgument):
            s.eigvals_batched_device(torch.tensor(db, device="cuda"), torch.tensor(eb[:, :-1], device="cuda"))
        with pytest.raises(br.InvalidArgument):
            s.eigvals_batched_device(torch.tensor(db.reshape(-1), device="cuda"), torch.tensor(eb, device="cuda"))
        w = s.eigvals_batched_device(torch.tensor(db, device="cuda"), torch.tensor(eb, device="cuda"))
        torch.cuda.synchronize()
        assert np.array_equal(w.cpu().numpy(), O.eigvals_batched(db, eb, 4, 64).reshape(4, 64))


def test_ledger_counts_every_allocation():
    """The ledger reports every device allocation of the handle, and the host-buffer
    path stays inside the 16N doubles / 7N ints contract (no extra staging)."""
    import torch
    n = 1 << 18
    d, e = G.generate("sym-uniform", n)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    with br.Solver(0) as s:
        s.eigvals(d, e)
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        L = s.ledger()
        assert L.peak_doubles <= L.limit_doubles and L.peak_ints <= L.limit_ints
        ledger_bytes = 8 * L.live_doubles + 4 * L.live_ints
        used = free0 - free1
        # device memory the handle took (allocations + the instantiated graph and
        # allocator granularity) is the ledger plus a bounded overhead
        assert used <= ledger_bytes + (96 << 20), (used, ledger_bytes)
        assert ledger_bytes >= 0.5 * (used - (96 << 20))
