"""Multi-GPU decomposition -- host logic on CPU.

* the ranges each rank solves in phase 1 are disjoint and cover every block that
  is split (big blocks: the 2^D depth-D subtrees; small blocks: contiguous chunks);
* the exchange (one in-place broadcast per owned range, rooted at its owner --
  exactly what csrc/api.cpp exchange_nccl issues) replicates the full state on
  every rank: checked with a world_size-2 (and 4) gloo process group.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2605_26599_b200 as br


def _covered(owned, n):
    cov = np.zeros(n, dtype=np.int32)
    for k, rs in enumerate(owned):
        for off, ln in rs:
            cov[off:off + ln] += 1
    return cov


@pytest.mark.parametrize("n", [1 << 10, 1 << 16, 1 << 20, 100_003])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_single_block_partition(n, P):
    owned = br.plan_owned(n, P)
    cov = _covered(owned, n)
    assert cov.max() == 1 and cov.min() == 1
    D = P.bit_length() - 1
    assert sum(len(r) for r in owned) == 2 ** D
    # balanced: depth-D subtree sizes differ by at most 1 per level of splitting
    sizes = [ln for rs in owned for _, ln in rs]
    assert max(sizes) - min(sizes) <= D + 1


def test_small_blocks_split_in_chunks():
    rng = np.random.default_rng(0)
    cuts = np.sort(rng.choice(np.arange(1, 50_000), size=300, replace=False))
    bstart = np.concatenate([[0], cuts, [50_000]]).astype(np.int32)
    owned = br.plan_owned(50_000, 4, bstart=bstart)
    cov = _covered(owned, 50_000)
    assert cov.max() == 1 and cov.min() == 1
    loads = [sum(ln for _, ln in rs) for rs in owned]
    assert min(loads) > 0


def test_no_split_when_single_rank():
    assert br.plan_owned(1 << 16, 1) == [[]]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    owned = br.plan_owned(n, world)
    state = torch.full((3, n), -1.0, dtype=torch.float64)
    for off, ln in owned[rank]:  # phase 1 result of this rank
        state[:, off:off + ln] = torch.arange(off, off + ln, dtype=torch.float64) * 3 + rank * 0.25
    # exchange_nccl: for every owner k, every owned range, in-place broadcast of lam, blo, bhi
    for k in range(world):
        for off, ln in owned[k]:
            for a in range(3):
                buf = state[a, off:off + ln].clone()
                dist.broadcast(buf, src=k)
                state[a, off:off + ln] = buf
    expect = torch.empty(n, dtype=torch.float64)
    for k, rs in enumerate(owned):
        for off, ln in rs:
            expect[off:off + ln] = torch.arange(off, off + ln, dtype=torch.float64) * 3 + k * 0.25
    ok = all(torch.equal(state[a], expect) for a in range(3))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_replicates_state_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, 50_000, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]


# ---------------------------------------------------------------------------
# root-range split of the shared top merges: index ownership and the in-place
# slot all-gather (csrc/kernels.cu k_xpack / k_xunpack, csrc/api.cpp
# exchange_allgather)
# ---------------------------------------------------------------------------
def _split_chunk(n, P):
    return (n + P - 1) // P


def _pack(vals, T, P, r, c, buf):
    """k_xpack: rank r's owned active indices g = k*P + r (k < c, g < T) into slot r."""
    for k in range(c):
        g = k * P + r
        if g < T:
            buf[r * c + k] = vals[g]


def _unpack(buf, T, P, r, c, out):
    """k_xunpack: every other rank's slot back to active indices."""
    for idx in range(P * c):
        rr, k = divmod(idx, c)
        g = k * P + rr
        if rr != r and g < T:
            out[g] = buf[idx]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("T,n", [(0, 100), (1, 100), (7, 100), (100, 100), (4097, 1 << 13)])
def test_root_split_ownership_covers_each_root_once(P, T, n):
    c = _split_chunk(n, P)
    own = np.zeros(T, dtype=np.int32)
    for r in range(P):
        for k in range(c):
            g = k * P + r
            if g < T:
                own[g] += 1
    assert own.size == 0 or (own.min() == 1 and own.max() == 1)
    vals = np.arange(T, dtype=np.float64) * 1.5 + 0.25
    for r in range(P):  # after pack + all-gather + unpack every rank holds every value
        local = np.full(T, -1.0)
        for g in range(r, T, P):
            local[g] = vals[g]  # what rank r computed
        gathered = np.zeros(P * c)
        for rr in range(P):
            _pack(vals, T, P, rr, c, gathered)
        _unpack(gathered, T, P, r, c, local)
        assert np.array_equal(local, vals)


def _allgather_worker(rank, world, port, n, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    c = _split_chunk(n, world)
    vals = np.arange(T, dtype=np.float64) * 3.0 - 1.0
    buf = np.zeros(world * c)
    _pack(vals, T, world, rank, c, buf)
    # in-place all-gather of slot `rank` (ncclAllGather(buf + rank*c, buf, c))
    t = torch.from_numpy(buf)
    chunks = [torch.empty(c, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(chunks, t[rank * c:(rank + 1) * c].clone())
    t.copy_(torch.cat(chunks))
    local = np.full(T, np.nan)
    local[rank::world] = vals[rank::world]
    _unpack(t.numpy(), T, world, rank, c, local)
    q.put((rank, bool(np.array_equal(local, vals))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_root_split_allgather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allgather_worker, args=(r, world, port, 4096, 3001, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]
