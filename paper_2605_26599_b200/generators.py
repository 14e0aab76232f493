"""Deterministic synthetic tridiagonal families.

PRNG: xorshift64* -- ``s ^= s >> 12; s ^= s << 25; s ^= s >> 27; out = s * 0x2545F4914F6CDD1D``
with ``seed = (family_id * 0x9E3779B97F4A7C15) xor n``.  A stream draws
``d[0..n)`` first, then ``e[0..n-1)``.  Uniform [0,1) = ``(out >> 11) * 2^-53``.

Families (ids recorded here; the BASELINE families are new):
  1 uniform        d ~ U[-1,1], e ~ U[0.10,0.30]           (paper)
  2 normal         d ~ N(0,1) (Box-Muller), e ~ U[0.10,0.30]
  3 toeplitz       d = 2, e = 0.25
  4 clustered      d_i = 1 + 1e-12 (i - (n+1)/2), e_i = 1e-4 (1 + 0.1 cos(0.33 i)), i 1-based
  5 sym-uniform    d, e ~ U(-1,1)                          (BASELINE configs 1, 2, 5)
  6 toeplitz121    d = 2, e = 1; lambda_k = 2 - 2 cos(k pi / (n+1))   (config 3)
  7 wilkinson      glued W21+: d_i = |i mod 21 - 10|, e = 1 inside, glue delta between
                   blocks (default 1e-10)                   (config 4)

The single-stream generator is vectorised with an exact GF(2) jump-ahead of the
(linear) xorshift state transition, so n = 2^20 takes well under a second.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
MUL = 0x2545F4914F6CDD1D
GOLD = 0x9E3779B97F4A7C15
BATCH_MIX = 0xD1B54A32D192ED03

FAMILIES = {"uniform": 1, "normal": 2, "toeplitz": 3, "clustered": 4, "sym-uniform": 5,
            "toeplitz121": 6, "wilkinson": 7}


def seed_for(family: str | int, n: int) -> int:
    fid = FAMILIES[family] if isinstance(family, str) else int(family)
    s = ((fid * GOLD) & M64) ^ int(n)
    return s if s else 0x9E3779B97F4A7C15


def _step(s: int) -> int:
    s ^= s >> 12
    s ^= (s << 25) & M64
    s ^= s >> 27
    return s


def _apply_matrix(cols: list[int], v: int) -> int:
    out = 0
    b = 0
    while v:
        if v & 1:
            out ^= cols[b]
        v >>= 1
        b += 1
    return out


def _jump_cols(steps: int) -> list[int]:
    """Columns of T^steps as a 64x64 GF(2) matrix (T = one xorshift step)."""
    cols = [_step(1 << b) for b in range(64)]  # T
    res = [1 << b for b in range(64)]          # identity
    k = steps
    while k:
        if k & 1:
            res = [_apply_matrix(cols, c) for c in res]
        cols = [_apply_matrix(cols, c) for c in cols]
        k >>= 1
    return res


_JCACHE: dict[int, np.ndarray] = {}


def xorshift_outputs(seed: int, count: int, block: int = 8192) -> np.ndarray:
    """First ``count`` xorshift64* outputs of one stream (uint64)."""
    if count <= 0:
        return np.zeros(0, np.uint64)
    nb = min(block, count)
    states = np.empty(nb, np.uint64)
    s = seed & M64
    for i in range(nb):
        s = _step(s)
        states[i] = s
    out = np.empty(count, np.uint64)
    out[:nb] = states
    if count > nb:
        if nb not in _JCACHE:
            _JCACHE[nb] = np.array(_jump_cols(nb), dtype=np.uint64)
        cols = _JCACHE[nb]
        pos = nb
        cur = states
        one = np.uint64(1)
        while pos < count:
            nxt = np.zeros(nb, np.uint64)
            for b in range(64):
                mask = (cur >> np.uint64(b)) & one
                nxt ^= mask * cols[b]
            take = min(nb, count - pos)
            out[pos:pos + take] = nxt[:take]
            cur = nxt
            pos += take
    with np.errstate(over="ignore"):
        return out * np.uint64(MUL)


def xorshift_lockstep(seeds: np.ndarray, count: int) -> np.ndarray:
    """``count`` outputs of many independent streams, shape (len(seeds), count)."""
    s = seeds.astype(np.uint64).copy()
    out = np.empty((len(s), count), np.uint64)
    with np.errstate(over="ignore"):
        for i in range(count):
            s ^= s >> np.uint64(12)
            s ^= s << np.uint64(25)
            s ^= s >> np.uint64(27)
            out[:, i] = s * np.uint64(MUL)
    return out


def _unit(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _from_uniform(family: str, n: int, u: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    ud, ue = _unit(u[..., :n]), _unit(u[..., n:])
    if family == "uniform":
        return 2.0 * ud - 1.0, 0.10 + 0.20 * ue
    if family == "sym-uniform":
        return 2.0 * ud - 1.0, 2.0 * ue - 1.0
    raise ValueError(family)


def generate(family: str, n: int, *, glue: float = 1e-10) -> tuple[np.ndarray, np.ndarray]:
    """(d, e) of order n for a named family (deterministic)."""
    if n <= 0:
        raise ValueError("n must be positive")
    if family in ("uniform", "sym-uniform"):
        u = xorshift_outputs(seed_for(family, n), 2 * n - 1)
        return _from_uniform(family, n, u)
    if family == "normal":
        u = _unit(xorshift_outputs(seed_for(family, n), 2 * n + (n - 1)))
        u1, u2 = 1.0 - u[:n], u[n:2 * n]
        d = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        return d, 0.10 + 0.20 * u[2 * n:]
    if family == "toeplitz":
        return np.full(n, 2.0), np.full(n - 1, 0.25)
    if family == "toeplitz121":
        return np.full(n, 2.0), np.full(n - 1, 1.0)
    if family == "clustered":
        i = np.arange(1, n + 1, dtype=np.float64)
        d = 1.0 + 1e-12 * (i - (n + 1) / 2.0)
        e = 1e-4 * (1.0 + 0.1 * np.cos(0.33 * i[:-1]))
        return d, e
    if family == "wilkinson":
        i = np.arange(n)
        d = np.abs((i % 21) - 10).astype(np.float64)
        e = np.ones(n - 1)
        e[(np.arange(n - 1) + 1) % 21 == 0] = glue
        return d, e
    raise ValueError(f"unknown family {family!r}")


def generate_batch(family: str, batch: int, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Config 2: batch of independent matrices; matrix b uses seed(family, n) xor b*0xD1B5...
    Returns d (batch, n), e (batch, n-1)."""
    base = seed_for(family, n)
    seeds = np.array([(base ^ ((b * BATCH_MIX) & M64)) or GOLD for b in range(batch)], dtype=np.uint64)
    u = xorshift_lockstep(seeds, 2 * n - 1)
    d, e = _from_uniform(family, n, u)
    return np.ascontiguousarray(d), np.ascontiguousarray(e)


def toeplitz121_exact(n: int) -> np.ndarray:
    k = np.arange(1, n + 1, dtype=np.float64)
    return np.sort(2.0 - 2.0 * np.cos(k * np.pi / (n + 1)))


def inf_norm(d: np.ndarray, e: np.ndarray) -> float:
    row = np.abs(d).astype(np.float64)
    if len(d) > 1:
        row[:-1] += np.abs(e)
        row[1:] += np.abs(e)
    return float(row.max())


def tolerance(d: np.ndarray, e: np.ndarray) -> float:
    """8 n eps ||T||_inf, eps = 2^-52 (BASELINE.json north_star)."""
    return 8.0 * len(d) * 2.0 ** -52 * inf_norm(d, e)
