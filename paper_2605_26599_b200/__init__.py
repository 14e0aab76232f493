"""B200-native boundary-row (BR) eigenvalue-only tridiagonal eigensolver.

Python mirror of the reference's public surface for this path
(/root/reference/proj/include/br/):

* ``TridiagonalMatrix(d, e)`` -- validates like tridiagonal.cpp:17-30 (InvalidArgument).
* ``eigenvalues(T)``            -- the ``std::vector<double> eigenvalues_qrql(const
  TridiagonalMatrix&)`` shape (qrql.hpp:20-23): all eigenvalues ascending, computed by the
  GPU BR solver through the C ABI (include/brgpu.h).
* ``br_eigenvalues(T, options)`` -- SPEC.md:348-356 ``BrResult{lambda, ledger}``.
* ``Solver``                     -- an explicit handle (device, options, host/device/batched calls).
* ``Error`` hierarchy            -- errors.hpp:9-60, one class per C-ABI status code.

There is no CPU fallback: every solve runs the sm_100a kernels in ``libbrgpu.so``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native

__all__ = [
    "Error", "InvalidArgument", "NoConvergence", "BudgetExceeded", "PoleHit", "ZeroDenominator",
    "MalformedCompactRoot", "DimensionMismatch", "DomainError", "DeviceError",
    "TridiagonalMatrix", "Block", "find_irreducible_blocks", "Solver", "BrOptions", "BrResult",
    "LedgerSnapshot", "eigenvalues", "br_eigenvalues", "workspace_query", "RowRequest",
    "split_row_request",
]


# --------------------------------------------------------------------- errors (errors.hpp:9-60)
class Error(RuntimeError):
    """Base class for all solver errors (br::Error)."""


class BudgetExceeded(Error):
    pass


class NoConvergence(Error):
    pass


class PoleHit(Error):
    pass


class ZeroDenominator(Error):
    pass


class MalformedCompactRoot(Error):
    pass


class DomainError(Error):
    pass


class DimensionMismatch(Error):
    pass


class InvalidArgument(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL / no-device failures (no reference counterpart)."""


_CODE = {1: InvalidArgument, 2: NoConvergence, 3: BudgetExceeded, 4: PoleHit, 5: ZeroDenominator,
         6: MalformedCompactRoot, 7: DimensionMismatch, 8: DomainError, 9: DeviceError}


def _raise(code: int, msg: str) -> None:
    raise _CODE.get(code, DeviceError)(msg or f"status {code}")


# ------------------------------------------------------------- input type (tridiagonal.hpp:12-25)
class TridiagonalMatrix:
    """Real symmetric tridiagonal matrix (diagonal d, off-diagonal e)."""

    def __init__(self, d, e=None):
        self.d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1)
        self.e = (np.ascontiguousarray(e, dtype=np.float64).reshape(-1) if e is not None
                  else np.zeros(0))
        self.n = len(self.d)
        self.validate()

    def validate(self) -> None:
        if self.n == 0:
            raise InvalidArgument("tridiagonal: order must be positive")
        if len(self.e) + 1 != self.n:
            raise InvalidArgument("tridiagonal: off-diagonal length != n-1")
        if not np.all(np.isfinite(self.d)):
            raise InvalidArgument("tridiagonal: non-finite diagonal entry")
        if not np.all(np.isfinite(self.e)):
            raise InvalidArgument("tridiagonal: non-finite off-diagonal entry")

    def inf_norm(self) -> float:
        row = np.abs(self.d).copy()
        if self.n > 1:
            row[:-1] += np.abs(self.e)
            row[1:] += np.abs(self.e)
        return float(row.max())


@dataclass(frozen=True)
class Block:
    offset: int
    size: int


def find_irreducible_blocks(T: TridiagonalMatrix, tol: float) -> list[Block]:
    """tridiagonal.cpp:45-58 (host mirror; the solver itself splits on the device)."""
    if tol < 0:
        raise InvalidArgument("find_irreducible_blocks: tol must be nonnegative")
    split = np.nonzero(np.abs(T.e) <= tol * (np.abs(T.d[:-1]) + np.abs(T.d[1:])))[0]
    starts = [0] + [int(i) + 1 for i in split] + [T.n]
    return [Block(a, b - a) for a, b in zip(starts[:-1], starts[1:])]


# --------------------------------------------------------------------------------- solver
@dataclass
class BrOptions:
    leaf_cutoff: int = 25
    zhat: bool = True
    patched_stop: bool = True
    use_graph: bool = True
    subtree: bool = True
    virtual_ranks: int = 1  # >1: run the multi-GPU decomposition on this device (test mode)
    exact_passes: bool = False  # test hook: every pole pass through the exact-reciprocal path
    root_split: bool = True  # multi-rank: split the shared top merges' roots across ranks
    sparse: bool = False  # opt-in: grid levels with <= C non-negligible poles per merge run the sparse pipeline
    live: bool = True  # top levels of large single-block solves on live lists (live.cu); dense fallback
    live_cluster: bool = True  # split-rule live levels: one merge per thread-block cluster (live.cu)
    live_flow: bool = True  # lane-arithmetic live levels as one dataflow launch (live.cu)


@dataclass
class LedgerSnapshot:
    live_doubles: int
    peak_doubles: int
    live_ints: int
    peak_ints: int
    limit_doubles: int
    limit_ints: int
    rows_doubles: int = 0  # requested-rows state, outside the values-only contract
    rows_ints: int = 0

    def limit_bytes(self) -> int:
        return self.limit_doubles * 8 + self.limit_ints * 4


@dataclass
class BrResult:
    lam: np.ndarray
    ledger: LedgerSnapshot
    stats: dict = field(default_factory=dict)
    selected_rows: np.ndarray | None = None  # |sigma| x n: Q[sigma_r, j], columns in lam's order


# ------------------------------------------------- row requests (Algorithm 1)
@dataclass(frozen=True)
class RowRequest:
    """Ordered local row indices sigma (1-based as in SPEC.md; duplicates allowed)."""
    sigma: tuple[int, ...] = ()

    def validate(self, size: int) -> None:
        if any(i < 1 or i > size for i in self.sigma):
            raise InvalidArgument("RowRequest: index outside the node")


def split_row_request(sigma, n_left: int, size: int | None = None):
    """SPEC.md:327-333 (Algorithm 1, "Map sigma_v and split-boundary requests"):
    sigma_L = the entries <= n_left (order kept) plus the left split-boundary row
    n_left; sigma_R = the entries > n_left shifted by -n_left (order kept) plus the
    right boundary row 1.  Returns (sigma_L, sigma_R) as RowRequests, the boundary
    row last.  The GPU solver realises this mapping positionally (a requested row
    lives in exactly one child; the other child's columns are zero, sigma.cu)."""
    sig = tuple(int(i) for i in (sigma.sigma if isinstance(sigma, RowRequest) else sigma))
    if size is not None:
        RowRequest(sig).validate(size)
    left = tuple(i for i in sig if i <= n_left) + (n_left,)
    right = tuple(i - n_left for i in sig if i > n_left) + (1,)
    return RowRequest(left), RowRequest(right)


def workspace_query(n: int) -> tuple[int, int]:
    dd, ii = C.c_int64(), C.c_int64()
    rc = _native.lib().brgpu_workspace_query(int(n), C.byref(dd), C.byref(ii))
    if rc:
        _raise(rc, "workspace_query")
    return dd.value, ii.value


class Solver:
    """One handle = one device + one stream (handles are independent; use one per thread)."""

    def __init__(self, device: int = 0, options: BrOptions | None = None, *, rank: int = 0,
                 nranks: int = 1, nccl_id: bytes | None = None):
        self._lib = _native.lib()
        h = C.c_void_p()
        if nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise InvalidArgument("distributed Solver needs the 128-byte NCCL unique id")
            buf = C.create_string_buffer(nccl_id, 128)
            rc = self._lib.brgpu_create_distributed(C.byref(h), int(device), int(rank), int(nranks), buf)
        else:
            rc = self._lib.brgpu_create(C.byref(h), int(device))
        if rc:
            _raise(rc, f"brgpu_create(device={device}): {self._lib.brgpu_status_string(rc).decode()}")
        self._h = h
        self.device = device
        self.rank, self.nranks = rank, nranks
        self.set_options(options or BrOptions())

    # options --------------------------------------------------------------
    def set_options(self, o: BrOptions) -> None:
        self._opt(_native.OPT_LEAF_CUTOFF, o.leaf_cutoff)
        self._opt(_native.OPT_ZHAT, int(o.zhat))
        self._opt(_native.OPT_PATCHED_STOP, int(o.patched_stop))
        self._opt(_native.OPT_USE_GRAPH, int(o.use_graph))
        self._opt(_native.OPT_SUBTREE, int(o.subtree))
        self._opt(_native.OPT_EXACT_PASSES, int(o.exact_passes))
        self._opt(_native.OPT_ROOT_SPLIT, int(o.root_split))
        if o.sparse or getattr(self, "_sparse_on", False):  # opt-in tier: set once enabled
            self._opt(_native.OPT_SPARSE, int(o.sparse))
            self._sparse_on = bool(o.sparse)
        if not o.live or getattr(self, "_live_off", False):  # default on: set only once turned off
            self._opt(_native.OPT_LIVE, int(o.live))
            self._live_off = not o.live
        if not o.live_cluster or getattr(self, "_cl_off", False):  # default on: set only once turned off
            self._opt(_native.OPT_LIVE_CLUSTER, int(o.live_cluster))
            self._cl_off = not o.live_cluster
        if not o.live_flow or getattr(self, "_lf_off", False):  # default on: set only once turned off
            self._opt(_native.OPT_LIVE_FLOW, int(o.live_flow))
            self._lf_off = not o.live_flow
        if self.nranks == 1:
            self._opt(_native.OPT_VIRTUAL_RANKS, int(o.virtual_ranks))
        self.options = o

    def _opt(self, k: int, v: int) -> None:
        rc = self._lib.brgpu_set_option(self._h, k, int(v))
        if rc:
            self._fail(rc)

    def _fail(self, rc: int) -> None:
        msg = self._lib.brgpu_last_error_message(self._h)
        _raise(rc, msg.decode() if msg else "")

    # solves ---------------------------------------------------------------
    def eigvals(self, d, e=None) -> np.ndarray:
        """Host arrays in, ascending eigenvalues out (H2D + solve + D2H)."""
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1)
        n = len(d)
        e = np.ascontiguousarray(e if e is not None else np.zeros(0), dtype=np.float64).reshape(-1)
        if n == 0:
            raise InvalidArgument("tridiagonal: order must be positive")
        if len(e) + 1 != n:
            raise InvalidArgument("tridiagonal: off-diagonal length != n-1")
        w = np.empty(n)
        rc = self._lib.brgpu_eigvals(self._h, n, d.ctypes.data, e.ctypes.data if n > 1 else None,
                                     w.ctypes.data)
        if rc:
            self._fail(rc)
        return w

    def eigvals_rows(self, d, e, rows) -> tuple[np.ndarray, np.ndarray]:
        """Eigenvalues and requested eigenvector rows (Algorithm 1's sigma): returns
        (w, R), R[r, j] = Q[rows[r], j] with column j belonging to w[j].  0-based
        row indices, duplicates and any order allowed (brgpu_eigvals_rows)."""
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1)
        n = len(d)
        e = np.ascontiguousarray(e if e is not None else np.zeros(0), dtype=np.float64).reshape(-1)
        if n == 0:
            raise InvalidArgument("tridiagonal: order must be positive")
        if len(e) + 1 != n:
            raise InvalidArgument("tridiagonal: off-diagonal length != n-1")
        sel = np.ascontiguousarray(rows, dtype=np.int64).reshape(-1)
        w = np.empty(n)
        R = np.empty((len(sel), n))
        rc = self._lib.brgpu_eigvals_rows(self._h, n, d.ctypes.data, e.ctypes.data if n > 1 else None,
                                          len(sel), sel.ctypes.data if len(sel) else None, w.ctypes.data,
                                          R.ctypes.data if len(sel) else None)
        if rc:
            self._fail(rc)
        return w, R

    def eigvals_device(self, d, e, w=None, stream: int | None = None):
        """torch.cuda float64 tensors in (resident in HBM), ascending eigenvalues in ``w``."""
        import torch
        n = d.numel()
        if n == 0:
            raise InvalidArgument("tridiagonal: order must be positive")
        if w is None:
            w = torch.empty(n, dtype=torch.float64, device=d.device)
        for t in (d, e, w):
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise InvalidArgument("eigvals_device: contiguous cuda float64 tensors required")
        if e.numel() + 1 != n:
            raise InvalidArgument("tridiagonal: off-diagonal length != n-1")
        if w.numel() != n:
            raise InvalidArgument("eigvals_device: w must hold n entries")
        if e.device != d.device or w.device != d.device:
            raise InvalidArgument("eigvals_device: tensors on different devices")
        s = stream if stream is not None else torch.cuda.current_stream(d.device).cuda_stream
        rc = self._lib.brgpu_eigvals_device(self._h, n, d.data_ptr(), e.data_ptr() if n > 1 else None,
                                            w.data_ptr(), s)
        if rc:
            self._fail(rc)
        return w

    def eigvals_dense_device(self, A, w=None, stream: int | None = None):
        """Dense symmetric torch.cuda float64 matrix (n x n, lower triangle used, OVERWRITTEN):
        cuSOLVER dsytrd to tridiagonal, then the BR solve (the paper's "reduced dense"
        family).  Returns ascending eigenvalues."""
        import torch
        if A.dtype != torch.float64 or not A.is_cuda or A.dim() != 2 or A.shape[0] != A.shape[1]:
            raise InvalidArgument("eigvals_dense_device: square cuda float64 matrix required")
        n = A.shape[0]
        if not A.is_contiguous():
            raise InvalidArgument("eigvals_dense_device: contiguous matrix required")
        if w is None:
            w = torch.empty(n, dtype=torch.float64, device=A.device)
        s = stream if stream is not None else torch.cuda.current_stream(A.device).cuda_stream
        # row-major contiguous storage of a symmetric matrix == its column-major storage
        rc = self._lib.brgpu_eigvals_dense_device(self._h, n, A.data_ptr(), n, w.data_ptr(), s)
        if rc:
            self._fail(rc)
        return w

    def eigvals_batched(self, d, e) -> np.ndarray:
        """d (batch, n), e (batch, n-1) host arrays -> (batch, n) ascending per matrix."""
        d = np.ascontiguousarray(d, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        batch, n = d.shape
        if e.shape != (batch, n - 1):
            raise InvalidArgument("batched: e must be (batch, n-1)")
        w = np.empty((batch, n))
        rc = self._lib.brgpu_eigvals_batched(self._h, batch, n, d.ctypes.data,
                                             e.ctypes.data if n > 1 else None, w.ctypes.data)
        if rc:
            self._fail(rc)
        return w

    def eigvals_batched_device(self, d, e, w=None, stream: int | None = None):
        """d (batch, n), e (batch, n-1) contiguous cuda float64 tensors; ascending
        eigenvalues per matrix in ``w`` (batch, n)."""
        import torch
        if not isinstance(d, torch.Tensor) or d.dim() != 2:
            raise InvalidArgument("eigvals_batched_device: d must be a (batch, n) tensor")
        batch, n = d.shape
        if batch <= 0 or n <= 0:
            raise InvalidArgument("eigvals_batched_device: batch and n must be positive")
        if w is None:
            w = torch.empty((batch, n), dtype=torch.float64, device=d.device)
        for t in (d, e, w):
            if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda \
                    or not t.is_contiguous():
                raise InvalidArgument("eigvals_batched_device: contiguous cuda float64 tensors required")
        if tuple(e.shape) != (batch, n - 1) and not (n == 1 and e.numel() == 0):
            raise InvalidArgument("batched: e must be (batch, n-1)")
        if tuple(w.shape) != (batch, n):
            raise InvalidArgument("batched: w must be (batch, n)")
        if e.device != d.device or w.device != d.device:
            raise InvalidArgument("eigvals_batched_device: tensors on different devices")
        s = stream if stream is not None else torch.cuda.current_stream(d.device).cuda_stream
        rc = self._lib.brgpu_eigvals_batched_device(self._h, batch, n, d.data_ptr(),
                                                    e.data_ptr() if n > 1 else None, w.data_ptr(), s)
        if rc:
            self._fail(rc)
        return w

    # introspection --------------------------------------------------------
    def reserve(self, n: int) -> None:
        rc = self._lib.brgpu_reserve(self._h, int(n))
        if rc:
            self._fail(rc)

    def stats(self) -> dict:
        s = _native.Stats()
        self._lib.brgpu_get_stats(self._h, C.byref(s))
        return {f: getattr(s, f) for f, _ in _native.Stats._fields_}

    def ledger(self) -> LedgerSnapshot:
        l = _native.Ledger()
        self._lib.brgpu_get_ledger(self._h, C.byref(l))
        return LedgerSnapshot(*(getattr(l, f) for f, _ in _native.Ledger._fields_))

    def timing(self) -> dict:
        """CUDA-event device time of the last solve (ms), on the handle's stream."""
        t = _native.Timing()
        self._lib.brgpu_get_timing(self._h, C.byref(t))
        return {f: getattr(t, f) for f, _ in _native.Timing._fields_}

    def profile_kernels(self, d, e, batch: int = 0) -> dict:
        """Kernel-by-kernel profile of one solve of device-resident torch tensors
        (a batch of ``batch`` matrices when batch > 0; d is then (batch, n)):
        {class: (total_ms, launches)} from CUDA events on the handle's stream."""
        ms = (C.c_double * _native.NCLASS)()
        cnt = (C.c_int32 * _native.NCLASS)()
        if batch:
            n = d.numel() // batch
            rc = self._lib.brgpu_profile_kernels_batched(self._h, batch, n, d.data_ptr(),
                                                         e.data_ptr() if n > 1 else None, ms, cnt)
        else:
            n = d.numel()
            rc = self._lib.brgpu_profile_kernels(self._h, n, d.data_ptr(),
                                                 e.data_ptr() if n > 1 else None, ms, cnt)
        if rc:
            self._fail(rc)
        return {self._lib.brgpu_kernel_class_name(c).decode(): (ms[c], cnt[c])
                for c in range(_native.NCLASS) if cnt[c]}

    def set_trace(self, on: bool) -> None:
        self._lib.brgpu_set_trace(self._h, int(on))

    def trace(self) -> list[tuple]:
        n = C.c_int64()
        self._lib.brgpu_get_trace(self._h, None, 0, C.byref(n))
        buf = (_native.Trace * max(n.value, 1))()
        self._lib.brgpu_get_trace(self._h, buf, n.value, C.byref(n))
        return [(t.level, t.is_root, t.offset, t.size, t.nn, t.k) for t in buf[: n.value]]

    def set_secular_trace(self, on: bool) -> None:
        """Record every merge's secular problem (rho, D_active, z_active) on the
        next solves (grid tier, bit-identical results) -- the Theorem 1 check."""
        rc = self._lib.brgpu_set_secular_trace(self._h, int(on))
        if rc:
            self._fail(rc)

    def secular_trace(self) -> list[tuple]:
        """Per merge of the last solve, in trace() order: (level, is_root, offset,
        size, K, rho, D_active, z_active)."""
        recs = self.trace()
        n = C.c_int64()
        rc = self._lib.brgpu_get_secular_trace(self._h, None, 0, C.byref(n))
        if rc:
            self._fail(rc)
        buf = np.empty(max(n.value, 1))
        self._lib.brgpu_get_secular_trace(self._h, buf.ctypes.data_as(C.POINTER(C.c_double)), n.value, C.byref(n))
        M = len(recs)
        rho, at, out = buf[:M], M, []
        for m, (lev, root, off, size, nn, k) in enumerate(recs):
            dz = buf[at:at + 2 * k].reshape(-1, 2)
            at += 2 * k
            out.append((lev, root, off, size, k, float(rho[m]), dz[:, 0].copy(), dz[:, 1].copy()))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.brgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be shared with the other ranks."""
    buf = C.create_string_buffer(128)
    rc = _native.lib().brgpu_nccl_unique_id(buf)
    if rc:
        _raise(rc, "brgpu_nccl_unique_id")
    return buf.raw


def distributed_solver(device: int | None = None, options: BrOptions | None = None) -> Solver:
    """One Solver per process over torch.distributed's world (torchrun): the NCCL id
    is created on rank 0 and broadcast with torch.distributed."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if device is None:
        import torch
        device = torch.cuda.current_device()
    return Solver(device, options, rank=rank, nranks=world, nccl_id=obj[0])


def plan_owned(n: int, nranks: int, leaf_cutoff: int = 25, bstart=None) -> list[list[tuple[int, int]]]:
    """Host-only: the [off, off+len) ranges each rank solves before the exchange."""
    import numpy as np
    cap = 4096
    counts = (C.c_int32 * nranks)()
    ranges = (C.c_int32 * (2 * cap * nranks))()
    b = None
    nblk = 0
    if bstart is not None:
        b = np.ascontiguousarray(bstart, dtype=np.int32)
        nblk = len(b) - 1
    rc = _native.lib().brgpu_plan_owned(int(n), int(leaf_cutoff), int(nranks),
                                        b.ctypes.data if b is not None else None, nblk, counts, ranges, cap)
    if rc:
        _raise(rc, "brgpu_plan_owned")
    return [[(ranges[2 * (k * cap + q)], ranges[2 * (k * cap + q) + 1]) for q in range(counts[k])]
            for k in range(nranks)]


_default: Solver | None = None


def _solver() -> Solver:
    global _default
    if _default is None:
        _default = Solver(0)
    return _default


def eigenvalues(T: TridiagonalMatrix) -> np.ndarray:
    """All eigenvalues of T, ascending (the eigenvalues_qrql shape, qrql.hpp:20-23)."""
    T.validate()
    s = _solver()
    s.set_options(BrOptions())
    return s.eigvals(T.d, T.e)


def br_eigenvalues(T: TridiagonalMatrix, options: BrOptions | None = None,
                   sigma: RowRequest | None = None) -> BrResult:
    """BR eigenvalues plus the workspace ledger snapshot, and
    the requested rows Q[sigma, :] when ``sigma`` (1-based RowRequest) is given."""
    T.validate()
    s = _solver()
    # options apply to this call only: the process-wide solver is reset to the
    # defaults on every call, so a previous call's options never leak
    s.set_options(options if options is not None else BrOptions())
    if sigma is not None and len(sigma.sigma):
        sigma.validate(T.n)
        lam, rows = s.eigvals_rows(T.d, T.e, np.asarray(sigma.sigma, dtype=np.int64) - 1)
        return BrResult(lam, s.ledger(), s.stats(), rows)
    lam = s.eigvals(T.d, T.e)
    return BrResult(lam, s.ledger(), s.stats())
