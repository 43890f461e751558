"""Recursive Sherman-Morrison-Woodbury factorization and tree solves on the
GPU (solver.py of the reference).

``factorize`` replays the operator's level program (hks_factorize): the leaf
level evaluates K_aa + lam I into its LU storage and runs batched partial-
pivot LU, phi = A^-1 P^T and theta = P phi; every internal level assembles
Z = I + [[0, th_l C], [th_r C^T, 0]], factors it (plus the dgecon estimate),
and forms theta / child_push from folded = B Z^-1 thhat -- solver.py:111-186.
``solve`` runs the up / down sweeps for all right-hand sides at once
(solver.py:189-270).  Host views of every factor are materialised lazily.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .linalg import DenseFactor, SingularMatrixError


_HOST_TRACE = bool(__import__("os").environ.get("HKS_HOST_TRACE"))


class FactorizationError(RuntimeError):
    """Reduced system singular; remedy is a larger lambda or tighter tau."""


@dataclass(frozen=True)
class NodeFactor:
    diag_lu: DenseFactor | None = None
    phi: np.ndarray | None = None
    theta: np.ndarray | None = None
    z_lu: DenseFactor | None = None
    child_push: np.ndarray | None = None
    z_cond: float = 0.0


class _Factors(Mapping):
    def __init__(self, f):
        # weak back-reference: no Factorization <-> _Factors cycle, so the
        # factor storage is released as soon as the Factorization is dropped
        self._f = weakref.proxy(f)
        self._cache = {}

    def __getitem__(self, i):
        i = int(i)
        if not 0 <= i < self._f.layout.nn:
            raise KeyError(i)
        if i not in self._cache:
            self._cache[i] = self._f._node_factor(i)
        return self._cache[i]

    def __iter__(self):
        return iter(range(self._f.layout.nn))

    def __len__(self):
        return self._f.layout.nn


class Factorization:
    """tree, skeletons, lam, factors, couplings, level_seconds, max_rank,
    solve(), z_cond_per_level() (solver.py:56-83)."""

    def __init__(self, op, lam, bufs, level_seconds, z_cond=None):
        self.op = op
        self.tree = op.tree
        self.skeletons = op.skeletons
        self.lam = lam
        self.layout = op.layout
        self.bufs = bufs
        self.couplings = op.couplings
        self.level_seconds = level_seconds
        ranks = op.skeletons.ranks
        self.max_rank = int(ranks[1:].max()) if ranks.size > 1 else 0
        self._zc = z_cond
        self.factors = _Factors(self)

    @property
    def _z_cond(self):
        """Per-node z_cond, read once the asynchronous dgecon estimates of
        this factorization are done (hks_factor_stats waits for them)."""
        if self._zc is None:
            z = np.zeros(self.layout.nn)
            N.call("hks_factor_stats", self.op.plan.handle, self.buffers(), z.ctypes.data_as(N._DP), None,
                   N.stream_ptr())
            self._zc = z
        return self._zc

    def join_cond(self):
        """Make the current stream wait (device-side) for the dgecon
        estimates (they run on op.plan.cond_stream)."""
        N.call("hks_cond_wait", self.op.plan.handle, N.stream_ptr())

    @property
    def n(self):
        return self.tree.n

    def solve(self, b, in_tree_order=False):
        return solve(self, b, in_tree_order=in_tree_order)

    def z_cond_per_level(self):
        out = {}
        for lev in range(self.tree.depth):
            first = (1 << lev) - 1
            out[lev] = float(self._z_cond[first: 2 * first + 1].max())
        return out

    def buffers(self):
        return self.op.buffers(self.bufs)

    # --- host views ------------------------------------------------------------
    def _mat(self, buf, i, rows, cols):
        off = int(self.layout.off[buf, i])
        if rows == 0 or cols == 0:
            return np.zeros((rows, cols))
        return self.bufs[buf][off: off + rows * cols].view(cols, rows).t().cpu().numpy().copy()

    def _node_factor(self, i):
        ranks = self.skeletons.ranks
        depth = self.tree.depth
        leaf = i >= (1 << depth) - 1
        r = int(ranks[i]) if i > 0 else 0
        if leaf:
            m = int(self.tree._end[i] - self.tree._begin[i])
            po = int(self.layout.off[N.BUF_LEAF_PIV, i])
            dl = DenseFactor(self._mat(N.BUF_LEAF_LU, i, m, m),
                             self.bufs[N.BUF_LEAF_PIV][po: po + m].cpu().numpy())
            if i == 0:
                return NodeFactor(diag_lu=dl)
            return NodeFactor(diag_lu=dl, phi=self._mat(N.BUF_PHI, i, m, r),
                              theta=self._mat(N.BUF_THETA, i, r, r))
        R = int(ranks[2 * i + 1] + ranks[2 * i + 2])
        po = int(self.layout.off[N.BUF_Z_PIV, i])
        zl = DenseFactor(self._mat(N.BUF_Z_LU, i, R, R), self.bufs[N.BUF_Z_PIV][po: po + R].cpu().numpy())
        if i == 0:
            return NodeFactor(z_lu=zl, z_cond=float(self._z_cond[i]))
        return NodeFactor(z_lu=zl, theta=self._mat(N.BUF_THETA, i, r, r),
                          child_push=self._mat(N.BUF_PUSH, i, R, r), z_cond=float(self._z_cond[i]))


class FactorStorage:
    """Reusable factor storage of one operator.  Each Factorization leases
    a set of the flat factor buffers; dropping it returns the set with an
    event on the condition stream (its dgecon estimates may still read
    Z_LU / STATS) and one on the caller's current stream (solves queued
    there may still read the factors; work on OTHER streams must be
    ordered before the drop by the caller, as for any torch tensor).  A set
    is handed out again only once both events have completed (queried, never waited for); otherwise a new set is
    allocated.  The pool therefore settles at the number of sets the
    caller's pattern keeps in flight, and steady-state factorizations
    allocate nothing: a GB-sized cudaMalloc inside a factorize costs tens
    to hundreds of milliseconds (measured)."""

    def __init__(self, layout, cond_stream, min_elems=None):
        self.layout = layout
        self.cond_stream = cond_stream
        self.min_elems = min_elems or {}
        self.free = []  # [bufs, event]
        self.created = 0  # sets allocated so far

    def _new(self):
        bufs = {b: self.layout.alloc(b, min_elems=self.min_elems.get(b, 1)) for b in _FACTOR_BUFS}
        self.created += 1
        return bufs

    def reserve(self, total):
        """Grow the pool to `total` sets up front (e.g. before a timed loop),
        or as many as device memory holds.  Returns the number of sets."""
        while self.created < total:
            try:
                self.free.append((self._new(), None))
            except N.torch().cuda.OutOfMemoryError:
                break
        return self.created

    def lease(self):
        for idx, (bufs, evs) in enumerate(self.free):
            if evs is None or all(e.query() for e in evs):
                del self.free[idx]
                return _Lease(self, bufs)
        try:
            return _Lease(self, self._new())
        except N.torch().cuda.OutOfMemoryError:
            if not self.free:
                raise
            bufs, evs = self.free.pop(0)  # device memory is the limit: wait for the oldest set instead
            for e in evs or ():
                N.torch().cuda.current_stream().wait_event(e)
            return _Lease(self, bufs)

    def __del__(self):  # the storage outlives its last estimates
        for _bufs, evs in getattr(self, "free", []):
            try:
                for e in evs or ():
                    e.synchronize()
            except Exception:  # interpreter shutdown
                pass


class _Lease:
    def __init__(self, pool, bufs):
        self.pool = pool
        self.bufs = bufs

    def __del__(self):
        # reusable once both the dgecon estimates (condition stream) and the
        # work the caller queued on its current stream -- e.g. a solve still
        # reading these factors -- have passed this point
        try:
            t = N.torch()
            evs = (t.cuda.Event(), t.cuda.Event())
            evs[0].record(self.pool.cond_stream)
            evs[1].record(t.cuda.current_stream())
            self.pool.free.append((self.bufs, evs))
        except Exception:  # interpreter shutdown: let the tensors go
            pass


_FACTOR_BUFS = (N.BUF_THETA, N.BUF_LEAF_LU, N.BUF_LEAF_PIV, N.BUF_PHI, N.BUF_Z_LU, N.BUF_Z_PIV,
                N.BUF_PUSH, N.BUF_STATS)


def factorize(op, lam, threads=1, with_cond=True):
    """Factor Ktilde + lam I bottom-up (solver.py:111-186).  ``threads`` is
    accepted for API parity (each level is one GPU batch)."""
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    lay = op.layout
    ta = time.perf_counter()
    if getattr(op, "_factor_pool", None) is None:
        op._factor_pool = FactorStorage(lay, op.plan.cond_stream)
    lease = op._factor_pool.lease()
    bufs = lease.bufs
    bad = ctypes.c_int64(-1)
    t0 = time.perf_counter()
    rc = N.fn("hks_factorize")(op.plan.handle, op.buffers(bufs), float(lam), int(bool(with_cond)),
                               ctypes.byref(bad), N.stream_ptr())
    elapsed = time.perf_counter() - t0
    if _HOST_TRACE:
        import sys
        print(f"HKS_HOST py alloc {(t0 - ta) * 1e6:.0f} us, hks_factorize {elapsed * 1e6:.0f} us", file=sys.stderr)
    if rc == N.HKS_ERR_SINGULAR:
        raise SingularMatrixError(N.last_error())
    if rc == N.HKS_ERR_REDUCED_SINGULAR:
        raise FactorizationError(N.last_error())
    if rc != N.HKS_OK:
        raise N.HksError(rc, N.last_error())
    depth = op.tree.depth
    ms = np.zeros(depth + 1)
    N.call("hks_factor_level_ms", op.plan.handle, ms.ctypes.data_as(N._DP))
    level_seconds = {lev: float(ms[lev]) * 1e-3 for lev in range(depth + 1)}  # device time per level
    fac = Factorization(op, float(lam), bufs, level_seconds)
    fac._lease = lease  # the storage returns to the operator's pool with the Factorization
    return fac


def solve_device(f, B):
    """(k, n) column-major device block of tree-ordered right-hand sides ->
    (k, n) solutions (hks_solve; no host traffic)."""
    t = N.torch()
    X = t.empty_like(B)
    N.call("hks_solve", f.op.plan.handle, f.buffers(), N.ptr(B), N.ptr(X), B.shape[0], N.stream_ptr())
    return X


def _solve_block(f, b, in_tree_order):
    """Host (numpy or torch) or device right-hand sides -> solutions of the
    same kind.  Host blocks travel as one H2D copy in and one D2H copy into
    pinned memory out; the tree-order permutation and the (n, k) <-> (k, n)
    transposes run on the device."""
    t = N.torch()
    host_tensor = isinstance(b, t.Tensor) and not b.is_cuda
    if host_tensor:  # e.g. a pinned host block: asynchronous H2D, host result
        b = b.to(device=N.device(), dtype=t.float64, non_blocking=True)
    dev = isinstance(b, t.Tensor) and b.is_cuda
    vec = b.dim() == 1 if dev else np.ndim(b) == 1
    if dev:
        B = b.to(t.float64).reshape(b.shape[0], -1)
    else:
        B = N.to_device(np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(np.shape(b)[0], -1)))
    if not in_tree_order:
        B = B[f.tree.device_perm()]
    X = solve_device(f, B.t().contiguous())
    if not in_tree_order:
        out = t.empty_like(X)
        out[:, f.tree.device_perm()] = X
        X = out
    if dev and not host_tensor:
        return X[0] if vec else X.t()
    Xn = X.t().contiguous()  # (n, k) on the device, then one copy into pinned host memory
    xh = t.empty(Xn.shape, dtype=t.float64, pin_memory=True)
    xh.copy_(Xn, non_blocking=True)
    t.cuda.current_stream().synchronize()
    if host_tensor:
        return xh[:, 0] if vec else xh
    x = xh.numpy()
    return x[:, 0] if vec else x


def solve(f, b, in_tree_order=False):
    """x with (Ktilde + lam I) x = b (solver.py:189-259)."""
    t = N.torch()
    n = f.tree.n
    shape = tuple(b.shape) if isinstance(b, t.Tensor) else np.shape(b)
    if shape != (n,):
        raise ValueError(f"right-hand side must have length {n}")
    return _solve_block(f, b, in_tree_order)


def solve_multi(f, b, in_tree_order=False):
    """All k columns in one batched up/down sweep; each column equals the
    single-RHS solve bit for bit (solver.py:262-270)."""
    t = N.torch()
    nd = b.dim() if isinstance(b, t.Tensor) else np.ndim(b)
    if nd != 2:
        raise ValueError("expected an (n, k) right-hand side block")
    if b.shape[0] != f.tree.n:
        raise ValueError(f"right-hand side must have {f.tree.n} rows")
    return _solve_block(f, b, in_tree_order)
