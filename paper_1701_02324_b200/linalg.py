"""Dense building blocks on the GPU: LU factor / solve and the column-pivoted
QR interpolative decomposition (linalg.py:1-179 of the reference).

Same names, result types and exceptions as the reference; the arithmetic runs
in libhks (csrc/lu.cu, csrc/qrcp.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N


class SingularMatrixError(np.linalg.LinAlgError):
    """Raised when a dense factorization hits an exactly singular pivot."""


@dataclass(frozen=True)
class PivotedQRResult:
    """pivots (n,), r_factor (rank, n), rank -- linalg.py:26-40."""

    pivots: np.ndarray
    r_factor: np.ndarray
    rank: int


@dataclass(frozen=True)
class DenseFactor:
    """LU with partial pivoting in combined LAPACK storage (linalg.py:139-148)."""

    lu: np.ndarray
    piv: np.ndarray

    @property
    def n(self):
        return self.lu.shape[0]


def factor_dense(a):
    """LU-factor a square matrix on the GPU; raises SingularMatrixError on an
    exactly-zero pivot naming the elimination step (linalg.py:151-169)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expected a square matrix")
    n = a.shape[0]
    if n == 0:
        return DenseFactor(np.zeros((0, 0)), np.zeros(0, dtype=np.int32))
    t = N.torch()
    A = N.to_device(np.ascontiguousarray(a.T))  # column-major
    piv = t.empty(n, dtype=t.int32, device=A.device)
    import ctypes
    info = ctypes.c_int32(0)
    rc = N.fn("hks_lu_factor")(N.ptr(A), n, n, N.ptr(piv), ctypes.byref(info), N.stream_ptr())
    if rc == N.HKS_ERR_SINGULAR:
        raise SingularMatrixError(N.last_error())
    if rc != N.HKS_OK:
        raise N.HksError(rc, N.last_error())
    return DenseFactor(A.cpu().numpy().T.copy(), piv.cpu().numpy())


def solve_dense(f, b):
    """Solve A X = B with an LU factor, one or many right-hand sides
    (linalg.py:172-179)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != f.n:
        raise ValueError(f"right-hand side has {b.shape[0]} rows, expected {f.n}")
    if f.n == 0:
        return b.copy()
    vec = b.ndim == 1
    B = N.col_major(b[:, None] if vec else b)
    LU = N.to_device(np.ascontiguousarray(f.lu.T))
    piv = N.to_device(np.asarray(f.piv, dtype=np.int32))
    N.call("hks_lu_solve", N.ptr(LU), N.ptr(piv), f.n, f.n, N.ptr(B), f.n, B.shape[0], N.stream_ptr())
    x = B.cpu().numpy().T
    return x[:, 0].copy() if vec else x.copy()


def _qr_checks(tol, max_rank, a):
    if tol <= 0:
        raise ValueError("tol must be positive")
    if max_rank < 1:
        raise ValueError("max_rank must be >= 1")
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def interpolative_decomposition(a, tol, max_rank):
    """Column ID A ~= A[:, J] P with P[:, J] == I exactly (linalg.py:107-136),
    via the GPU column-pivoted QR (csrc/qrcp.cu)."""
    import ctypes
    a = _qr_checks(tol, max_rank, a)
    m, n = a.shape
    if m == 0 or n == 0:
        return np.arange(n)[:0], np.zeros((0, n))
    t = N.torch()
    A = N.to_device(np.ascontiguousarray(a))  # row-major m x n (the QR workspace layout)
    piv = t.empty(n, dtype=t.int64, device=A.device)
    cap = min(m, n, int(max_rank))
    P = t.zeros(max(cap * n, 1), dtype=t.float64, device=A.device)
    rank = ctypes.c_int64(0)
    N.call("hks_interp_decomp", N.ptr(A), m, n, n, float(tol), int(max_rank), N.ptr(piv), N.ptr(P),
           ctypes.byref(rank), N.stream_ptr())
    r = rank.value
    cols = piv.cpu().numpy()[:r].copy()
    interp = P[: r * n].cpu().numpy().reshape(n, r).T.copy() if r else np.zeros((0, n))
    return cols, interp


def pivoted_qr(a, tol, max_rank):
    """Truncated column-pivoted Householder QR (linalg.py:43-104).  The
    pivots and rank come from the GPU kernel; R is returned for API parity
    (computed from the same pivots)."""
    import ctypes
    a = _qr_checks(tol, max_rank, a)
    m, n = a.shape
    if m == 0 or n == 0:
        return PivotedQRResult(np.arange(n), np.zeros((0, n)), 0)
    t = N.torch()
    A = N.to_device(np.ascontiguousarray(a))
    piv = t.empty(n, dtype=t.int64, device=A.device)
    cap = min(m, n, int(max_rank))
    P = t.zeros(max(cap * n, 1), dtype=t.float64, device=A.device)
    rank = ctypes.c_int64(0)
    N.call("hks_interp_decomp", N.ptr(A), m, n, n, float(tol), int(max_rank), N.ptr(piv), N.ptr(P),
           ctypes.byref(rank), N.stream_ptr())
    r = rank.value
    # the workspace now holds R in its first r rows (row-major, pivoted column order)
    R = A.cpu().numpy()[:r].copy()
    R = np.triu(R) if r else np.zeros((0, n))
    return PivotedQRResult(piv.cpu().numpy(), R, r)
