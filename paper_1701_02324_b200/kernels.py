"""Kernel families and dense block evaluation on the GPU.

Drop-in for hikersolve.kernels (kernels.py:1-105): same KernelSpec
validation and messages; ``eval_block`` runs the sm_100a eval kernel
(csrc/eval.cu) and returns a host array like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

FAMILIES = ("gaussian", "laplace3d", "polynomial")


@dataclass(frozen=True)
class KernelSpec:
    """Kernel family + parameters + the diagonal regularization lambda
    (kernels.py:23-48).  lambda is never added by eval_block."""

    family: str = "gaussian"
    h: float = 0.5
    degree: int = 2
    shift: float = 1.0
    regularization: float = 1e-3

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown kernel family {self.family!r}")
        if self.family == "gaussian" and not self.h > 0:
            raise ValueError("gaussian bandwidth h must be positive")
        if self.family == "polynomial":
            if self.degree < 1:
                raise ValueError("polynomial degree must be >= 1")
            if self.shift < 0:
                raise ValueError("polynomial shift must be nonnegative")
        if self.regularization < 0:
            raise ValueError("regularization must be nonnegative")


def eval_system_diag_shift(kernel):
    """The configured diagonal regularization lambda (kernels.py:51-53)."""
    return kernel.regularization


def _check_dims(kernel, d_t, d_s):
    if d_t != d_s:
        raise ValueError(f"dimension mismatch: targets are {d_t}-d, sources {d_s}-d")
    if kernel.family == "laplace3d" and d_t != 3:
        raise ValueError("laplace3d kernel requires 3-d points")


def eval_block_device(kernel, X, rows=None, cols=None, row0=0, nrows=None, col0=0, ncols=None,
                      row_major=False, diag=0.0):
    """K(X[rows], X[cols]) on the device (X: (n, d) CUDA float64 tensor in
    the same order as the indices).  Returns a CUDA tensor (nrows, ncols)."""
    t = N.torch()
    nr = int(rows.numel()) if rows is not None else int(nrows)
    nc = int(cols.numel()) if cols is not None else int(ncols)
    if row_major:
        out = t.empty((nr, nc), dtype=t.float64, device=X.device)
        ldo = nc
    else:
        out = t.empty((nc, nr), dtype=t.float64, device=X.device)  # column-major view
        ldo = nr
    if nr and nc:
        N.call("hks_eval_block", N.ptr(X), X.shape[1], N.kernel_struct(kernel), N.ptr(rows), row0, nr,
               N.ptr(cols), col0, nc, N.ptr(out), ldo, int(row_major), float(diag), N.stream_ptr())
    return out if row_major else out.t()


def eval_block(kernel, xt, xs):
    """Dense K(xt, xs), (m, n) float64, no regularization (kernels.py:64-105)."""
    xt = np.atleast_2d(np.asarray(xt, dtype=np.float64))
    xs = np.atleast_2d(np.asarray(xs, dtype=np.float64))
    _check_dims(kernel, xt.shape[1], xs.shape[1])
    m, n = xt.shape[0], xs.shape[0]
    if m == 0 or n == 0:
        return np.empty((m, n))
    if xt.shape == xs.shape and np.array_equal(xt, xs):
        # K(X, X): one copy of the points, rows and columns the same ids --
        # a point against itself is d^2 = 0 exactly on either distance path
        out = eval_block_device(kernel, N.to_device(xt), row0=0, nrows=m, col0=0, ncols=n, row_major=True)
        return out.cpu().numpy()
    X = N.to_device(np.concatenate([xt, xs], axis=0))
    out = eval_block_device(kernel, X, row0=0, nrows=m, col0=m, ncols=n, row_major=True)
    return out.cpu().numpy()
