"""Kernel-summation consumers beyond the factorization: KRR prediction
(cli.py:359-422, ``_cross_predict``) and the GPU-scale sampled-row error
report (the dense ``oracle.error_report`` of
oracle.py:68-140 is limited to n <= 8192).

Both are one ``hks_cross_sum``: K(queries, sources) W with K never
materialised, the sources split into column chunks across the GPU and the
partial sums added in a fixed order.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .data import PointSet
from .solver import solve_device
from .treecode import hmatvec_device


def cross_sum(kernel, xq, xs, W, rows=None):
    """U = K(xq[rows], xs) W on the device.  xq, xs: (n, d) float64 device
    tensors (row-major); W: (k, ns) device block (column-major ns x k);
    rows: optional device int64 indices into xq.  Returns (k, nq)."""
    t = N.torch()
    xq = xq.to(t.float64).contiguous()
    xs = xs.to(t.float64).contiguous()
    W = W.reshape(-1, xs.shape[0]).to(t.float64).contiguous()
    if xq.shape[1] != xs.shape[1]:
        raise ValueError("query and source points must have the same dimension")
    nq = int(rows.shape[0]) if rows is not None else int(xq.shape[0])
    k = int(W.shape[0])
    U = t.empty((k, nq), dtype=t.float64, device=N.device())
    kern = N.kernel_struct(kernel)
    N.call("hks_cross_sum", N.ptr(xq), int(xq.shape[0]) if rows is None else nq, N.ptr(xs), int(xs.shape[0]),
           int(xs.shape[1]), kern, N.ptr(rows) if rows is not None else None, N.ptr(W), int(xs.shape[0]), k,
           N.ptr(U), nq, 0.0, N.stream_ptr())
    return U


def cross_predict(kernel, test, train_points, w_tree):
    """KRR prediction K(test, train) w (cli.py:415-422): test a PointSet /
    array in any order, train_points the tree-ordered training PointSet,
    w_tree the weights in tree order.  Returns a host vector (or a CUDA
    tensor when w_tree is one)."""
    t = N.torch()
    test = test if isinstance(test, PointSet) else PointSet(np.asarray(test, dtype=np.float64))
    train = train_points if isinstance(train_points, PointSet) else PointSet(np.asarray(train_points))
    dev = isinstance(w_tree, t.Tensor) and w_tree.is_cuda
    w = w_tree if dev else N.to_device(np.asarray(w_tree, dtype=np.float64))
    if w.shape[0] != train.n:
        raise ValueError(f"weights must have length {train.n}")
    U = cross_sum(kernel, test.device(), train.device(), w.reshape(1, -1))[0]
    return U if dev else U.cpu().numpy()


def sample_rows(n, count=256, seed=0):
    """The sampled-row set of the accuracy metrics: default_rng([seed, 77])
    draws `count` distinct rows (sorted), BASELINE.md 4.2 definitions."""
    rng = np.random.default_rng([int(seed), 77])
    return np.sort(rng.choice(n, size=min(int(count), n), replace=False))


def sampled_error_report(op, f, b=None, rows=256, seed=0):
    """Accuracy of the compressed operator and the solve at any N, on
    sampled rows of the TRUE kernel matrix (BASELINE.md 4.2 definitions):

      matvec_relerr_vs_K   ||Ktilde w - K w||_R / ||K w||_R, w from
                           default_rng([seed, 78]) (all n entries);
      true_residual        ||(K + lam I) x - b||_R / ||b||_R for x = solve(b)
                           (b: the first column given, else default_rng([seed, 79]));
      residual_vs_Ktilde   ||(Ktilde + lam I) x - b|| / ||b|| over all rows.

    R = the sampled rows; K(R, :) v is a fused kernel summation over all n
    sources (never stored).  Everything in tree order."""
    t = N.torch()
    n = op.n
    lam = f.lam
    x_pts = op.tree.device_points()
    R = sample_rows(n, rows, seed)
    Rd = N.to_device(R.astype(np.int64))
    w = N.to_device(np.random.default_rng([int(seed), 78]).standard_normal(n)).reshape(1, -1)
    kw = cross_sum(op.kernel, x_pts, x_pts, w, rows=Rd)[0]
    ktw = hmatvec_device(op, w, 0.0)[0][Rd]
    if b is None:
        b = np.random.default_rng([int(seed), 79]).standard_normal(n)
    bd = N.to_device(np.asarray(b, dtype=np.float64)).reshape(-1, n)[:1].contiguous()
    x = solve_device(f, bd)
    kx = cross_sum(op.kernel, x_pts, x_pts, x, rows=Rd)[0] + lam * x[0][Rd]
    res_true = kx - bd[0][Rd]
    res_tilde = hmatvec_device(op, x, lam)[0] - bd[0]
    nrm = t.linalg.vector_norm
    return {
        "rows": int(R.size),
        "matvec_relerr_vs_K": float(nrm(ktw - kw) / nrm(kw)),
        "true_residual": float(nrm(res_true) / nrm(bd[0][Rd])),
        "residual_vs_Ktilde": float(nrm(res_tilde) / nrm(bd[0])),
    }
