"""Kernel-summation consumers beyond the factorization: KRR prediction
(cli.py:359-422, ``_cross_predict``) and the GPU-scale sampled-row error
report (the dense ``oracle.error_report`` of
oracle.py:68-140 is limited to n <= 8192).

Both are one ``hks_cross_sum``: K(queries, sources) W with K never
materialised, the sources split into column chunks across the GPU and the
partial sums added in a fixed order.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Callable

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


# --------------------------------------------------------------------------
# Scaling benchmark (oracle.py:147-232 of the reference)
# --------------------------------------------------------------------------

DENSE_MAX_POINTS = 8192


@dataclass(frozen=True)
class BenchmarkPipeline:
    """The fast-path stages a scaling benchmark times (oracle.py:147-155):
    build(PointSet) -> tree, skeletonize(tree) -> skeletons,
    assemble(tree, skeletons) -> operator, factorize(operator) ->
    factorization, solve(factorization, b) -> x."""

    build: Callable
    skeletonize: Callable
    assemble: Callable
    factorize: Callable
    solve: Callable


def _median_time(fn, repeats, warmup=False):
    """Median wall time of `fn` over `repeats` calls (oracle.py:158-167),
    with the device drained on both sides of every call so asynchronous
    GPU work is inside the interval it belongs to."""
    sync = N.torch().cuda.synchronize
    times, result = [], None
    if warmup:
        fn()
    for _ in range(repeats):
        sync()
        t0 = time.perf_counter()
        result = fn()
        sync()
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), result


def fit_exponent(sizes, seconds):
    """Slope p of the least-squares line log t = p log n + c (the scaling
    exponent the reference fits, oracle.py:170-174), in closed form:
    cov(log n, log t) / var(log n)."""
    ln = np.log(np.asarray(sizes, dtype=np.float64))
    lt = np.log(np.asarray(seconds, dtype=np.float64))
    dn = ln - ln.mean()
    return float(np.dot(dn, lt - lt.mean()) / np.dot(dn, dn))


def dense_kernel_matrix(kernel, ps, lam):
    """K(X, X) + lam I as a host array, evaluated on the GPU (oracle.py:27-33;
    same n <= 8192 limit and message)."""
    if ps.n > DENSE_MAX_POINTS:
        raise ValueError(f"dense oracle is limited to n <= {DENSE_MAX_POINTS}")
    from .kernels import eval_block
    out = eval_block(kernel, ps.coords, ps.coords)
    out[np.diag_indices(ps.n)] += lam
    return out


# Stage table of the fast-path sweep: (report key, repeats, warm-up call
# first).  Each stage consumes the previous stage's product (oracle.py:
# 192-205: build, skeletonize and assemble timed once, factorize 3 times,
# solve `solve_repeats` times after one warm-up call).
_FAST_STAGES = (("build", 1, False), ("skeletonize", 1, False), ("assemble", 1, False),
                ("factorize", 3, False), ("solve", None, True))
_DENSE_STAGES = ("dense_assemble", "dense_factor", "dense_solve")


def _fast_sweep(sizes, cfg, seed, pipeline, solve_repeats):
    from . import data
    table = {key: [] for key, _, _ in _FAST_STAGES}
    for n in sizes:
        ps = data.generate(cfg.shape, n, seed, d=cfg.d)
        rhs = np.random.default_rng([int(seed), 23, int(n)]).standard_normal(n)  # oracle.py:203
        calls = {
            "build": lambda st: pipeline.build(ps),
            "skeletonize": lambda st: pipeline.skeletonize(st["build"]),
            "assemble": lambda st: pipeline.assemble(st["build"], st["skeletonize"]),
            "factorize": lambda st: pipeline.factorize(st["assemble"]),
            "solve": lambda st: pipeline.solve(st["factorize"], rhs),
        }
        state = {}
        for key, reps, warm in _FAST_STAGES:
            t, state[key] = _median_time(lambda: calls[key](state), reps or solve_repeats, warmup=warm)
            table[key].append(t)
    return table


def _dense_sweep(dense_sizes, cfg, seed, solve_repeats):
    from . import data
    from .linalg import factor_dense, solve_dense
    lam = cfg.kernel.regularization
    table = {key: [] for key in _DENSE_STAGES}
    for n in dense_sizes:
        ps = data.generate(cfg.shape, n, seed, d=cfg.d)
        rhs = np.random.default_rng([int(seed), 29, int(n)]).standard_normal(n)  # oracle.py:216
        t_a, a = _median_time(lambda: dense_kernel_matrix(cfg.kernel, ps, lam), solve_repeats)
        t_f, fd = _median_time(lambda: factor_dense(a), solve_repeats)
        t_s, _ = _median_time(lambda: solve_dense(fd, rhs), solve_repeats)
        for key, t in zip(_DENSE_STAGES, (t_a, t_f, t_s)):
            table[key].append(t)
    return table


def scaling_benchmark(sizes, cfg, seed, pipeline=None, dense_sizes=None, solve_repeats=5):
    """Per-stage wall times of the injected fast path over `sizes` and of the
    dense factor + solve contrast over `dense_sizes`, each with its fitted
    log-log exponent.  Same contract as oracle.py:177-232 (report keys
    sizes / timings / exponents / dense_sizes, RNG streams, repeat counts,
    "fast-path sizes need an injected pipeline"); `cfg` provides `shape`,
    `d` and `kernel` (lambda = kernel.regularization).  Unlike the CPU
    original, each timed call is bracketed by device synchronisation."""
    sizes = [int(n) for n in (sizes or [])]
    report = {"sizes": sizes, "timings": {}, "exponents": {}}
    sweeps = []
    if sizes:
        if pipeline is None:
            raise ValueError("fast-path sizes need an injected pipeline")
        sweeps.append((sizes, _fast_sweep(sizes, cfg, seed, pipeline, solve_repeats)))
    if dense_sizes:
        report["dense_sizes"] = [int(n) for n in dense_sizes]
        sweeps.append((report["dense_sizes"], _dense_sweep(dense_sizes, cfg, seed, solve_repeats)))
    for ns, table in sweeps:
        for key, ts in table.items():
            report["timings"][key] = [float(t) for t in ts]
            report["exponents"][key] = fit_exponent(ns, ts)
    return report
