"""GEMM-form distances on the FP64 tensor path (eval.cu: eval_mma_kernel,
ksum_mma_kernel; d >= 64): d^2 = |x|^2 + |y|^2 - 2 x.y with the dot-product
tiles on DMMA.884.  Checked against the oracle's diff-form kernel blocks
(kernels.py:56-105) within the GEMM-form roundoff (eps (|x|^2 + |y|^2) in
d^2), and for the diff form's exact properties: K(X, X) symmetric bit for
bit with an exact unit diagonal, K(X, Y) == K(Y, X)^T."""

import numpy as np
import pytest

from oracle import hks_oracle as O

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


def _tol(ref, x, y, h, d):
    nn = (x * x).sum(1)[:, None] + (y * y).sum(1)[None, :]
    return 8 * np.spacing(np.abs(ref)) + np.abs(ref) * 4 * np.sqrt(d) * EPS * nn / (2 * h * h) + 1e-300


@pytest.mark.parametrize("d", [64, 100, 784])
def test_eval_gemm_form_vs_oracle(d):
    import paper_1701_02324_b200 as hk
    rng = np.random.default_rng(d)
    x = rng.random((133, d)) / np.sqrt(d / 4)
    y = rng.random((70, d)) / np.sqrt(d / 4)
    kern = hk.KernelSpec("gaussian", h=0.8)
    got = hk.eval_block(kern, x, y)
    ref = O.kernel_block("gaussian", x, y, h=0.8)
    assert np.all(np.abs(got - ref) <= _tol(ref, x, y, 0.8, d))
    assert np.array_equal(got, hk.eval_block(kern, y, x).T)
    kk = hk.eval_block(kern, x, x)
    assert np.array_equal(kk, kk.T) and np.all(np.diag(kk) == 1.0)
    assert np.all(np.abs(kk - O.kernel_block("gaussian", x, x, h=0.8)) <= _tol(kk, x, x, 0.8, d))


def test_eval_gemm_form_polynomial():
    import paper_1701_02324_b200 as hk
    rng = np.random.default_rng(5)
    x, y = rng.random((90, 96)) * 0.1, rng.random((65, 96)) * 0.1
    kern = hk.KernelSpec("polynomial", degree=3, shift=0.5)
    got = hk.eval_block(kern, x, y)
    ref = O.kernel_block("polynomial", x, y, degree=3, shift=0.5)
    assert np.allclose(got, ref, rtol=1e-13, atol=0)


def test_leaf_block_exact_symmetry_784():
    """The factorization's leaf blocks K_aa + lam I at d = 784 (C5's
    dimension): exactly symmetric, diagonal exactly 1 + lam."""
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import workloads as W
    w = W.CONFIGS["C5"].scaled(1024)
    x = W.points(w, 0)
    tree = hk.build_tree(hk.PointSet(x), 512, seed=0)
    blk = hk.eval_block(hk.KernelSpec("gaussian", h=1.0), tree.points.coords[:512], tree.points.coords[:512])
    assert np.array_equal(blk, blk.T) and np.all(np.diag(blk) == 1.0)
    ref = O.kernel_block("gaussian", tree.points.coords[:512], tree.points.coords[:512], h=1.0)
    xs = np.asarray(tree.points.coords[:512])
    assert np.all(np.abs(blk - ref) <= _tol(ref, xs, xs, 1.0, 784))


@pytest.mark.parametrize("k", [1, 8, 20])
def test_ksum_gemm_form_vs_dense(k):
    """hks_cross_sum (ksum_mma_kernel) at d = 784 against the oracle's dense
    K @ W, with more source columns than one tile and a ragged last tile."""
    from paper_1701_02324_b200 import metrics as M
    import paper_1701_02324_b200 as hk
    import torch
    rng = np.random.default_rng(k)
    xq = rng.random((150, 784))
    xq /= np.linalg.norm(xq, axis=1)[:, None]
    xs = rng.random((301, 784))
    xs /= np.linalg.norm(xs, axis=1)[:, None]
    W = rng.standard_normal((k, 301))
    kern = hk.KernelSpec("gaussian", h=1.0)
    U = M.cross_sum(kern, torch.from_numpy(xq).cuda(), torch.from_numpy(xs).cuda(), torch.from_numpy(W).cuda())
    ref = O.kernel_block("gaussian", xq, xs, h=1.0) @ W.T
    got = U.cpu().numpy().T
    assert np.allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max() + 1e-300)
