"""Kernel-summation consumers (paper_1701_02324_b200/metrics.py): KRR
prediction (cli.py:415-422 _cross_predict) and the sampled-row error report,
checked against the CPU oracle's dense kernel rows (oracle/hks_oracle.py)."""

import numpy as np
import pytest

from oracle import hks_oracle as O

pytestmark = pytest.mark.gpu


def test_cross_predict_matches_dense_rows():
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import metrics as M
    rng = np.random.default_rng([11, 0])
    train = rng.random((5003, 6))
    test = rng.random((301, 6))
    w = rng.standard_normal(5003)
    kern = hk.KernelSpec("gaussian", h=0.4, regularization=0.0)
    got = M.cross_predict(kern, test, train, w)
    ref = O.kernel_block("gaussian", test, train, h=0.4) @ w
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    # deterministic: the chunked partial sums are added in a fixed order
    assert np.array_equal(got, M.cross_predict(kern, test, train, w))
    # polynomial family, more queries than one row tile, several columns
    kp = hk.KernelSpec("polynomial", degree=2, shift=1.0, regularization=0.0)
    W = rng.standard_normal((3, 5003))
    t = __import__("torch")
    U = M.cross_sum(kp, t.from_numpy(test).cuda(), t.from_numpy(train).cuda(), t.from_numpy(W).cuda())
    refp = O.kernel_block("polynomial", test, train, degree=2, shift=1.0) @ W.T
    np.testing.assert_allclose(U.cpu().numpy().T, refp, rtol=1e-13, atol=1e-11 * np.abs(refp).max())


def test_cross_predict_rejects_bad_lengths():
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import metrics as M
    kern = hk.KernelSpec("gaussian", h=0.4, regularization=0.0)
    with pytest.raises(ValueError):
        M.cross_predict(kern, np.zeros((3, 2)), np.zeros((10, 2)), np.zeros(9))


def test_sampled_error_report_matches_oracle():
    """GPU metrics on sampled rows vs the same quantities from dense oracle
    rows of K, for the C2 generator at n = 8192."""
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import metrics as M
    from paper_1701_02324_b200 import workloads as W
    w = W.CONFIGS["C2"].scaled(8192)
    x = W.points(w, 0)
    kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, w.lam)
    b = np.random.default_rng([0, 5]).standard_normal(tree.n)
    rep = M.sampled_error_report(op, f, b=b, rows=256, seed=3)
    # the same metrics from dense oracle rows
    xt = np.asarray(tree.points.coords)
    R = M.sample_rows(tree.n, 256, 3)
    KR = O.kernel_block("gaussian", xt[R], xt, h=w.h)
    wv = np.random.default_rng([3, 78]).standard_normal(tree.n)
    kw = KR @ wv
    ktw = hk.hmatvec(op, wv, 0.0)[R]
    xs = hk.solve(f, b, in_tree_order=True)
    res = KR @ xs + w.lam * xs[R] - b[R]
    assert rep["rows"] == 256
    assert rep["matvec_relerr_vs_K"] == pytest.approx(np.linalg.norm(ktw - kw) / np.linalg.norm(kw), rel=1e-9)
    assert rep["true_residual"] == pytest.approx(np.linalg.norm(res) / np.linalg.norm(b[R]), rel=1e-7)
    assert rep["residual_vs_Ktilde"] < 1e-9
    # the configuration's approximation error (0.185 at N = 16384) is O(0.1), not roundoff
    assert 0.01 < rep["matvec_relerr_vs_K"] < 1.0
