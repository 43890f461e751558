"""Approximate kNN (tree.knn_approx): random-projection-tree leaves + merge,
checked against the exact search (knn_bruteforce, itself bit-exact with the
reference, tests/test_gpu_pipeline.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _points(n, d, seed):
    rng = np.random.default_rng([seed, 0])
    c = rng.standard_normal((6, d)) * 2.0
    return c[rng.integers(0, 6, n)] + rng.standard_normal((n, d))


def test_single_leaf_is_exact():
    import paper_1701_02324_b200 as hk
    x = _points(3000, 5, 1)
    ps = hk.PointSet(x)
    assert np.array_equal(np.asarray(hk.knn_approx(ps, 12, trees=1, leaf_size=4000)),
                          np.asarray(hk.knn_bruteforce(ps, 12)))


def test_recall_order_and_distinctness():
    import paper_1701_02324_b200 as hk
    x = _points(40000, 6, 2)
    ps = hk.PointSet(x)
    k = 16
    ex = np.asarray(hk.knn_bruteforce(ps, k))
    ap = np.asarray(hk.knn_approx(ps, k, trees=8, leaf_size=512, seed=3))
    assert ap.shape == ex.shape
    rows = np.arange(ap.shape[0])[:, None]
    assert not np.any(ap == rows)  # self excluded
    s = np.sort(ap, axis=1)
    assert not np.any(s[:, 1:] == s[:, :-1])  # no duplicate neighbours
    recall = np.mean([len(np.intersect1d(a, e)) / k for a, e in zip(ap, ex)])
    assert recall > 0.9, recall
    # every row is ranked as the exact search ranks it: (d^2, index) order
    d2 = ((x[ap] - x[:, None, :]) ** 2).sum(-1)
    assert np.all(np.diff(d2, axis=1) >= -1e-9 * (1 + d2[:, 1:]))
    # more trees never lose a neighbour the exact search ranks first
    ap16 = np.asarray(hk.knn_approx(ps, k, trees=16, leaf_size=512, seed=3))
    rec16 = np.mean([len(np.intersect1d(a, e)) / k for a, e in zip(ap16, ex)])
    assert rec16 >= recall - 1e-12


def test_approx_knn_feeds_the_solver():
    """knn_augmented skeletons from approximate lists: the solver's residual
    against its own Ktilde stays at roundoff (the lists only steer row
    sampling)."""
    import paper_1701_02324_b200 as hk
    x = _points(8192, 5, 4)
    tree = hk.build_tree(hk.PointSet(x), 256, seed=0)
    knn = hk.knn_approx(tree.points, 16, trees=4, leaf_size=512)
    kern = hk.KernelSpec("gaussian", h=1.0, regularization=1e-2)
    cfg = hk.SkeletonConfig(tau=1e-300, max_rank=48, samples=192, sample_mode="knn_augmented", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, 1e-2)
    b = np.random.default_rng(5).standard_normal(tree.n)
    xs = hk.solve(f, b, in_tree_order=True)
    r = hk.hmatvec(op, xs, 1e-2) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-8
