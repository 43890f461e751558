"""Cached leaf blocks (hks_plan_cache_leaves; the reference's build_operator
keeps leaf_blocks too, treecode.py:48-51) against the re-evaluating path
(HKS_LEAF_CACHE=0: eval into the LU storage, fused kernel summation in the
hmatvec): same factors, solutions and matvecs to roundoff, and the
leaf_blocks view returns the values both paths use."""

import numpy as np
import pytest

from oracle import hks_oracle as O

pytestmark = pytest.mark.gpu


def _pipe(monkeypatch, cache, d=6, n=3000, lam=1e-2):
    import paper_1701_02324_b200 as hk
    monkeypatch.setenv("HKS_LEAF_CACHE", "1" if cache else "0")
    x = np.random.default_rng([7, d]).standard_normal((n, d))
    tree = hk.build_tree(hk.PointSet(x), 256, seed=0)
    knn = hk.knn_bruteforce(tree.points, 8)
    kern = hk.KernelSpec("gaussian", h=1.2, regularization=lam)
    cfg = hk.SkeletonConfig(tau=1e-7, max_rank=48, samples=192, sample_mode="knn_augmented", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, sk, kern)
    assert op.leaf_cache == cache
    f = hk.factorize(op, lam)
    b = np.random.default_rng([7, 1]).standard_normal((n, 3))
    xs = hk.solve_multi(f, b, in_tree_order=True)
    u = hk.hmatvec(op, b[:, 0], lam)
    return hk, tree, op, f, xs, u


@pytest.mark.parametrize("d", [6, 96])
def test_cached_leaf_blocks_match_reevaluation(monkeypatch, d):
    hk, tree, op1, f1, x1, u1 = _pipe(monkeypatch, True, d=d)
    _, _, op0, f0, x0, u0 = _pipe(monkeypatch, False, d=d)
    assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)
    assert np.linalg.norm(u1 - u0) <= 1e-13 * np.linalg.norm(u0)
    leaf = (1 << tree.depth) - 1
    assert np.array_equal(op1.leaf_blocks[leaf], op0.leaf_blocks[leaf])  # same kernel evaluation either way
    lu1, lu0 = f1.factors[leaf].diag_lu, f0.factors[leaf].diag_lu
    assert np.array_equal(lu1.piv, lu0.piv) and np.array_equal(lu1.lu, lu0.lu)  # K + lam I bit for bit
    xt = np.asarray(tree.points.coords)
    nd = tree.nodes[leaf]
    ref = O.kernel_block("gaussian", xt[nd.begin:nd.end], xt[nd.begin:nd.end], h=1.2)
    assert np.allclose(op1.leaf_blocks[leaf], ref, rtol=1e-13, atol=1e-15)


def test_cache_after_first_use_is_refused(monkeypatch):
    from paper_1701_02324_b200 import _native as N
    hk, tree, op, f, xs, u = _pipe(monkeypatch, False)
    with pytest.raises(N.HksError, match="already built"):
        N.call("hks_plan_cache_leaves", op.plan.handle, N.stream_ptr())
