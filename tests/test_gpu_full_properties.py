"""Parity at the benchmarked size through size-independent properties.

The reference cannot run C3 (its kNN refuses more than 65536 points and its
dense oracle more than 8192), so at N = 1,048,576 the GPU path is checked
against what every correct implementation of solver.py:111-270 /
treecode.py:65-128 / tree.py:87-188 must satisfy, on the bench's own
instance (paper_1701_02324_b200.workloads, seed 0):

* the tree permutation is a permutation and every leaf holds leaf_size points;
* kNN lists: no self, no duplicates, distances ascending -- recomputed in
  float64 on the host for sampled rows -- and the k-th neighbour is no farther
  than any sampled non-neighbour (exactness on a sample);
* every skeleton is a subset of its candidates (the node's own points for a
  leaf, the children's skeletons above) with rank <= max_rank;
* solve -> hmatvec round trip: (lam I + Ktilde) solve(b) = b to the residual
  the bench reports (1e-5 here; the measured value is 6e-7, section 5 of
  DESIGN.md explains its growth with N);
* linearity: solve(a b1 + c b2) = a solve(b1) + c solve(b2);
* solve_multi columns equal the single-RHS solves bit for bit
  (solver.py:262-270) at full size;
* Ktilde is symmetric: <u, Ktilde v> = <Ktilde u, v> (treecode.py:76-127
  uses one coupling block for both directions)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_STATE = {}


def _c3():
    if _STATE:
        return _STATE
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import workloads as W
    w = W.CONFIGS["C3"]
    x = W.points(w, 0)
    kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, w.lam)
    _STATE.update(hk=hk, w=w, x=x, tree=tree, knn=np.asarray(knn), sk=sk, op=op, f=f)
    return _STATE


def test_c3_tree_and_knn_structure():
    s = _c3()
    w, tree, knn = s["w"], s["tree"], s["knn"]
    n = w.n
    perm = np.asarray(tree.perm)
    assert perm.shape == (n,) and np.array_equal(np.sort(perm), np.arange(n))
    sizes = np.asarray(tree._end) - np.asarray(tree._begin)
    first_leaf = (1 << tree.depth) - 1
    assert np.all(sizes[first_leaf:] == w.leaf_size)
    xs = np.asarray(tree.points.coords)  # tree order: kNN indices refer to it
    assert np.array_equal(xs[:1024], s["x"][perm[:1024]])
    assert knn.shape == (n, w.kappa) and knn.min() >= 0 and knn.max() < n
    rng = np.random.default_rng(7)
    rows = rng.choice(n, size=256, replace=False)
    probe = rng.choice(n, size=4096, replace=False)
    for q in rows:
        nb = knn[q]
        assert q not in nb and np.unique(nb).size == w.kappa
        d2 = ((xs[nb] - xs[q]) ** 2).sum(axis=1)
        assert np.all(np.diff(d2) >= -1e-12 * d2.max())
        other = probe[(probe != q) & ~np.isin(probe, nb)]
        d2o = ((xs[other] - xs[q]) ** 2).sum(axis=1)
        assert d2o.min() >= d2[-1] * (1 - 1e-12)


def test_c3_skeletons_nested():
    s = _c3()
    w, tree, sk = s["w"], s["tree"], s["sk"]
    ranks = np.asarray(sk.ranks)
    assert ranks[1:].max() <= w.max_rank and ranks[1:].min() >= 1
    rng = np.random.default_rng(11)
    first_leaf = (1 << tree.depth) - 1
    nodes = list(rng.choice(np.arange(first_leaf, 2 * first_leaf + 1), size=16, replace=False))
    nodes += list(rng.choice(np.arange(1, first_leaf), size=16, replace=False))
    for i in nodes:
        i = int(i)
        idx = np.asarray(sk[i].indices)
        assert idx.size == ranks[i] and np.unique(idx).size == idx.size
        if i >= first_leaf:
            assert idx.min() >= tree._begin[i] and idx.max() < tree._end[i]
        else:
            kids = np.concatenate([np.asarray(sk[2 * i + 1].indices), np.asarray(sk[2 * i + 2].indices)])
            assert np.all(np.isin(idx, kids))


def test_c3_solve_properties():
    s = _c3()
    hk, w, op, f = s["hk"], s["w"], s["op"], s["f"]
    n = w.n
    rng = np.random.default_rng([3, 5])
    b = rng.standard_normal((n, 2))
    xm = hk.solve_multi(f, b, in_tree_order=True)
    # round trip through the treecode matvec
    for j in range(2):
        u = hk.hmatvec(op, xm[:, j], w.lam)
        assert np.linalg.norm(u - b[:, j]) <= 1e-5 * np.linalg.norm(b[:, j])
    # columns of the batched solve == single solves, bit for bit
    x0 = hk.solve(f, b[:, 0], in_tree_order=True)
    assert np.array_equal(x0, xm[:, 0])
    # linearity
    a, c = 0.75, -1.5
    xl = hk.solve(f, a * b[:, 0] + c * b[:, 1], in_tree_order=True)
    ref = a * xm[:, 0] + c * xm[:, 1]
    assert np.linalg.norm(xl - ref) <= 1e-6 * np.linalg.norm(ref)


def test_c3_ktilde_symmetric():
    s = _c3()
    hk, w, op = s["hk"], s["w"], s["op"]
    rng = np.random.default_rng([2, 9])
    u, v = rng.standard_normal(w.n), rng.standard_normal(w.n)
    ku, kv = hk.hmatvec(op, u, 0.0), hk.hmatvec(op, v, 0.0)
    lhs, rhs = float(u @ kv), float(ku @ v)
    assert abs(lhs - rhs) <= 1e-9 * (np.linalg.norm(u) * np.linalg.norm(kv))
