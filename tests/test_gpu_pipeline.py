"""GPU setup stages against the reference's golden fixtures: tree
permutation and kNN lists bit-exact, skeleton index sets exact except at
pivot near-ties, then the whole device pipeline's solve / matvec."""

import numpy as np
import pytest

from golden_cases import (ALL_CASES, GOLDEN, coords_for, load, matvec_w, rhs_for, sketch_vec,
                          skel_list)

pytestmark = pytest.mark.gpu

_CACHE = {}


def pipeline(name):
    if name in _CACHE:
        return _CACHE[name]
    import paper_1701_02324_b200 as hk
    g = load(name)
    m = g["meta"]
    x = coords_for(name)
    tree = hk.build_tree(hk.PointSet(x), m["leaf"], seed=m["seed"])
    knn = hk.knn_bruteforce(tree.points, m["kappa"]) if m["mode"] == "knn_augmented" else None
    cfg = hk.SkeletonConfig(tau=m["tau"], max_rank=m["max_rank"], samples=m["samples"],
                            sample_mode=m["mode"], seed=m["seed"])
    kern = hk.KernelSpec(m["family"], h=m["h"], degree=m["degree"], shift=m["shift"],
                         regularization=m["lam"])
    skels = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, skels, kern)
    f = hk.factorize(op, m["lam"])
    _CACHE[name] = (hk, g, m, tree, knn, skels, op, f)
    return _CACHE[name]


@pytest.mark.parametrize("name", ALL_CASES)
def test_tree_perm_bit_exact(name):
    hk, g, m, tree, knn, skels, op, f = pipeline(name)
    assert np.array_equal(np.asarray(tree.perm), g["perm"])
    assert tree.depth == m["depth"]
    for nd in tree.nodes:
        if not nd.is_leaf:
            ref = g["split_value"][nd.index]
            assert nd.split_value == pytest.approx(ref, rel=1e-12, abs=1e-12)
    assert np.array_equal(tree.points.coords, coords_for(name)[g["perm"]])


@pytest.mark.parametrize("name", [c for c in ALL_CASES if load(c)["meta"]["mode"] == "knn_augmented"])
def test_knn_bit_exact(name):
    hk, g, m, tree, knn, skels, op, f = pipeline(name)
    assert np.array_equal(np.asarray(knn), g["knn"])


def test_knn_small_and_ties():
    import paper_1701_02324_b200 as hk
    z = np.load(GOLDEN / "knn_n200.npz")
    assert np.array_equal(np.asarray(hk.knn_bruteforce(hk.PointSet(z["coords"]), 5)), z["knn"])
    pts = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 0.0], [0.0, 1.0], [5.0, 5.0]])
    nb = np.asarray(hk.knn_bruteforce(hk.PointSet(pts), 2))
    assert list(nb[0]) == [1, 2]  # ties go to the lower index (tests/test_tree.py:121-127)
    with pytest.raises(ValueError):
        hk.knn_bruteforce(hk.PointSet(pts), 5)


@pytest.mark.parametrize("name", ALL_CASES)
def test_skeletons_match_golden(name):
    hk, g, m, tree, knn, skels, op, f = pipeline(name)
    assert np.array_equal(skels.ranks[1:], g["ranks"][1:])
    assert np.array_equal(skels.rows_count[1:], g["rows_count"][1:])
    mismatched, loose = [], []
    at = 0
    for i in range(1, len(g["ranks"])):
        s = skels[i]
        ref = skel_list(g, i)
        if not np.array_equal(s.indices, ref):
            mismatched.append(i)
        r = s.interp.shape[0]
        sk = s.interp @ sketch_vec(77, i, s.interp.shape[1]) if r else np.zeros(0)
        refs = g["interp_sketch"][at:at + r]
        at += r
        if i not in mismatched and r and np.linalg.norm(sk - refs) > 1e-6 * max(np.linalg.norm(refs), 1.0):
            loose.append(i)
    # skeleton index sets must match except where pivots tie (north_star)
    assert not mismatched, f"skeletons differ at nodes {mismatched}"
    # the ID coefficients R11^-1 R12 are ill-determined when a fixed rank
    # exceeds the block's numerical rank (tau = 1e-300 configs at the top
    # levels): both implementations return valid IDs that differ in the
    # near-null space; allowed only at the two top levels, where the
    # downstream matvec / solve parity below is the arbiter
    assert all(i < 7 for i in loose), f"interp differs below the top levels: {loose}"


@pytest.mark.parametrize("name", ALL_CASES)
def test_pipeline_solve_and_matvec(name):
    hk, g, m, tree, knn, skels, op, f = pipeline(name)
    b = rhs_for(m)
    x = hk.solve_multi(f, b, in_tree_order=True)
    # residual against the device's own Ktilde, within 10x the residual the
    # reference's own x leaves on the same operator
    for j in range(b.shape[1]):
        bn = np.linalg.norm(b[:, j])
        res_g = np.linalg.norm(hk.hmatvec(op, x[:, j], m["lam"]) - b[:, j]) / bn
        res_o = np.linalg.norm(hk.hmatvec(op, g["x"][:, j], m["lam"]) - b[:, j]) / bn
        assert res_g <= max(10 * res_o, 1e-10), (res_g, res_o)
    ill = name in {"gauss_uniform_n2000"}
    assert np.linalg.norm(x - g["x"]) <= (5e-2 if ill else 1e-6) * np.linalg.norm(g["x"])
    u = hk.hmatvec(op, matvec_w(m), m["lam"])
    assert np.linalg.norm(u - g["u"]) <= 1e-9 * np.linalg.norm(g["u"])


def test_interpolative_decomposition_and_pivoted_qr():
    import paper_1701_02324_b200 as hk
    from oracle import hks_oracle as O
    z = np.load(GOLDEN / "id_cases.npz")
    for t in range(12):
        tol, mr = z[f"tol{t}"]
        a = z[f"a{t}"]
        cols, p = hk.interpolative_decomposition(a, tol, int(mr))
        assert np.array_equal(cols, z[f"cols{t}"]), t
        assert np.array_equal(p[:, cols], np.eye(cols.size))
        # backward-error bound of the reference's own test (tests/test_linalg.py:113-123)
        r = cols.size
        if 0 < r < int(mr):  # rank set by tau (not by the cap): the bound applies
            assert np.linalg.norm(a - a[:, cols] @ p) <= 10 * np.sqrt(a.shape[1] * r) * tol * np.linalg.norm(a) + 1e-14
        # coefficients agree to roundoff amplified by cond(R11)
        piv, rf, rank = O.qrcp(a, tol, int(mr))
        c11 = np.linalg.cond(rf[:, :rank]) if rank else 1.0
        assert np.linalg.norm(p - z[f"p{t}"]) <= 1e-14 * c11 * max(np.linalg.norm(z[f"p{t}"]), 1.0) + 1e-12
        qr = hk.pivoted_qr(a, tol, int(mr))
        assert qr.rank == rank and np.array_equal(qr.pivots, piv)
        assert np.allclose(np.abs(qr.r_factor), np.abs(rf), rtol=1e-9, atol=1e-12 * np.abs(rf).max(initial=1))


def test_skeletonize_threads_invariant_and_deterministic():
    import paper_1701_02324_b200 as hk
    x = np.random.default_rng(12).random((512, 3))
    kern = hk.KernelSpec("gaussian", h=0.3, regularization=1e-2)
    tree = hk.build_tree(hk.PointSet(x), 64, seed=0)
    cfg = hk.SkeletonConfig(tau=1e-6, max_rank=64, samples=128, sample_mode="uniform")
    a = hk.build_skeletons(tree, kern, cfg, threads=1)
    b = hk.build_skeletons(tree, kern, cfg, threads=4)
    for i in range(1, 2 ** (tree.depth + 1) - 1):
        assert np.array_equal(a[i].indices, b[i].indices)
        assert np.array_equal(a[i].interp, b[i].interp)


@pytest.mark.parametrize("k", [16, 20])
def test_solve_multi_columns_bit_identical(k):
    """solve_multi == solve column by column, bit for bit (tests/test_solver.py:174-185
    of the reference), on both GEMM paths: k <= 16 right-hand sides use the
    skinny 128 x 16 tiles, k > 16 the 64 x 64 tiles, single columns the
    skinny ones -- the k order per output element is the same in all."""
    hk, g, m, tree, knn, skels, op, f = pipeline(sorted(ALL_CASES)[0])
    B = np.random.default_rng(k).standard_normal((op.n, k))
    X = hk.solve_multi(f, B, in_tree_order=True)
    for j in (0, k // 2, k - 1):
        np.testing.assert_array_equal(X[:, j], hk.solve(f, B[:, j], in_tree_order=True))
    U = np.stack([hk.hmatvec(op, B[:, j], m["lam"]) for j in (0, k - 1)], axis=1)
    assert np.all(np.isfinite(U))
