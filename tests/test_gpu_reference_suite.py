"""The reference's known-answer suite, restated against the GPU package.

Every check below is one the reference makes of itself
(/root/reference/pkg/tests; cited per test), run here through
paper_1701_02324_b200's drop-in API on instances built the way the
reference's helpers build them (helpers.py:92-133: frozen instance =
uniform_cube d = 3, seed 3, gaussian h = 0.3, lam 1e-2, leaf 256, tau 1e-7,
max_rank 384, exact sampling).  Independent dense references (numpy) are the
judges, as in the reference; tolerances are the reference's own, except for
the five checks the reference itself fails (REF_MEASURED)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_CACHE = {}

# Five of the reference's checks fail for the unmodified reference itself in
# this container (pytest /root/reference/pkg/tests/test_solver.py
# test_skeleton.py: huge_lambda, roundtrip_2048, inverse_action_symmetric,
# offdiag_reconstruction_bound; test_treecode.py:
# solver_consistency_roundtrip).  For those the GPU path is held to the
# reference's own measured values (the same quantities computed by importing
# the unmodified reference here, numpy 2.3 / OpenBLAS) instead of the bound
# the reference misses.
REF_MEASURED = {
    "roundtrip_2048": 1.4012468159207929e-07,        # ||x - w|| / ||w||
    "inverse_action_asymmetry": 3.1381111043060628e-09,  # max over the 8 seeded pairs
    "offdiag_worst": 5.906015803805912e-05,          # worst sibling-block reconstruction error
    "huge_lambda": 6.7043572417015575e-06,           # ||x - b / lam|| / ||b / lam||
    "consistency_roundtrip": 5.916857720642211e-09,  # test_treecode.py:149-157, ||x - w|| / ||w||
}


def _instance(ps, kern, leaf=64, tau=1e-7, max_rank=256, sample_mode="exact", samples=256, seed=0, factor=True):
    import paper_1701_02324_b200 as hk
    tree = hk.build_tree(ps, leaf, seed=seed)
    sk = hk.build_skeletons(tree, kern, hk.SkeletonConfig(tau=tau, max_rank=max_rank, samples=samples,
                                                          sample_mode=sample_mode, seed=seed))
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, kern.regularization) if factor else None
    return dict(hk=hk, ps=ps, kern=kern, tree=tree, sk=sk, op=op, f=f)


def _frozen(n):  # helpers.py:113-133
    if n not in _CACHE:
        import paper_1701_02324_b200 as hk
        ps = hk.generate("uniform_cube", n, 3, d=3)
        kern = hk.KernelSpec(family="gaussian", h=0.3, regularization=1e-2)
        _CACHE[n] = _instance(ps, kern, leaf=256, tau=1e-7, max_rank=384, sample_mode="exact", seed=3)
    return _CACHE[n]


def _basis(tree, sk, node):
    """Dense telescoped interpolation operator of a node (oracle.py:49-65)."""
    s = sk[node.index]
    if node.is_leaf:
        return np.asarray(s.interp)
    left, right = tree.children(node)
    bl, br = _basis(tree, sk, left), _basis(tree, sk, right)
    stacked = np.zeros((bl.shape[0] + br.shape[0], node.end - node.begin))
    split = left.end - left.begin
    stacked[: bl.shape[0], :split] = bl
    stacked[bl.shape[0]:, split:] = br
    return np.asarray(s.interp) @ stacked


def _dense(inst):
    """K(X, X) + lam I in tree order, float64 numpy (oracle.py:27-33)."""
    x = np.asarray(inst["tree"].points.coords)
    d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
    k = np.exp(-d2 / (2.0 * inst["kern"].h ** 2))
    return k + inst["kern"].regularization * np.eye(x.shape[0])


def test_smw_identity_through_gpu_dense_solves():
    """test_solver.py:16-65: the reduced-system identity against the dense
    inverse, 2 x 100 random instances; every solve here is the GPU LU."""
    import paper_1701_02324_b200 as hk
    for zero_diag, seed in ((True, 20), (False, 21)):
        rng = np.random.default_rng(seed)
        for _ in range(100):
            sizes = rng.integers(2, 17, size=2)
            ranks = rng.integers(1, 9, size=2)
            m, r = int(sizes.sum()), int(ranks.sum())
            d = np.zeros((m, m))
            at = 0
            for s in sizes:
                mat = rng.standard_normal((s, s))
                d[at:at + s, at:at + s] = mat @ mat.T + np.eye(s)
                at += s
            u, v = rng.standard_normal((m, r)), rng.standard_normal((m, r))
            if zero_diag:
                bmat = np.zeros((r, r))
                coup = rng.standard_normal((int(ranks[0]), int(ranks[1])))
                bmat[: ranks[0], ranks[0]:] = coup
                bmat[ranks[0]:, : ranks[0]] = coup.T
            else:
                bmat = rng.standard_normal((r, r))
            rhs = rng.standard_normal(m)
            fd = hk.factor_dense(d)
            dinv_b, dinv_u = hk.solve_dense(fd, rhs), hk.solve_dense(fd, u)
            z = np.eye(r) + (v.T @ dinv_u) @ bmat
            got = dinv_b - dinv_u @ (bmat @ hk.solve_dense(hk.factor_dense(z), v.T @ dinv_b))
            expect = np.linalg.inv(d + u @ bmat @ v.T) @ rhs
            assert np.linalg.norm(got - expect) <= 1e-10 * np.linalg.norm(expect)


def test_single_leaf_matches_dense():  # test_solver.py:68-78
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 50, seed=1, d=3)
    kern = hk.KernelSpec("gaussian", h=0.4, regularization=1e-2)
    inst = _instance(ps, kern, leaf=64)
    assert len(inst["f"].factors) == 1
    b = np.random.default_rng(2).standard_normal(50)
    x = hk.solve(inst["f"], b, in_tree_order=True)
    expect = np.linalg.solve(_dense(inst), b)
    assert np.linalg.norm(x - expect) <= 1e-12 * np.linalg.norm(expect)


def test_rank_zero_decouples_to_leaf_solves():  # test_solver.py:81-93
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 128, seed=3, d=2)
    kern = hk.KernelSpec("gaussian", h=1e-9, regularization=1e-1)
    inst = _instance(ps, kern, leaf=32, tau=1e-4, max_rank=8)
    assert inst["f"].max_rank == 0
    b = np.random.default_rng(4).standard_normal(128)
    x = hk.solve(inst["f"], b, in_tree_order=True)
    for leaf in inst["tree"].leaves():
        block = np.asarray(inst["op"].leaf_blocks[leaf.index]) + 1e-1 * np.eye(leaf.size)
        expect = np.linalg.solve(block, b[leaf.begin:leaf.end])
        got = x[leaf.begin:leaf.end]
        assert np.linalg.norm(got - expect) <= 1e-12 * np.linalg.norm(expect)


def test_theta_matches_dense_projection():  # test_solver.py:96-111
    inst = _frozen(2048)
    hk, tree, sk, f = inst["hk"], inst["tree"], inst["sk"], inst["f"]
    kt = hk.materialize_ktilde(inst["op"], f.lam)
    for node in tree.nodes:
        if node.level == 0:
            continue
        basis = _basis(tree, sk, node)
        sub = kt[node.begin:node.end, node.begin:node.end]
        ref = basis @ np.linalg.inv(sub) @ basis.T
        assert np.linalg.norm(f.factors[node.index].theta - ref) <= 1e-8 * max(np.linalg.norm(ref), 1e-300)


def test_theta_symmetric():  # test_solver.py:114-120
    inst = _frozen(1024)
    for node in inst["tree"].nodes:
        if node.level == 0:
            continue
        th = inst["f"].factors[node.index].theta
        if th.size:
            assert np.linalg.norm(th - th.T) <= 1e-10 * np.linalg.norm(th)


def test_huge_lambda_diagonal_dominance():  # test_solver.py:123-130
    import paper_1701_02324_b200 as hk
    lam = 1e6
    ps = hk.generate("uniform_cube", 256, seed=5, d=3)
    kern = hk.KernelSpec("gaussian", h=0.4, regularization=lam)
    inst = _instance(ps, kern, leaf=64, tau=1e-6)
    b = np.random.default_rng(6).standard_normal(256)
    x = hk.solve(inst["f"], b, in_tree_order=True)
    # The reference asserts ||x - b / lam|| <= 2e-6 ||b / lam||; the unmodified
    # reference itself returns 6.70e-6 on this instance (measured here: its
    # own test fails), because x = b / lam - K b / lam^2 + ... deviates by
    # ||K|| / lam.  The restated check is the bound with the right constant,
    # and agreement with the dense solve.
    dense = _dense(inst)
    knorm = np.linalg.norm(dense - lam * np.eye(256), 2)
    assert np.linalg.norm(x - b / lam) <= 1.01 * knorm / lam * np.linalg.norm(b / lam)
    dev = np.linalg.norm(x - b / lam) / np.linalg.norm(b / lam)
    assert abs(dev - REF_MEASURED["huge_lambda"]) <= 1e-6 * REF_MEASURED["huge_lambda"]
    expect = np.linalg.solve(dense, b)
    assert np.linalg.norm(x - expect) <= 1e-10 * np.linalg.norm(expect)


def test_roundtrip_2048():  # test_solver.py:133-139
    inst = _frozen(2048)
    hk = inst["hk"]
    w = np.random.default_rng(7).standard_normal(2048)
    b = hk.hmatvec(inst["op"], w, inst["f"].lam)
    x = hk.solve(inst["f"], b, in_tree_order=True)
    # The reference's bound is 1e-9; the unmodified reference itself reaches
    # 1.40e-7 on this instance (REF_MEASURED below: its own test fails --
    # reduced systems of condition ~1e7 amplify roundoff).  Parity criterion:
    # within a small factor of the reference's own round-trip error.
    assert np.linalg.norm(x - w) <= 4 * REF_MEASURED["roundtrip_2048"] * np.linalg.norm(w)


def test_solve_vs_true_dense():  # test_solver.py:142-149
    inst = _frozen(1024)
    b = np.random.default_rng(8).standard_normal(1024)
    x = inst["hk"].solve(inst["f"], b, in_tree_order=True)
    expect = np.linalg.solve(_dense(inst), b)
    assert np.linalg.norm(x - expect) <= 1e-4 * np.linalg.norm(expect)


def test_inverse_action_symmetric():  # test_solver.py:152-163
    inst = _frozen(1024)
    hk, n = inst["hk"], inst["tree"].n
    rng = np.random.default_rng(9)
    for _ in range(8):
        i, j = rng.integers(0, n, size=2)
        ei, ej = np.zeros(n), np.zeros(n)
        ei[i] = ej[j] = 1.0
        xj = hk.solve(inst["f"], ej, in_tree_order=True)
        xi = hk.solve(inst["f"], ei, in_tree_order=True)
        # reference bound 1e-9; the reference's own worst pair is 3.14e-9 (REF_MEASURED)
        assert abs(ei @ xj - ej @ xi) <= 2 * REF_MEASURED["inverse_action_asymmetry"]


def test_input_order_and_multi_and_validation():  # test_solver.py:166-204, 215-218
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 256, 11, d=3)
    kern = hk.KernelSpec("gaussian", h=0.3, regularization=1e-1)
    inst = _instance(ps, kern, leaf=64, tau=1e-10, max_rank=256, seed=11)
    f = inst["f"]
    rng = np.random.default_rng(10)
    b = rng.standard_normal(256)
    perm = np.asarray(inst["tree"].perm)
    assert np.array_equal(hk.solve(f, b, in_tree_order=False)[perm], hk.solve(f, b[perm], in_tree_order=True))
    block = np.random.default_rng(11).standard_normal((256, 4))
    got = hk.solve_multi(f, block, in_tree_order=True)
    for j in range(4):
        assert np.array_equal(got[:, j], hk.solve(f, block[:, j], in_tree_order=True))
    assert np.all(hk.solve_multi(f, np.zeros((256, 3)), in_tree_order=True) == 0.0)
    with pytest.raises(ValueError):
        hk.solve_multi(f, np.zeros(256))
    assert f.lam == 1e-1
    with pytest.raises(ValueError):
        hk.factorize(inst["op"], -1.0)
    with pytest.raises(ValueError):
        hk.solve(f, np.zeros(5))


def test_build_stats_populated():  # test_solver.py:233-239
    f = _frozen(1024)["f"]
    assert set(f.level_seconds) == {0, 1, 2}
    assert f.max_rank > 0
    assert all(c >= 1.0 for c in f.z_cond_per_level().values())


def test_offdiag_reconstruction_bound():  # test_skeleton.py:174-182, 208-227
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 512, seed=10, d=3)
    tree = hk.build_tree(ps, 64, seed=10)
    assert tree.depth == 3
    tau = 1e-6
    kern = hk.KernelSpec("gaussian", h=0.4)
    sk = hk.build_skeletons(tree, kern, hk.SkeletonConfig(tau=tau, max_rank=64, sample_mode="exact", seed=10))
    coords = np.asarray(tree.points.coords)
    worst = 0.0
    for node in tree.nodes:
        if node.is_leaf:
            continue
        left, right = tree.children(node)
        block = hk.eval_block(kern, coords[left.begin:left.end], coords[right.begin:right.end])
        mid = hk.eval_block(kern, coords[np.asarray(sk[left.index].indices)], coords[np.asarray(sk[right.index].indices)])
        approx = _basis(tree, sk, left).T @ mid @ _basis(tree, sk, right)
        denom = np.linalg.norm(block)
        if denom > 0:
            worst = max(worst, np.linalg.norm(block - approx) / denom)
    # reference bound 10 tau (depth + 1) = 4e-5; the reference's own worst
    # block is 5.906e-5 (REF_MEASURED: its own test fails).  The skeletons are
    # identical, so the GPU value equals the reference's to roundoff.
    assert abs(worst - REF_MEASURED["offdiag_worst"]) <= 1e-6 * REF_MEASURED["offdiag_worst"]


# ---------------------------------------------------------------- treecode
# test_treecode.py restated: upward pass, hmatvec, materialize_ktilde.

def _tiny(n=96, h=0.5, lam=1e-2, leaf=16, tau=1e-7, seed=0, d=2, factor=False):  # test_treecode.py:12-17
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", n, seed=seed, d=d)
    kern = hk.KernelSpec("gaussian", h=h, regularization=lam)
    return _instance(ps, kern, leaf=leaf, tau=tau, max_rank=64, sample_mode="exact", seed=seed, factor=factor)


def test_upward_pass_known_answers():  # test_treecode.py:20-50
    import paper_1701_02324_b200 as hk
    inst = _tiny()
    n = inst["tree"].n
    assert all(np.all(w == 0.0) for w in hk.upward_pass(inst["op"], np.zeros(n)).values())
    w = np.random.default_rng(3).standard_normal(n)
    weights = hk.upward_pass(inst["op"], w)
    for node in inst["tree"].nodes:
        if node.level == 0:
            continue
        expect = _basis(inst["tree"], inst["sk"], node) @ w[node.begin:node.end]
        assert np.allclose(weights[node.index], expect, atol=1e-12)
    with pytest.raises(ValueError):
        hk.upward_pass(inst["op"], np.zeros(3))
    ps = hk.generate("uniform_cube", 64, seed=2, d=2)
    inst0 = _instance(ps, hk.KernelSpec("gaussian", h=1e-9), leaf=16, tau=1e-4, max_rank=8, factor=False)
    assert all(v.size == 0 for v in hk.upward_pass(inst0["op"], np.ones(64)).values())


def test_hmatvec_known_answers():  # test_treecode.py:53-110
    import paper_1701_02324_b200 as hk
    # single leaf: exact
    ps = hk.generate("uniform_cube", 40, seed=4, d=3)
    kern = hk.KernelSpec("gaussian", h=0.4, regularization=1e-3)
    inst = _instance(ps, kern, leaf=64, factor=False)
    assert inst["tree"].depth == 0
    w = np.random.default_rng(5).standard_normal(40)
    dense = _dense(inst)
    got = hk.hmatvec(inst["op"], w, 1e-3)
    assert np.linalg.norm(got - dense @ w) <= 1e-13 * np.linalg.norm(dense @ w)
    # huge bandwidth: K -> ones
    ps = hk.generate("uniform_cube", 128, seed=6, d=2)
    diam = np.linalg.norm(ps.coords.max(0) - ps.coords.min(0))
    inst = _instance(ps, hk.KernelSpec("gaussian", h=1e6 * diam), leaf=32, tau=1e-10, factor=False)
    e = np.zeros(128)
    e[17] = 1.0
    assert np.max(np.abs(hk.hmatvec(inst["op"], e, 0.0) - 1.0)) <= 1e-6
    # frozen instance against the dense matvec
    ps = hk.generate("uniform_cube", 1024, 3, d=3)
    kern = hk.KernelSpec(family="gaussian", h=0.3, regularization=1e-2)
    inst = _instance(ps, kern, leaf=256, tau=1e-7, max_rank=384, sample_mode="exact", seed=3, factor=False)
    w = np.random.default_rng(7).standard_normal(1024)
    ref = _dense(inst) @ w
    assert np.linalg.norm(hk.hmatvec(inst["op"], w, 1e-2) - ref) <= 1e-5 * np.linalg.norm(ref)
    # linearity, length check
    inst = _tiny()
    rng = np.random.default_rng(8)
    w1, w2 = rng.standard_normal(96), rng.standard_normal(96)
    a, b = 0.7, -2.3
    lhs = hk.hmatvec(inst["op"], a * w1 + b * w2, 1e-2)
    rhs = a * hk.hmatvec(inst["op"], w1, 1e-2) + b * hk.hmatvec(inst["op"], w2, 1e-2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(lhs)
    with pytest.raises(ValueError):
        hk.hmatvec(inst["op"], np.zeros(5), 0.0)


def test_hmatvec_monotone_in_tau():  # test_treecode.py:93-105
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 256, seed=9, d=3)
    errs = []
    for tau in (1e-2, 1e-4, 1e-6):
        kern = hk.KernelSpec("gaussian", h=0.4, regularization=0.0)
        inst = _instance(ps, kern, leaf=64, tau=tau, max_rank=256, sample_mode="exact", factor=False)
        w = np.random.default_rng(10).standard_normal(256)
        ref = _dense(inst) @ w
        errs.append(np.linalg.norm(hk.hmatvec(inst["op"], w, 0.0) - ref) / np.linalg.norm(ref))
    assert errs[0] >= errs[1] >= errs[2]


def test_materialize_known_answers():  # test_treecode.py:113-133
    import paper_1701_02324_b200 as hk
    ps = hk.PointSet(np.array([[0.1, 0.2]]))
    kern = hk.KernelSpec("gaussian", h=0.5, regularization=0.25)
    out = hk.materialize_ktilde(_instance(ps, kern, leaf=4, factor=False)["op"], 0.25)
    assert out.shape == (1, 1) and out[0, 0] == 1.25
    kt = hk.materialize_ktilde(_tiny()["op"], 1e-2)
    assert np.linalg.norm(kt - kt.T) <= 1e-12 * np.linalg.norm(kt)
    inst = _tiny(n=48, leaf=8)
    kt = hk.materialize_ktilde(inst["op"], 0.5)
    e = np.zeros(48)
    for i in (0, 13, 47):
        e[:] = 0.0
        e[i] = 1.0
        assert np.array_equal(kt[:, i], hk.hmatvec(inst["op"], e, 0.5))


def test_solver_consistency_roundtrip():  # test_treecode.py:149-157
    import paper_1701_02324_b200 as hk
    inst = _tiny(n=256, leaf=32, factor=True)
    w = np.random.default_rng(11).standard_normal(256)
    b = hk.hmatvec(inst["op"], w, inst["f"].lam)
    x = hk.solve(inst["f"], b, in_tree_order=True)
    # reference bound 1e-9; the unmodified reference itself reaches 5.92e-9 here (REF_MEASURED)
    assert np.linalg.norm(x - w) <= 4 * REF_MEASURED["consistency_roundtrip"] * np.linalg.norm(w)


# ------------------------------------------------------------------ linalg
# test_linalg.py restated: pivoted QR, interpolative decomposition, dense LU.

def _decaying(rng, m, n, decay=0.5, rank=None):  # helpers.py:55-62
    rank = rank or min(m, n)
    u, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    v, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    return (u * decay ** np.arange(rank)) @ v.T


def test_pivoted_qr_known_answers():  # test_linalg.py:15-78
    import paper_1701_02324_b200 as hk
    res = hk.pivoted_qr(np.eye(3), 1e-12, 10)
    assert res.rank == 3 and np.allclose(np.abs(np.diag(res.r_factor)), 1.0)
    rng = np.random.default_rng(0)
    assert hk.pivoted_qr(np.outer(rng.standard_normal(5), rng.standard_normal(7)), 1e-10, 10).rank == 1
    # rank against the SVD oracle (singular values 2^-j)
    a = _decaying(np.random.default_rng(1), 50, 80)
    tol = 1e-6
    sigma = np.linalg.svd(a, compute_uv=False)
    oracle_rank = int(np.sum(sigma / sigma[0] > tol))
    assert oracle_rank == int(np.sum(0.5 ** np.arange(50) > tol))
    assert abs(hk.pivoted_qr(a, tol, 64).rank - oracle_rank) <= 1
    # |R_kk| non-increasing
    rng = np.random.default_rng(2)
    for _ in range(100):
        m, n = rng.integers(2, 40, size=2)
        res = hk.pivoted_qr(_decaying(rng, m, n, decay=rng.uniform(0.3, 0.9)), 1e-14, 64)
        assert np.all(np.diff(np.abs(np.diag(res.r_factor[:, : res.rank]))) <= 0.0)
    # empty / zero / cap / column space / bad arguments
    res = hk.pivoted_qr(np.zeros((0, 4)), 1e-8, 4)
    assert res.rank == 0 and res.r_factor.shape == (0, 4)
    assert hk.pivoted_qr(np.zeros((3, 0)), 1e-8, 4).rank == 0
    assert hk.pivoted_qr(np.zeros((5, 5)), 1e-8, 4).rank == 0
    assert hk.pivoted_qr(np.random.default_rng(3).standard_normal((20, 20)), 1e-15, 7).rank == 7
    a = _decaying(np.random.default_rng(4), 30, 25, decay=0.25)
    res = hk.pivoted_qr(a, 1e-9, 30)
    q, _ = np.linalg.qr(a[:, res.pivots[: res.rank]])
    assert np.linalg.norm(a - q @ (q.T @ a)) <= 10 * 1e-9 * np.linalg.norm(a)
    with pytest.raises(ValueError):
        hk.pivoted_qr(np.eye(2), -1.0, 3)
    with pytest.raises(ValueError):
        hk.pivoted_qr(np.eye(2), 1e-8, 0)


def test_interpolative_decomposition_known_answers():  # test_linalg.py:81-123
    import paper_1701_02324_b200 as hk
    rng = np.random.default_rng(5)
    c0, c2 = rng.standard_normal(6), rng.standard_normal(6)
    a = np.column_stack([c0, c0, c2])
    cols, interp = hk.interpolative_decomposition(a, 1e-12, 10)
    assert len(cols) == 2 and np.linalg.norm(a - a[:, cols] @ interp) <= 1e-12 * np.linalg.norm(a)
    rng = np.random.default_rng(6)
    a = rng.standard_normal((40, 3)) @ rng.standard_normal((3, 60))
    cols, interp = hk.interpolative_decomposition(a, 1e-10, 40)
    assert len(cols) == 3 and np.linalg.norm(a - a[:, cols] @ interp) <= 1e-9 * np.linalg.norm(a)
    cols, interp = hk.interpolative_decomposition(np.zeros((4, 6)), 1e-10, 4)
    assert cols.size == 0 and interp.shape == (0, 6)
    rng = np.random.default_rng(7)
    for _ in range(100):
        m, n = rng.integers(3, 30, size=2)
        a = _decaying(rng, m, n, decay=rng.uniform(0.2, 0.8))
        cols, interp = hk.interpolative_decomposition(a, 1e-8, 20)
        assert np.array_equal(interp[:, cols], np.eye(len(cols)))
    rng = np.random.default_rng(8)
    tol = 1e-6
    for _ in range(100):
        m, n = int(rng.integers(10, 50)), int(rng.integers(10, 50))
        a = _decaying(rng, m, n, decay=0.4)
        cols, interp = hk.interpolative_decomposition(a, tol, min(m, n))
        r = max(len(cols), 1)
        assert np.linalg.norm(a - a[:, cols] @ interp) <= 10 * np.sqrt(n * r) * tol * np.linalg.norm(a)


def test_dense_factor_known_answers():  # test_linalg.py:126-190
    import paper_1701_02324_b200 as hk
    b = np.random.default_rng(9).standard_normal((4, 3))
    assert np.allclose(hk.solve_dense(hk.factor_dense(np.eye(4)), b), b)
    assert np.allclose(hk.solve_dense(hk.factor_dense(np.diag([2.0, 2.0, 2.0])), np.array([2.0, 4.0, 6.0])), [1.0, 2.0, 3.0])
    rng = np.random.default_rng(10)
    m = rng.standard_normal((8, 8))
    a = m.T @ m + np.eye(8)
    rhs = rng.standard_normal(8)
    x = hk.solve_dense(hk.factor_dense(a), rhs)
    # hand-rolled elimination with partial pivoting as the oracle (helpers.py:18-37)
    aa, bb = a.copy(), rhs.copy()
    for col in range(8):
        piv = col + int(np.argmax(np.abs(aa[col:, col])))
        if piv != col:
            aa[[col, piv]], bb[[col, piv]] = aa[[piv, col]], bb[[piv, col]]
        for row in range(col + 1, 8):
            f = aa[row, col] / aa[col, col]
            aa[row, col:] -= f * aa[col, col:]
            bb[row] -= f * bb[col]
    xo = np.zeros(8)
    for row in range(7, -1, -1):
        xo[row] = (bb[row] - aa[row, row + 1:] @ xo[row + 1:]) / aa[row, row]
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    # condition number 1e6 by construction
    rng = np.random.default_rng(11)
    u, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    v, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    a = (u * np.logspace(0, -6, 12)) @ v.T
    xt = rng.standard_normal(12)
    assert np.linalg.norm(hk.solve_dense(hk.factor_dense(a), a @ xt) - xt) <= 1e-9 * np.linalg.norm(xt)
    with pytest.raises(hk.SingularMatrixError, match="step"):
        hk.factor_dense(np.array([[1.0, 2.0], [2.0, 4.0]]))
    with pytest.raises(hk.SingularMatrixError):
        hk.factor_dense(np.zeros((3, 3)))
    # P L U = A
    a = np.random.default_rng(12).standard_normal((9, 9))
    f = hk.factor_dense(a)
    lower, upper = np.tril(f.lu, -1) + np.eye(9), np.triu(f.lu)
    perm = np.arange(9)
    for i, p in enumerate(f.piv):
        perm[[i, p]] = perm[[p, i]]
    pmat = np.zeros((9, 9))
    pmat[perm, np.arange(9)] = 1.0
    assert np.linalg.norm(pmat @ lower @ upper - a) <= 1e-12 * np.linalg.norm(a)
    with pytest.raises(ValueError):
        hk.factor_dense(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        hk.solve_dense(hk.factor_dense(np.eye(3)), np.zeros(4))
    assert hk.solve_dense(hk.factor_dense(np.zeros((0, 0))), np.zeros(0)).shape == (0,)


# -------------------------------------------------------------- tree / kNN
# test_tree.py restated.

def _check_structure(hk, tree, n, m):  # test_tree.py:11-30
    perm = np.asarray(tree.perm)
    assert sorted(perm) == list(range(n))
    assert np.array_equal(perm[np.asarray(tree.inv_perm)], np.arange(n))
    for node in tree.nodes:
        assert node.size >= 1
        if not node.is_leaf:
            left, right = tree.children(node)
            assert (left.begin, right.end) == (node.begin, node.end)
            assert left.end == right.begin
            assert abs(left.size - right.size) <= 1
    for leaf in tree.leaves():
        assert leaf.size <= m
        if n >= m:
            assert leaf.size >= -(m // -2)
    for level_nodes in hk.levels(tree, bottom_up=False):
        spans = [(nd.begin, nd.end) for nd in level_nodes]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
            assert e0 == b1


def test_tree_known_answers():  # test_tree.py:33-100
    import paper_1701_02324_b200 as hk
    t = np.linspace(0, 1, 8)
    tree = hk.build_tree(hk.PointSet(np.column_stack([t, 2 * t])), 2, seed=0)
    assert len(tree.leaves()) == 4 and all(leaf.size == 2 for leaf in tree.leaves())
    tree = hk.build_tree(hk.generate("uniform_cube", 5, seed=1, d=2), 8, seed=0)
    assert tree.depth == 0 and len(tree.nodes) == 1
    _check_structure(hk, tree, 5, 8)
    rng = np.random.default_rng(3)
    coords = np.vstack([rng.normal(0.0, 0.1, (16, 2)), rng.normal(50.0, 0.1, (16, 2))])
    labels = np.array([0] * 16 + [1] * 16)
    tree = hk.build_tree(hk.PointSet(coords), 8, seed=2)
    left, right = tree.children(tree.nodes[0])
    perm = np.asarray(tree.perm)
    gl, gr = labels[perm[left.begin:left.end]], labels[perm[right.begin:right.end]]
    assert len(set(gl)) == 1 and len(set(gr)) == 1 and set(gl) != set(gr)
    for n, m, seed in [(17, 4, 0), (64, 8, 1), (100, 7, 2), (1000, 32, 3), (3, 2, 4), (257, 16, 5)]:
        ps = hk.generate("uniform_cube", n, seed=seed, d=3)
        tree = hk.build_tree(ps, m, seed=seed)
        _check_structure(hk, tree, n, m)
        assert np.array_equal(np.asarray(tree.points.coords), ps.coords[np.asarray(tree.perm)])
    tree = hk.build_tree(hk.generate("uniform_cube", 64, seed=6, d=2), 16, seed=0)
    assert [len(lv) for lv in hk.levels(tree, bottom_up=True)] == [4, 2, 1]
    assert [len(lv) for lv in hk.levels(tree, bottom_up=False)] == [1, 2, 4]
    ps = hk.generate("uniform_cube", 200, seed=7, d=3)
    t1, t2 = hk.build_tree(ps, 16, seed=9), hk.build_tree(ps, 16, seed=9)
    assert np.array_equal(np.asarray(t1.perm), np.asarray(t2.perm))
    with pytest.raises(ValueError):
        hk.build_tree(hk.generate("uniform_cube", 10, seed=0, d=2), 1)


def test_knn_known_answers():  # test_tree.py:103-137
    import paper_1701_02324_b200 as hk
    nb = np.asarray(hk.knn_bruteforce(hk.PointSet(np.array([[0.0], [1.0], [2.0]])), 1))
    assert nb[0, 0] == 1 and nb[2, 0] == 1
    nb = np.asarray(hk.knn_bruteforce(hk.generate("uniform_cube", 9, seed=8, d=2), 8))
    for i in range(9):
        assert sorted(nb[i]) == sorted(set(range(9)) - {i})
    ps = hk.generate("uniform_cube", 200, seed=12, d=3)
    got = np.asarray(hk.knn_bruteforce(ps, 5))
    expect = np.empty((200, 5), dtype=np.int64)  # per-point scan with explicit (distance, index) sorting
    for i in range(200):
        pairs = sorted((float((ps.coords[i] - ps.coords[j]) @ (ps.coords[i] - ps.coords[j])), j)
                       for j in range(200) if j != i)
        expect[i] = [j for _, j in pairs[:5]]
    assert np.array_equal(got, expect)
    nb = np.asarray(hk.knn_bruteforce(hk.PointSet(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])), 2))
    assert list(nb[3]) == [1, 2] and list(nb[0]) == [1, 2]
    ps = hk.generate("uniform_cube", 10, seed=0, d=2)
    with pytest.raises(ValueError):
        hk.knn_bruteforce(ps, 0)
    with pytest.raises(ValueError):
        hk.knn_bruteforce(ps, 10)


# --------------------------------------------------------------- skeletons
# test_skeleton.py restated (structure; the bound is above).

def test_skeleton_structure_known_answers():  # test_skeleton.py:95-161
    import paper_1701_02324_b200 as hk
    ps = hk.generate("uniform_cube", 64, seed=3, d=3)
    diameter = np.linalg.norm(ps.coords.max(0) - ps.coords.min(0))
    tree = hk.build_tree(ps, 16, seed=0)
    sk = hk.build_skeletons(tree, hk.KernelSpec("gaussian", h=1e6 * diameter),
                            hk.SkeletonConfig(tau=1e-8, max_rank=32, sample_mode="exact", seed=0))
    assert all(sk[i].rank == 1 for i in range(1, len(tree.nodes)))
    tree = hk.build_tree(hk.generate("uniform_cube", 32, seed=5, d=2), 8, seed=0)
    sk = hk.build_skeletons(tree, hk.KernelSpec("gaussian", h=1e-9),
                            hk.SkeletonConfig(tau=1e-4, max_rank=8, sample_mode="exact", seed=0))
    assert all(sk[i].rank == 0 for i in range(1, len(tree.nodes)))
    tree = hk.build_tree(hk.generate("uniform_cube", 6, seed=0, d=2), 8, seed=0)
    assert len(hk.build_skeletons(tree, hk.KernelSpec("gaussian"), hk.SkeletonConfig(sample_mode="exact"))) == 0
    tree = hk.build_tree(hk.generate("uniform_cube", 64, seed=1, d=2), 16, seed=0)
    assert tree.depth == 2
    assert len(hk.build_skeletons(tree, hk.KernelSpec("gaussian", h=0.4), hk.SkeletonConfig(sample_mode="exact"))) == 6
    # nestedness and the exact identity block
    # (the reference draws generate("gaussian_mixture", 300, seed=2, d=2) here, which never
    # returns in the unmodified reference -- four centres 12 sigma apart do not fit its 2-D box and
    # the rejection loop is unbounded; the package raises ValueError instead.  Same check on a cube.)
    with pytest.raises(ValueError, match="mixture"):
        hk.generate("gaussian_mixture", 300, seed=2, d=2)
    ps = hk.generate("uniform_cube", 300, seed=2, d=2)
    tree = hk.build_tree(ps, 32, seed=1)
    sk = hk.build_skeletons(tree, hk.KernelSpec("gaussian", h=1.0),
                            hk.SkeletonConfig(tau=1e-6, max_rank=24, samples=64, sample_mode="uniform", seed=7))
    for node in tree.nodes:
        if node.level == 0:
            continue
        s = sk[node.index]
        if node.is_leaf:
            cands = np.arange(node.begin, node.end)
        else:
            left, right = tree.children(node)
            cands = np.concatenate([np.asarray(sk[left.index].indices), np.asarray(sk[right.index].indices)])
            assert set(np.asarray(s.indices)) <= set(cands)
        pos = [int(np.flatnonzero(cands == q)[0]) for q in np.asarray(s.indices)]
        assert np.array_equal(np.asarray(s.interp)[:, pos], np.eye(s.rank))
        assert s.rank <= min(len(cands), 24)
    # accuracy monotone in tau
    ps = hk.generate("uniform_cube", 256, seed=9, d=3)
    tree = hk.build_tree(ps, 64, seed=9)
    kern = hk.KernelSpec("gaussian", h=0.4)
    coords = np.asarray(tree.points.coords)
    errs = []
    for tau in (1e-2, 1e-4, 1e-6):
        sk = hk.build_skeletons(tree, kern, hk.SkeletonConfig(tau=tau, max_rank=64, sample_mode="exact", seed=9))
        worst = 0.0
        for node in tree.nodes:
            if node.is_leaf:
                continue
            left, right = tree.children(node)
            block = hk.eval_block(kern, coords[left.begin:left.end], coords[right.begin:right.end])
            mid = hk.eval_block(kern, coords[np.asarray(sk[left.index].indices)], coords[np.asarray(sk[right.index].indices)])
            approx = _basis(tree, sk, left).T @ mid @ _basis(tree, sk, right)
            worst = max(worst, np.linalg.norm(block - approx) / np.linalg.norm(block))
        errs.append(worst)
    assert errs[0] >= errs[1] >= errs[2]


# ------------------------------------------------------------------ krylov
# test_krylov.py restated (the golden baseline run is tests/test_gpu_dense.py).

def test_gmres_known_answers():  # test_krylov.py:18-95
    import paper_1701_02324_b200 as hk
    b = np.random.default_rng(0).standard_normal(32)
    x, rep = hk.gmres(lambda v: v, lambda v: v, b, tol=1e-12)
    assert rep.iterations == 1 and rep.converged and np.allclose(x, b, atol=1e-12)
    rng = np.random.default_rng(1)
    m = rng.standard_normal((64, 64))
    a = m @ m.T + 64 * np.eye(64)
    a_inv = np.linalg.inv(a)
    b = rng.standard_normal(64)
    x, rep = hk.gmres(lambda v: a @ v, lambda v: a_inv @ v, b, tol=1e-12)
    assert rep.iterations == 1 and rep.final_residual <= 1e-12
    rng = np.random.default_rng(2)
    m = rng.standard_normal((80, 80))
    a = m @ m.T + 10 * np.eye(80)
    b = rng.standard_normal(80)
    x, rep = hk.gmres(lambda v: a @ v, lambda v: v, b, tol=1e-10, restart=30)
    assert abs(rep.final_residual - np.linalg.norm(b - a @ x) / np.linalg.norm(b)) <= 1e-12
    assert rep.residuals[-1] == rep.final_residual
    rng = np.random.default_rng(3)
    m = rng.standard_normal((120, 120))
    a = m @ m.T + 5 * np.eye(120)
    b = rng.standard_normal(120)
    x, rep = hk.gmres(lambda v: a @ v, lambda v: v, b, tol=1e-10, restart=25)
    for i in range(1, len(rep.residuals)):
        if i % 25:
            assert rep.residuals[i] <= rep.residuals[i - 1] * (1.0 + 1e-9)
    x, rep = hk.gmres(lambda v: v, lambda v: v, np.zeros(5))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
    with pytest.raises(ValueError, match="shape"):
        hk.gmres(lambda v: v[:2], lambda v: v, np.ones(4))
    rng = np.random.default_rng(4)
    m = rng.standard_normal((60, 60))
    a = m @ m.T + 30 * np.eye(60)
    b = rng.standard_normal(60)
    x, rep = hk.gmres(lambda v: a @ v, lambda v: v, b, tol=1e-9, restart=5, max_iter=400)
    assert rep.converged and rep.restarts > 0 and np.linalg.norm(b - a @ x) <= 1e-9 * np.linalg.norm(b)
    rng = np.random.default_rng(5)
    m = rng.standard_normal((50, 50))
    a = m @ m.T + 1e-8 * np.eye(50)
    b = rng.standard_normal(50)
    x, rep = hk.gmres(lambda v: a @ v, lambda v: v, b, tol=1e-14, restart=10, max_iter=20)
    assert rep.iterations <= 20 and (not rep.converged or rep.final_residual <= 1e-14)


# ----------------------------------------------------------------- kernels
# test_kernels.py restated (closed forms, conventions, validation, symmetry).

def test_kernel_known_answers():  # test_kernels.py:7-92
    import paper_1701_02324_b200 as hk
    x = np.array([[0.3, -0.2, 1.0]])
    assert hk.eval_block(hk.KernelSpec("gaussian", h=0.7), x, x)[0, 0] == 1.0
    val = hk.eval_block(hk.KernelSpec("gaussian", h=1.0), np.array([[0.0, 0.0]]), np.array([[1.0, 1.0]]))[0, 0]
    assert abs(val - 0.3678794412) < 1e-9
    lap = hk.KernelSpec("laplace3d")
    o, e1 = np.array([[0.0, 0.0, 0.0]]), np.array([[1.0, 0.0, 0.0]])
    assert abs(hk.eval_block(lap, o, e1)[0, 0] - 0.0795774715) < 1e-9
    assert hk.eval_block(lap, o, o)[0, 0] == 0.0  # self-interaction convention
    poly = hk.KernelSpec("polynomial", degree=3, shift=1.0)
    assert abs(hk.eval_block(poly, np.array([[1.0, 2.0]]), np.array([[0.5, 0.25]]))[0, 0] - 2.0 ** 3) < 1e-12
    k = hk.KernelSpec("gaussian", h=0.5, regularization=0.25)
    x = np.random.default_rng(0).random((4, 2))
    assert np.all(np.diag(hk.eval_block(k, x, x)) == 1.0)  # lambda is not added
    assert hk.eval_system_diag_shift(hk.KernelSpec("gaussian", regularization=0.0)) == 0.0
    assert hk.eval_system_diag_shift(hk.KernelSpec("gaussian", regularization=1e-2)) == 1e-2
    with pytest.raises(ValueError, match="dimension mismatch"):
        hk.eval_block(hk.KernelSpec("gaussian"), np.zeros((2, 3)), np.zeros((2, 2)))
    with pytest.raises(ValueError, match="3-d"):
        hk.eval_block(hk.KernelSpec("laplace3d"), np.zeros((2, 2)), np.zeros((2, 2)))
    for spec in (dict(family="gaussian", h=0.0), dict(family="gaussian", h=-1.0), dict(family="polynomial", degree=0),
                 dict(family="polynomial", shift=-0.5), dict(family="gaussian", regularization=-1e-3),
                 dict(family="matern")):
        with pytest.raises(ValueError):
            hk.KernelSpec(**spec)
    rng = np.random.default_rng(13)
    xt, xs = rng.random((37, 3)), rng.random((21, 3))
    for family, kw in (("gaussian", dict(h=0.4)), ("laplace3d", {}), ("polynomial", dict(degree=2, shift=0.3))):
        kk = hk.KernelSpec(family, **kw)
        assert np.array_equal(hk.eval_block(kk, xt, xs), hk.eval_block(kk, xs, xt).T)
    x = np.random.default_rng(14).random((30, 3))
    g = hk.eval_block(hk.KernelSpec("gaussian", h=0.2), x, x)
    assert np.all(g > 0.0) and np.all(g <= 1.0)
    assert np.all(hk.eval_block(lap, x, x)[~np.eye(30, dtype=bool)] > 0.0)
    # entries do not depend on how the rows are split over launches
    rng = np.random.default_rng(15)
    xt, xs = rng.random((700, 3)), rng.random((11, 3))
    k = hk.KernelSpec("gaussian", h=0.3)
    full = hk.eval_block(k, xt, xs)
    parts = np.vstack([hk.eval_block(k, xt[i:i + 64], xs) for i in range(0, 700, 64)])
    assert np.array_equal(full, parts)
