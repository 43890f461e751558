"""GPU parity of the factorize / solve / matvec core against the oracle.

The oracle's own tree and skeletons (pinned to the reference by
test_oracle_golden.py) are uploaded, so these tests isolate the device
build_operator / factorize / solve / hmatvec from the setup stages.
Tolerances are relative to the quantity's norm and stated per check; they
follow the reference's own tests (tests/test_solver.py, test_treecode.py).
"""

import numpy as np
import pytest

from golden_cases import ALL_CASES, kern_of, load, matvec_w, oracle_instance, rhs_for

pytestmark = pytest.mark.gpu

CASES = ["tiny_n10", "rank0_n128", "frozen_n1024", "laplace_n1024", "poly_n1024",
         "gauss_uniform_n2000", "c1_n4096", "c2_n8192", "c3_n8192", "c4_n8192", "c5_n2048"]


def _gpu_instance(name):
    import paper_1701_02324_b200 as hk
    g = load(name)
    m = g["meta"]
    inst = oracle_instance(name)
    tr = inst["tree"]
    tree = hk.PartitionTree.from_host(tr.coords, tr.perm, m["leaf"], tr.split_dir, tr.split_val)
    cfg = hk.SkeletonConfig(tau=m["tau"], max_rank=m["max_rank"], samples=m["samples"],
                            sample_mode=m["mode"], seed=m["seed"])
    skels = hk.SkeletonSet.from_host(tree, inst["skel"], cfg)
    kern = hk.KernelSpec(m["family"], h=m["h"], degree=m["degree"], shift=m["shift"],
                         regularization=m["lam"])
    op = hk.build_operator(tree, skels, kern)
    f = hk.factorize(op, m["lam"])
    return hk, inst, op, f, m


_CACHE = {}


def gpu_instance(name):
    if name not in _CACHE:
        _CACHE[name] = _gpu_instance(name)
    return _CACHE[name]


def eval_tol(ref, xa, xb, m):
    """8 ulp plus the conditioning of the kernel in the squared distance:
    a relative error ~ sqrt(d) eps in sq becomes sq / (2 h^2) times that in
    exp(-sq / 2h^2) (the far-field entries of root couplings)."""
    sq = ((xa[:, None, :] - xb[None, :, :]) ** 2).sum(-1)
    cond = sq / (2 * m["h"] ** 2) if m["family"] == "gaussian" else np.ones_like(sq)
    return 8 * np.spacing(np.abs(ref)) + np.abs(ref) * 4 * np.sqrt(xa.shape[1]) * 2.3e-16 * (1 + cond) + 1e-300


@pytest.mark.parametrize("name", CASES)
def test_couplings_and_leaf_blocks(name):
    hk, inst, op, f, m = gpu_instance(name)
    x = inst["tree"].coords
    for i, c in inst["coup"].items():
        got = op.couplings[i]
        assert got.shape == c.shape
        xa, xb = x[inst["skel"][2 * i + 1][0]], x[inst["skel"][2 * i + 2][0]]
        assert np.all(np.abs(got - c) <= eval_tol(c, xa, xb, m)), f"node {i}"
    for i, blk in inst["leaf"].items():
        got = op.leaf_blocks[i]
        b, e = inst["tree"].begin[i], inst["tree"].end[i]
        assert np.all(np.abs(got - blk) <= eval_tol(blk, x[b:e], x[b:e], m))
        assert np.array_equal(got, got.T)  # exact symmetry (tests/test_kernels.py:69-81)
        if m["family"] == "gaussian":
            assert np.all(np.diag(got) == 1.0)


# instances whose compressed operator is itself ill-conditioned: Ktilde +
# lam I of gauss_uniform_n2000 has cond 8.9e6 and eigenvalues with real part
# down to -1.7, the reduced matrices reach cond 7e6 -- roundoff differences
# between two correct implementations are amplified to ~1e-2, so parity is
# judged by the residual against Ktilde (north_star: "relative residual ...
# matching the oracle's to within a stated factor")
ILL_CONDITIONED = {"gauss_uniform_n2000"}


def factor_tol(name):
    return 5e-2 if name in ILL_CONDITIONED else 1e-8


@pytest.mark.parametrize("name", CASES)
def test_theta_and_push_match_oracle(name):
    hk, inst, op, f, m = gpu_instance(name)
    tol = factor_tol(name)
    for i, fo in inst["fac"].items():
        fg = f.factors[i]
        if "theta" in fo:
            ref = fo["theta"]
            err = np.linalg.norm(fg.theta - ref)
            assert err <= tol * max(np.linalg.norm(ref), 1e-300), f"theta node {i}: {err}"
        if "push" in fo:
            ref = fo["push"]
            assert np.linalg.norm(fg.child_push - ref) <= tol * max(np.linalg.norm(ref), 1e-300)
        if "z_cond" in fo and np.isfinite(fo["z_cond"]):
            assert fg.z_cond == pytest.approx(fo["z_cond"], rel=1e-3 if tol < 1e-3 else 0.5), f"z_cond node {i}"


@pytest.mark.parametrize("name", CASES)
def test_solve_matches_oracle_and_golden(name):
    hk, inst, op, f, m = gpu_instance(name)
    g = load(name)
    b = rhs_for(m)
    x = hk.solve_multi(f, b, in_tree_order=True)
    # golden x from the unmodified reference; the oracle agrees to 1e-7
    # (test_oracle_golden.py), the GPU must agree at the same level (or, for
    # the ill-conditioned instance, at a residual within 10x the oracle's)
    from oracle import hks_oracle as O
    t, sk, lf, cp = inst["tree"], inst["skel"], inst["leaf"], inst["coup"]
    for j in range(b.shape[1]):
        res_g = np.linalg.norm(O.matvec(t, sk, lf, cp, x[:, j], m["lam"]) - b[:, j]) / np.linalg.norm(b[:, j])
        res_o = np.linalg.norm(O.matvec(t, sk, lf, cp, g["x"][:, j], m["lam"]) - b[:, j]) / np.linalg.norm(b[:, j])
        assert res_g <= 10 * res_o + 1e-13, (res_g, res_o)
    xtol = 5e-2 if name in ILL_CONDITIONED else 1e-7
    assert np.linalg.norm(x - g["x"]) <= xtol * np.linalg.norm(g["x"])
    for j in range(b.shape[1]):
        xj = hk.solve(f, b[:, j], in_tree_order=True)
        assert np.array_equal(xj, x[:, j])  # columns bitwise (tests/test_solver.py:174-185)


@pytest.mark.parametrize("name", CASES)
def test_hmatvec_matches_golden(name):
    hk, inst, op, f, m = gpu_instance(name)
    g = load(name)
    u = hk.hmatvec(op, matvec_w(m), m["lam"])
    assert np.linalg.norm(u - g["u"]) <= 1e-12 * np.linalg.norm(g["u"])


@pytest.mark.parametrize("name", ["frozen_n1024", "c1_n4096", "c2_n8192"])
def test_roundtrip(name):
    hk, inst, op, f, m = gpu_instance(name)
    w = np.random.default_rng(7).standard_normal(op.n)
    x = hk.solve(f, hk.hmatvec(op, w, m["lam"]), in_tree_order=True)
    xo = inst["tree"]  # oracle round trip error sets the bar
    from oracle import hks_oracle as O
    xr = O.solve(inst["tree"], inst["skel"], inst["coup"], inst["fac"],
                 O.matvec(inst["tree"], inst["skel"], inst["leaf"], inst["coup"], w, m["lam"]))
    err_o = np.linalg.norm(xr - w) / np.linalg.norm(w)
    err_g = np.linalg.norm(x - w) / np.linalg.norm(w)
    assert err_g <= max(10 * err_o, 1e-12)


def test_input_order_flag():
    hk, inst, op, f, m = gpu_instance("gauss_uniform_n2000")
    b = np.random.default_rng(10).standard_normal(op.n)
    perm = op.tree.perm
    x_in = hk.solve(f, b, in_tree_order=False)
    x_tree = hk.solve(f, b[perm], in_tree_order=True)
    assert np.array_equal(x_in[perm], x_tree)


def test_upward_pass_matches_oracle():
    hk, inst, op, f, m = gpu_instance("c1_n4096")
    from oracle import hks_oracle as O
    w = np.random.default_rng(3).standard_normal(op.n)
    got = hk.upward_pass(op, w)
    ref = O.upward(inst["tree"], inst["skel"], w)
    for i, v in ref.items():
        assert np.allclose(got[i], v, rtol=1e-12, atol=1e-12)


def test_materialize_symmetric_and_columns():
    hk, inst, op, f, m = gpu_instance("frozen_n1024")
    kt = hk.materialize_ktilde(op, m["lam"])
    assert np.linalg.norm(kt - kt.T) <= 1e-12 * np.linalg.norm(kt)
    e = np.zeros(op.n)
    e[17] = 1.0
    assert np.array_equal(kt[:, 17], hk.hmatvec(op, e, m["lam"]))


def test_lambda_validation_and_independent_factorizations():
    hk, inst, op, f, m = gpu_instance("gauss_uniform_n2000")
    with pytest.raises(ValueError):
        hk.factorize(op, -1.0)
    other = hk.factorize(op, 0.5)
    assert other.lam == 0.5 and f.lam == m["lam"]
    b = rhs_for(m)[:, 0]
    assert np.array_equal(hk.solve(f, b, in_tree_order=True), hk.solve_multi(f, rhs_for(m), in_tree_order=True)[:, 0])
    with pytest.raises(ValueError, match="lambda"):
        hk.hybrid_solve(op, other, b)


def test_hybrid_compressed():
    hk, inst, op, f, m = gpu_instance("frozen_n1024")
    g = load("frozen_n1024")
    b = rhs_for(m)[:, 0]
    x, rep = hk.hybrid_solve(op, f, b, tol=1e-10, restart=50, operator_mode="compressed")
    assert rep.iterations <= int(g["hybrid_iterations"]) + 1
    assert np.linalg.norm(x - g["hybrid_x"]) <= 1e-7 * np.linalg.norm(g["hybrid_x"])


def test_hybrid_dense_oracle_corrects_compression():
    hk, inst, op, f, m = gpu_instance("frozen_n1024")
    b = np.random.default_rng(7).standard_normal(op.n)
    x, rep = hk.hybrid_solve(op, f, b, tol=1e-10, operator_mode="dense_oracle")
    assert rep.converged and rep.iterations <= 15
    from oracle import hks_oracle as O
    tr = inst["tree"]
    dense = O.kernel_block("gaussian", tr.coords, tr.coords, h=m["h"])
    dense[np.diag_indices(op.n)] += m["lam"]
    assert np.linalg.norm(b - dense @ x) / np.linalg.norm(b) <= 1e-10
