"""GPU dense primitives vs the reference's known answers and the oracle
(tests/test_kernels.py, tests/test_linalg.py, tests/test_krylov.py of the
reference)."""

import numpy as np
import pytest
import scipy.linalg

from golden_cases import GOLDEN
from oracle import hks_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hk():
    import paper_1701_02324_b200 as hk
    return hk


def test_kernel_known_answers(hk):
    x = np.array([[0.3, -0.2, 1.0]])
    assert hk.eval_block(hk.KernelSpec("gaussian", h=0.7), x, x)[0, 0] == 1.0
    v = hk.eval_block(hk.KernelSpec("gaussian", h=1.0), [[0.0, 0.0]], [[1.0, 1.0]])[0, 0]
    assert abs(v - 0.3678794412) < 1e-9
    k = hk.KernelSpec("laplace3d")
    assert abs(hk.eval_block(k, [[0.0, 0, 0]], [[1.0, 0, 0]])[0, 0] - 0.0795774715) < 1e-9
    assert hk.eval_block(k, [[0.0, 0, 0]], [[0.0, 0, 0]])[0, 0] == 0.0
    kp = hk.KernelSpec("polynomial", degree=3, shift=1.0)
    assert abs(hk.eval_block(kp, [[1.0, 2.0]], [[0.5, 0.25]])[0, 0] - 8.0) < 1e-12
    xs = np.random.default_rng(0).random((4, 2))
    assert np.all(np.diag(hk.eval_block(hk.KernelSpec("gaussian", regularization=0.25), xs, xs)) == 1.0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        hk.eval_block(hk.KernelSpec("gaussian"), np.zeros((2, 3)), np.zeros((2, 2)))
    with pytest.raises(ValueError, match="3-d"):
        hk.eval_block(hk.KernelSpec("laplace3d"), np.zeros((2, 2)), np.zeros((2, 2)))


@pytest.mark.parametrize("family,d", [("gaussian", 8), ("gaussian", 784), ("laplace3d", 3), ("polynomial", 5)])
def test_eval_block_vs_oracle_and_symmetry(hk, family, d):
    rng = np.random.default_rng(d)
    x = rng.random((150, d))
    y = rng.random((97, d))
    kern = hk.KernelSpec(family, h=0.9, degree=3, shift=0.5)
    got = hk.eval_block(kern, x, y)
    ref = O.kernel_block(family, x, y, h=0.9, degree=3, shift=0.5)
    # 8 ulp plus the conditioning of exp(-sq / 2h^2): a relative error of
    # ~sqrt(d) eps in sq becomes an absolute error of that size times the
    # exponent in the value (d = 784 leaves exponents of ~80)
    sq = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    cond = sq / (2 * 0.9 ** 2) if family == "gaussian" else np.ones_like(sq)
    if d >= 64:  # GEMM-form distances on the tensor path: the roundoff scales with |x|^2 + |y|^2, not d^2
        nn = (x * x).sum(1)[:, None] + (y * y).sum(1)[None, :]
        cond = nn / (2 * 0.9 ** 2)
    tol = 8 * np.spacing(np.abs(ref)) + np.abs(ref) * 4 * np.sqrt(d) * 2.3e-16 * cond + 1e-300
    assert np.all(np.abs(got - ref) <= tol)
    if family != "polynomial":
        assert np.array_equal(got, hk.eval_block(kern, y, x).T)


def test_chunk_invariance_large_block(hk):
    rng = np.random.default_rng(3)
    x = rng.random((1300, 4))
    kern = hk.KernelSpec("gaussian", h=0.3)
    full = hk.eval_block(kern, x, x)
    part = hk.eval_block(kern, x[600:700], x)
    assert np.array_equal(full[600:700], part)


@pytest.mark.parametrize("n", [1, 7, 64, 300, 700, 1024])
def test_factor_solve_vs_scipy(hk, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + n * 0.05 * np.eye(n)
    f = hk.factor_dense(a)
    lu, piv = scipy.linalg.lu_factor(a)
    # same pivot sequence as LAPACK on a generic matrix, LU to roundoff
    assert np.array_equal(f.piv, piv)
    assert np.allclose(f.lu, lu, rtol=1e-9, atol=1e-11 * np.abs(lu).max())
    b = rng.standard_normal((n, 3))
    x = hk.solve_dense(f, b)
    assert np.linalg.norm(a @ x - b) <= 1e-10 * np.linalg.norm(a) * np.linalg.norm(x)
    x1 = hk.solve_dense(f, b[:, 1])
    assert np.array_equal(x1, x[:, 1])


def test_singular_reports_step(hk):
    a = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [0.0, 0.0, 0.0]])
    with pytest.raises(hk.SingularMatrixError, match="step"):
        hk.factor_dense(a)


def test_gmres_unpreconditioned_golden(hk):
    z = np.load(GOLDEN / "gmres_n512.npz")
    tree = O.build_tree(np.random.default_rng([3, 0, 0]).random((512, 3)), 512, 3)
    dense = O.kernel_block("gaussian", tree.coords, tree.coords, h=0.5)
    dense[np.diag_indices(512)] += 1e-6
    b = np.random.default_rng([3, 41]).standard_normal(512)
    x, rep = hk.gmres(lambda v: dense @ v, lambda v: v, b, tol=1e-8, max_iter=500, restart=50)
    assert rep.iterations == int(z["iterations"])
    assert rep.converged == bool(z["converged"])
    assert rep.final_residual == pytest.approx(float(z["final_residual"]), rel=1e-3)


def test_gmres_identity_and_shape_check(hk):
    b = np.random.default_rng(0).standard_normal(32)
    x, rep = hk.gmres(lambda v: v, lambda v: v, b, tol=1e-12)
    assert rep.iterations == 1 and rep.converged
    assert np.allclose(x, b, atol=1e-12)
    with pytest.raises(ValueError, match="shape"):
        hk.gmres(lambda v: v[:2], lambda v: v, np.ones(4))
    x, rep = hk.gmres(lambda v: v, lambda v: v, np.zeros(5))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
