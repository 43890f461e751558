"""Lockstep multi-RHS GMRES (krylov.gmres_multi / hybrid_solve_multi): every
column must be the single-column hybrid_solve bit for bit -- same iteration
count, residual history and solution (the batched matvec / solve are
column-independent)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _instance(lam=1e-3, tau=1e-5, s=48):
    import paper_1701_02324_b200 as hk
    rng = np.random.default_rng([9, 0])
    x = rng.random((4096, 3))
    tree = hk.build_tree(hk.PointSet(x), 128, seed=0)
    kern = hk.KernelSpec("gaussian", h=0.25, regularization=lam)
    cfg = hk.SkeletonConfig(tau=tau, max_rank=s, samples=4 * s, sample_mode="uniform", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg)
    op = hk.build_operator(tree, sk, kern)
    return hk, op, hk.factorize(op, lam)


@pytest.mark.parametrize("tol,restart", [(1e-10, 50), (1e-12, 2)])
def test_multi_equals_single(tol, restart):
    hk, op, f = _instance()
    from paper_1701_02324_b200.krylov import hybrid_solve_multi
    B = np.random.default_rng(3).standard_normal((op.n, 4))
    B[:, 2] = 0.0  # a zero right-hand side converges at once
    X, reps = hybrid_solve_multi(op, f, B, tol=tol, max_iter=20, restart=restart)
    for j in range(B.shape[1]):
        xj, rj = hk.hybrid_solve(op, f, B[:, j], tol=tol, max_iter=20, restart=restart)
        assert reps[j].iterations == rj.iterations and reps[j].restarts == rj.restarts
        assert reps[j].converged == rj.converged
        np.testing.assert_array_equal(np.asarray(reps[j].residuals), np.asarray(rj.residuals))
        np.testing.assert_array_equal(X[:, j], xj)
        assert reps[j].final_residual == rj.final_residual


def test_multi_unpreconditioned_like_case():
    """A weak preconditioner (large tau, small ranks): several iterations and
    restarts per column, columns finishing at different counts."""
    hk, op, f = _instance(lam=1e-4, tau=1e-2, s=8)
    from paper_1701_02324_b200.krylov import hybrid_solve_multi
    B = np.random.default_rng(4).standard_normal((op.n, 3))
    X, reps = hybrid_solve_multi(op, f, B, tol=1e-9, max_iter=40, restart=5)
    for j in range(3):
        xj, rj = hk.hybrid_solve(op, f, B[:, j], tol=1e-9, max_iter=40, restart=5)
        assert reps[j].iterations == rj.iterations
        np.testing.assert_array_equal(X[:, j], xj)
