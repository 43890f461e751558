"""Tall-skinny QR pre-reduction (csrc/tsqr.cu) in front of the pivoted QR:
tall blocks (rows >= 1024 and >= 2 x columns) are reduced to their
triangular factor before linalg.py:43-136's pivoting runs, so pivots, rank,
|R| and the interpolation coefficients must still equal the oracle's, which
pivots on the block itself."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _kernel_block(rng, m, n, d=3, h=0.7):
    """A numerically low-rank Gaussian kernel block (the matrices the path
    actually factors: singular values decay to roundoff)."""
    xt = rng.random((m, d)) + 1.5
    xs = rng.random((n, d))
    d2 = ((xt[:, None, :] - xs[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (2 * h * h))


CASES = [
    # m, n, tol, max_rank, kind
    (1024, 32, 1e-10, 32, "random"),        # one slab chunk, single panel
    (1500, 100, 1e-8, 64, "kernel"),        # ragged rows / columns (partial slab, partial panel and tile)
    (4097, 257, 1e-6, 200, "kernel"),       # columns not a multiple of 16
    (3000, 512, 1e-5, 256, "kernel"),       # the C3 leaf shape
    (40000, 64, 1e-9, 64, "kernel"),        # many chunks: exercises the merge tree
    (2048, 96, 1e-300, 96, "random"),       # full rank, rank set by the cap
]


@pytest.mark.parametrize("m,n,tol,mr,kind", CASES)
def test_prereduced_qrcp_equals_oracle(m, n, tol, mr, kind):
    import paper_1701_02324_b200 as hk
    from oracle import hks_oracle as O
    rng = np.random.default_rng([m, n])
    a = _kernel_block(rng, m, n) if kind == "kernel" else rng.standard_normal((m, n))
    piv, rf, rank = O.qrcp(a, tol, mr)
    qr = hk.pivoted_qr(a, tol, mr)
    assert qr.rank == rank
    assert np.array_equal(qr.pivots[:rank], piv[:rank])
    # |R| rows agree relative to the largest entry (signs follow the reflectors)
    scale = np.abs(rf).max(initial=1.0)
    assert np.abs(np.abs(qr.r_factor) - np.abs(rf)).max(initial=0.0) <= 1e-11 * scale
    cols, p = hk.interpolative_decomposition(a, tol, mr)
    ocols, op = O.interp_decomp(a, tol, mr)
    assert np.array_equal(cols, ocols)
    assert np.array_equal(p[:, cols], np.eye(cols.size))
    c11 = np.linalg.cond(rf[:, :rank]) if rank else 1.0
    assert np.linalg.norm(p - op) <= 1e-13 * c11 * max(np.linalg.norm(op), 1.0) + 1e-12


def test_column_norms_preserved():
    """R^T R == A^T A to roundoff: read R back through pivoted_qr with no
    truncation (rank = n) and compare the Gram matrices."""
    import paper_1701_02324_b200 as hk
    rng = np.random.default_rng(5)
    a = rng.standard_normal((6000, 80))
    qr = hk.pivoted_qr(a, 1e-300, 80)
    assert qr.rank == 80
    r = qr.r_factor
    g = a[:, qr.pivots].T @ a[:, qr.pivots]
    assert np.abs(r.T @ r - g).max() <= 1e-12 * np.abs(g).max()
