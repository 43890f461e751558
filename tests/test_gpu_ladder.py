"""Reduced-N parity ladder: the BASELINE configurations'
generators, kernels and ranks at N = 16384 and 65536 (the largest N the
reference's kNN guard admits, tree.py:159,170-171), GPU path against
fixtures made by the UNMODIFIED reference (tests/golden/make_golden.py,
``ladder_*``):

* tree permutation, kNN lists (SHA-256 of the full int64 array) and every
  skeleton index set / rank: bit-exact;
* the reference's own residual ||(lam I + Ktilde) x - b|| / ||b||: the
  GPU's within a factor 10 either way, no absolute floor;
* the sampled-row metrics (256 rows of the exact K + lam I, BASELINE.md
  4.2): within a factor 1.5 of the reference's;
* x against the reference's x (sketches on 8 Gaussian vectors, the whole x
  at N = 16384): within 1e-6 relative -- both solve the same Ktilde system,
  whose reduced matrices reach z_cond ~ 1e6 at C3;
* C5: the hybrid GMRES iteration count equals the reference's.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem[len("ladder_"):] for p in GOLDEN.glob("ladder_*.npz"))
RESID_FACTOR = 10.0
SAMPLED_FACTOR = 1.5
_CACHE = {}


def _load(name):
    z = np.load(GOLDEN / f"ladder_{name}.npz")
    g = {k: z[k] for k in z.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def _run(name):
    if name in _CACHE:
        return _CACHE[name]
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import workloads as W
    g = _load(name)
    m = g["meta"]
    w = W.CONFIGS[m["workload"]].scaled(m["n"])
    x = W.points(w, 0)
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == str(g["coords_sha256"])
    kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
    skels = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, skels, kern)
    f = hk.factorize(op, w.lam)
    b = np.random.default_rng([0, 1000]).standard_normal((w.n, 2))
    xs = hk.solve_multi(f, b, in_tree_order=True)
    _CACHE[name] = (hk, w, g, tree, knn, skels, op, f, b, xs)
    return _CACHE[name]


@pytest.mark.parametrize("name", CASES)
def test_ladder_structure_bit_exact(name):
    hk, w, g, tree, knn, skels, op, f, b, xs = _run(name)
    assert tree.depth == g["meta"]["depth"]
    assert np.array_equal(np.asarray(tree.perm), g["perm"].astype(np.int64))
    k64 = np.ascontiguousarray(np.asarray(knn, dtype=np.int64))
    if hashlib.sha256(k64.tobytes()).hexdigest() != str(g["knn_sha256"]):
        head = g["knn_head"]
        bad = np.flatnonzero((k64[: head.shape[0]] != head).any(axis=1))
        pytest.fail(f"kNN lists differ from the reference's (first differing head rows {bad[:5].tolist()})")
    ranks = skels.ranks
    assert np.array_equal(ranks[1:], g["ranks"][1:])
    off, idx = g["skel_off"], g["skel_idx"]
    ref = {i: idx[off[i]: off[i + 1]].astype(np.int64) for i in range(1, len(ranks))}
    diff = [i for i in range(1, len(ranks)) if not np.array_equal(np.asarray(skels[i].indices), ref[i])]
    # "skeleton index sets must match except where pivots tie" (north star):
    # every node whose candidates are the reference's and whose pivot
    # sequence still differs must diverge either at a near-tie of two column
    # norms or past the block's numerical rank -- fixed-rank configurations
    # (tau = 1e-300) keep pivoting on residual columns of norm ~1e-16 of the
    # first pivot's, where the choice is decided by rounding (the reference
    # itself picks differently there with 1 and 8 BLAS threads: C4 N=16384
    # node 8 at step 220, |R_kk| / |R_00| = 9e-17).  Audited with the
    # oracle's QRCP (linalg.py:43-104); ancestors may then differ too.
    tainted = set()
    for i in sorted(diff, reverse=True):
        kids = (2 * i + 1, 2 * i + 2)
        if tree.nodes[i].is_leaf or not (set(kids) & tainted):
            gap, floor = _tie_gap(w, tree, knn, i, np.asarray(skels[i].indices), ref[i], ref)
            assert gap <= 1e-10 or floor <= 1e-13, (
                f"node {i}: pivot sequences diverge at a column-norm gap of {gap:.2e} "
                f"(remaining norms {floor:.2e} of the first pivot's)")
        tainted.add(i)


def _tie_gap(w, tree, knn, i, got, want, ref):
    """At the first step where the GPU's pivot sequence `got` leaves the
    reference's `want` for node i, with the oracle's QRCP (from-scratch
    norms, oracle/hks_oracle.py) advanced along the reference's pivots:
    (|n_ref - n_gpu| / n_max of the two competing columns' residual norms,
    n_max / the first pivot's norm)."""
    from oracle import hks_oracle as O
    nd = tree.nodes[i]
    x = np.asarray(tree.points.coords)
    rows = O.sample_rows(w.n, nd.begin, nd.end, i, w.samples, "knn_augmented", 0, np.asarray(knn))
    cands = np.arange(nd.begin, nd.end) if nd.is_leaf else np.concatenate([ref[2 * i + 1], ref[2 * i + 2]])
    a = O.kernel_block("gaussian", x[rows], x[cands], h=w.h)
    pos = {int(c): j for j, c in enumerate(cands)}
    k = int(np.flatnonzero(got[: len(want)] != want[: len(got)])[0])
    r = a.copy()
    first = np.sqrt(np.sum(r ** 2, axis=0)).max()
    cols = list(range(r.shape[1]))
    for step in range(k):  # Householder steps along the reference's pivots
        j = cols.index(pos[int(want[step])])
        cols[step], cols[j] = cols[j], cols[step]
        r[:, [step, j]] = r[:, [j, step]]
        v = r[step:, step].copy()
        alpha = -np.copysign(np.linalg.norm(v), v[0]) if v[0] != 0 else -np.linalg.norm(v)
        v[0] -= alpha
        vn = np.linalg.norm(v)
        if vn > 0:
            v /= vn
            r[step:, step:] -= 2.0 * np.outer(v, v @ r[step:, step:])
    norms = np.sqrt(np.sum(r[k:, k:] ** 2, axis=0))
    n_ref = norms[cols.index(pos[int(want[k])]) - k]
    n_gpu = norms[cols.index(pos[int(got[k])]) - k]
    return abs(n_ref - n_gpu) / norms.max(), norms.max() / first


@pytest.mark.parametrize("name", CASES)
def test_ladder_residual_and_solution(name):
    hk, w, g, tree, knn, skels, op, f, b, xs = _run(name)
    ref = g["relres_ktilde"]
    got = np.array([np.linalg.norm(hk.hmatvec(op, xs[:, j], w.lam) - b[:, j]) / np.linalg.norm(b[:, j])
                    for j in range(2)])
    for j in range(2):
        assert ref[j] / RESID_FACTOR <= got[j] <= ref[j] * RESID_FACTOR, (name, j, got[j], ref[j])
    # x vs the reference's x: both solve the same Ktilde system; the
    # difference is bounded by the two solves' residuals times
    # ||(lam I + Ktilde)^-1|| <= 1 / lam_min -- measured far below; the bound
    # used is 1e-6 relative (C3's z_cond reaches 1e6)
    G = np.random.default_rng([0, 4242]).standard_normal((8, w.n))
    sk = G @ xs
    rel = np.linalg.norm(sk - g["x_sketch"]) / np.linalg.norm(g["x_sketch"])
    assert rel <= 1e-6, (name, rel)
    assert np.allclose(np.linalg.norm(xs, axis=0), g["x_norm"], rtol=1e-6)
    if "x0" in g:
        e0 = np.linalg.norm(xs[:, 0] - g["x0"]) / np.linalg.norm(g["x0"])
        assert e0 <= 1e-6, (name, e0)


@pytest.mark.parametrize("name", CASES)
def test_ladder_sampled_metrics(name):
    from paper_1701_02324_b200 import metrics as M
    hk, w, g, tree, knn, skels, op, f, b, xs = _run(name)
    assert np.array_equal(M.sample_rows(w.n, 256, 0), g["sampled_rows"])
    rep = M.sampled_error_report(op, f, b=b[:, 0], rows=256, seed=0)
    for key, ref in (("matvec_relerr_vs_K", float(g["sampled_matvec_relerr"])),
                     ("true_residual", float(g["sampled_true_residual"]))):
        assert ref / SAMPLED_FACTOR <= rep[key] <= ref * SAMPLED_FACTOR, (name, key, rep[key], ref)
    assert rep["residual_vs_Ktilde"] <= RESID_FACTOR * float(g["relres_ktilde"][0])
    u = hk.hmatvec(op, np.random.default_rng([0, 78]).standard_normal(w.n), w.lam)
    G = np.random.default_rng([0, 4242]).standard_normal((8, w.n))
    assert np.linalg.norm(G @ u - g["u_sketch"]) <= 1e-11 * np.linalg.norm(g["u_sketch"])


@pytest.mark.parametrize("name", [c for c in CASES if c.startswith("c5")])
def test_ladder_hybrid_iterations(name):
    from paper_1701_02324_b200.krylov import hybrid_solve
    hk, w, g, tree, knn, skels, op, f, b, xs = _run(name)
    xb, rep = hybrid_solve(op, f, b[:, 0], tol=w.gmres_tol, restart=w.gmres_restart)
    assert rep.iterations == int(g["hybrid_iterations"])
    G = np.random.default_rng([0, 4242]).standard_normal((8, w.n))
    rel = np.linalg.norm(G @ xb - g["hybrid_x_sketch"]) / np.linalg.norm(g["hybrid_x_sketch"])
    assert rel <= 1e-6, rel
