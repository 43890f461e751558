"""Full-size structure parity: at C2's full N = 262144 the GPU tree
permutation and exact kNN lists -- and at C3's N = 1,048,576 the permutation
and the lists of 4096 sampled query rows -- equal the CPU oracle's bit for bit
(SHA-256 of the int64 arrays, tests/golden/full_c2_digest.json made by
tools/make_full_digests.py).  The oracle is the reference's algorithm
(tree.py:87-144, 163-188), pinned to the unmodified reference up to the
reference's own kNN limit of 65536 points (tests/test_gpu_ladder.py,
tests/test_oracle_golden.py); near-ties between distances first become
likely at this size."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem[len("full_"):-len("_digest")] for p in GOLDEN.glob("full_*_digest.json"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", CASES)
def test_full_size_perm_and_knn(name):
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import workloads as W
    g = json.loads((GOLDEN / f"full_{name}_digest.json").read_text())
    w = W.CONFIGS[g["workload"]]
    x = W.points(w, 0)
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["coords_sha256"]
    tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
    perm = np.asarray(tree.perm)
    assert perm[:64].tolist() == g["perm_head"]
    assert _sha(perm) == g["perm_sha256"]
    knn = np.asarray(hk.knn_bruteforce(tree.points, w.kappa))
    if "knn_sha256" in g:
        assert knn[:64].tolist() == g["knn_head"]
        assert _sha(knn) == g["knn_sha256"]
    else:  # N = 1M: the oracle's lists of a seeded sample of query rows (each against all N points)
        rows = np.asarray(g["knn_sample_rows"], dtype=np.int64)
        assert knn[rows[:8]].tolist() == g["knn_sample_head"]
        assert _sha(knn[rows]) == g["knn_sample_sha256"]


SKEL_CASES = sorted(p.stem[len("full_"):-len("_skeletons")] for p in GOLDEN.glob("full_*_skeletons.json"))


@pytest.mark.parametrize("name", SKEL_CASES)
def test_full_size_skeleton_subtree(name):
    """Skeleton index sets of one depth-2 subtree at the configuration's full
    N (tools/make_full_skeleton_digest.py: the oracle's skeleton.py:84-182 /
    linalg.py:43-136 on the sampled blocks themselves) against the GPU path,
    whose blocks of 3.3 k - 9 k rows go through the tall-skinny QR
    pre-reduction (csrc/tsqr.cu) before the pivoting: same row counts, same
    ranks, same pivot order."""
    import os
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import workloads as W
    g = json.loads((GOLDEN / f"full_{name}_skeletons.json").read_text())
    w = W.CONFIGS[g["workload"]]
    if (w.n > (1 << 21) or w.d > 64) and not os.environ.get("HKS_TEST_FULL_LARGE"):
        pytest.skip("minutes of setup at this size: set HKS_TEST_FULL_LARGE=1 (result recorded under profiles/)")
    x = W.points(w, 0)
    kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    for node, ref in g["nodes"].items():
        i = int(node)
        assert int(sk.rows_count[i]) == ref["rows"], node
        assert np.array_equal(np.asarray(sk[i].indices), np.asarray(ref["indices"], dtype=np.int64)), node
    # the subtree's factorization against the oracle's (solver.py:111-186 on
    # the same seven nodes; it depends on nothing outside the subtree):
    # theta of every node and push of the internal ones by norm, the subtree
    # root's theta / push by 8 Gaussian sketches, to the tolerance of the
    # reduced-N parity tests (1e-8, scaled by the node's z_cond where the
    # reduced system amplifies roundoff), and LAPACK's condition estimate
    fx = GOLDEN / f"full_{name}_factor.npz"
    if not fx.exists():
        return
    z = np.load(fx)
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, float(z["lam"]))
    root = int(g["subtree_root"])
    for node in g["nodes"]:
        i = int(node)
        nf = f.factors[i]
        tol = 1e-8 * max(1.0, float(z[f"z_cond_{i}"]) / 1e4) if f"z_cond_{i}" in z else 1e-8
        ref = float(z[f"theta_norm_{i}"])
        assert abs(np.linalg.norm(nf.theta) - ref) <= tol * ref, node
        if f"z_cond_{i}" in z:
            pref = float(z[f"push_norm_{i}"])
            assert abs(np.linalg.norm(nf.child_push) - pref) <= tol * pref, node
            assert abs(nf.z_cond - float(z[f"z_cond_{i}"])) <= 1e-3 * float(z[f"z_cond_{i}"]), node
    if "upward_root" in z:  # treecode upward pass of a weight vector supported on the subtree
        b0, e0 = int(tree._begin[root]), int(tree._end[root])
        wv = np.zeros(w.n)
        wv[b0:e0] = np.random.default_rng([31, root]).standard_normal(e0 - b0)
        up = hk.upward_pass(op, wv)[root]
        assert np.linalg.norm(up - z["upward_root"]) <= 1e-8 * np.linalg.norm(z["upward_root"])
    nf = f.factors[root]
    gs = np.random.default_rng([29, root]).standard_normal((nf.theta.shape[1], 8))
    tol = 1e-8 * max(1.0, float(z[f"z_cond_{root}"]) / 1e4)
    for got, key in ((nf.theta @ gs, "theta_root_sketch"), (nf.child_push @ gs, "push_root_sketch")):
        assert np.linalg.norm(got - z[key]) <= tol * np.linalg.norm(z[key]), key
