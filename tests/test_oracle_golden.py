"""Pin the CPU oracle (oracle/hks_oracle.py) to the reference's own outputs.

The golden fixtures were produced by running the unmodified reference
(tests/golden/make_golden.py).  Integer structure must match bit for bit;
floating-point arrays to roundoff (the oracle calls the same numpy / LAPACK
routines in the same order, so the tolerances here are tight).
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import hks_oracle as O
from golden_cases import (ALL_CASES, GOLDEN, coords_for, kern_of, load,
                          matvec_w, oracle_instance, rhs_for, sketch_vec,
                          skel_list)

CASES = ALL_CASES


@pytest.mark.parametrize("name", CASES)
def test_coords_regenerate_bitwise(name):
    import hashlib
    g = load(name)
    x = coords_for(name)
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == str(g["coords_sha256"])


@pytest.mark.parametrize("name", CASES)
def test_tree_perm_and_splits_exact(name):
    g = load(name)
    inst = oracle_instance(name)
    t = inst["tree"]
    assert np.array_equal(t.perm, g["perm"])
    # The split value is a BLAS dot product inside the power iteration
    # (tree.py:70-84); its last bits follow the BLAS thread count, so it is
    # compared to 1e-12 relative while the permutation stays bit-exact.
    for i, v in t.split_val.items():
        assert v == pytest.approx(float(g["split_value"][i]), rel=1e-12, abs=1e-15)
    assert t.depth == g["meta"]["depth"]


@pytest.mark.parametrize("name", [c for c in CASES if load(c)["meta"]["mode"] == "knn_augmented"])
def test_knn_exact(name):
    g = load(name)
    assert np.array_equal(oracle_instance(name)["knn"], g["knn"])


def test_knn_small_and_ties():
    z = np.load(GOLDEN / "knn_n200.npz")
    assert np.array_equal(O.knn(z["coords"], 5), z["knn"])
    # exact duplicates: ties go to the lower index (tests/test_tree.py:121-127)
    pts = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 0.0], [0.0, 1.0], [5.0, 5.0]])
    nb = O.knn(pts, 2)
    assert list(nb[0]) == [1, 2]


@pytest.mark.parametrize("name", CASES)
def test_skeletons_exact(name):
    g = load(name)
    inst = oracle_instance(name)
    skel, rows = inst["skel"], inst["rows"]
    for i, (idx, p) in skel.items():
        assert np.array_equal(idx, skel_list(g, i)), f"node {i}"
        assert idx.size == g["ranks"][i]
        assert rows[i].size == g["rows_count"][i]


@pytest.mark.parametrize("name", CASES)
def test_interp_and_theta_sketches(name):
    g = load(name)
    inst = oracle_instance(name)
    skel, fac = inst["skel"], inst["fac"]
    at_i = at_t = 0
    for i in sorted(skel):
        p = skel[i][1]
        r = p.shape[0]
        si = p @ sketch_vec(77, i, p.shape[1])
        ref = g["interp_sketch"][at_i:at_i + r]
        at_i += r
        assert np.linalg.norm(si - ref) <= 1e-9 * max(np.linalg.norm(ref), 1.0)
        th = fac[i]["theta"]
        st = th @ sketch_vec(78, i, th.shape[1])
        reft = g["theta_sketch"][at_t:at_t + th.shape[0]]
        at_t += th.shape[0]
        assert np.linalg.norm(st - reft) <= 1e-7 * max(np.linalg.norm(reft), 1e-300)
    for i, f in fac.items():
        if "z_cond" in f:
            assert f["z_cond"] == pytest.approx(g["z_cond"][i], rel=1e-6)


@pytest.mark.parametrize("name", CASES)
def test_solve_and_matvec(name):
    g = load(name)
    m = g["meta"]
    inst = oracle_instance(name)
    t = inst["tree"]
    b = rhs_for(m)
    x = np.stack([O.solve(t, inst["skel"], inst["coup"], inst["fac"], b[:, j])
                  for j in range(b.shape[1])], axis=1)
    assert np.linalg.norm(x - g["x"]) <= 1e-7 * np.linalg.norm(g["x"])
    u = O.matvec(t, inst["skel"], inst["leaf"], inst["coup"], matvec_w(m), m["lam"])
    assert np.linalg.norm(u - g["u"]) <= 1e-12 * np.linalg.norm(g["u"])


def test_interpolative_decomposition_cases():
    z = np.load(GOLDEN / "id_cases.npz")
    for t in range(12):
        tol, mr = z[f"tol{t}"]
        cols, p = O.interp_decomp(z[f"a{t}"], tol, int(mr))
        assert np.array_equal(cols, z[f"cols{t}"])
        assert np.allclose(p, z[f"p{t}"], rtol=1e-10, atol=1e-12)
        assert np.array_equal(p[:, cols], np.eye(cols.size))


def test_gmres_unpreconditioned_golden():
    z = np.load(GOLDEN / "gmres_n512.npz")
    tree = O.build_tree(np.random.default_rng([3, 0, 0]).random((512, 3)), 512, 3)
    dense = O.kernel_block("gaussian", tree.coords, tree.coords, h=0.5)
    dense[np.diag_indices(512)] += 1e-6
    b = np.random.default_rng([3, 41]).standard_normal(512)
    x, rep = O.gmres(lambda v: dense @ v, lambda v: v, b, tol=1e-8, max_iter=500, restart=50)
    assert rep["iterations"] == int(z["iterations"])
    assert rep["converged"] == bool(z["converged"])
    assert rep["final_residual"] == pytest.approx(float(z["final_residual"]), rel=1e-6)


def test_gmres_identity_one_iteration_no_alias():
    # SPEC.md:462 contract; the reference's in-place update aliases basis[0]
    b = np.random.default_rng(0).standard_normal(32)
    x, rep = O.gmres(lambda v: v, lambda v: v, b, tol=1e-12)
    assert rep["iterations"] == 1 and rep["converged"]
    assert np.allclose(x, b, atol=1e-12)


@pytest.mark.parametrize("name", ["frozen_n1024", "c1_n4096", "c5_n2048"])
def test_hybrid_golden(name):
    g = load(name)
    m = g["meta"]
    inst = oracle_instance(name)
    t, sk, lf, cp, fac = inst["tree"], inst["skel"], inst["leaf"], inst["coup"], inst["fac"]
    b = rhs_for(m)[:, 0]
    x, rep = O.gmres(lambda v: O.matvec(t, sk, lf, cp, v, m["lam"]),
                     lambda v: O.solve(t, sk, cp, fac, v), b, tol=1e-10, restart=50)
    assert rep["iterations"] == int(g["hybrid_iterations"])
    assert np.linalg.norm(x - g["hybrid_x"]) <= 1e-7 * np.linalg.norm(g["hybrid_x"])


@pytest.mark.parametrize("name", ["c2_n16384", "c3_n16384", "c4_n16384"])
def test_oracle_tree_knn_vs_ladder_fixture(name):
    """The oracle's tree permutation and exact kNN lists equal the
    unmodified reference's on the N = 16384 ladder instances
    (tests/golden/ladder_*.npz; tree.py:87-144, 163-188)."""
    import hashlib
    import json
    from paper_1701_02324_b200 import workloads as W
    z = np.load(GOLDEN / f"ladder_{name}.npz")
    meta = json.loads(str(z["meta"]))
    w = W.CONFIGS[meta["workload"]].scaled(meta["n"])
    tree = O.build_tree(W.points(w, 0), w.leaf_size, 0)
    assert np.array_equal(tree.perm, z["perm"].astype(np.int64))
    nl = O.knn(tree.coords, w.kappa)
    assert hashlib.sha256(np.ascontiguousarray(nl, dtype=np.int64).tobytes()).hexdigest() == str(z["knn_sha256"])


def test_knn_rows_equals_knn_table():
    """oracle.knn_rows (full-size spot checks, tools/make_full_digests.py) is
    the row-restricted oracle.knn: same lists on the reference-pinned table."""
    from oracle import hks_oracle as O
    rng = np.random.default_rng(4)
    x = rng.random((3000, 5))
    full = O.knn(x, 9)
    rows = np.sort(rng.choice(3000, size=400, replace=False))
    assert np.array_equal(O.knn_rows(x, 9, rows, chunk=64), full[rows])


def test_full_size_fixtures_well_formed():
    """The full-size fixtures of tests/test_gpu_full_structure.py (made by
    tools/make_full_digests.py / make_full_skeleton_digest.py from the
    oracle): consistent sizes, skeleton indices inside their candidates'
    ranges, nested parents, finite factor quantities."""
    import json
    from oracle import hks_oracle as O
    from paper_1701_02324_b200 import workloads as W
    golden = Path(__file__).resolve().parent / "golden"
    for key in ("c2", "c3", "c4", "c5"):
        s = json.loads((golden / f"full_{key}_skeletons.json").read_text())
        w = W.CONFIGS[s["workload"]]
        assert s["n"] == w.n
        if (golden / f"full_{key}_digest.json").exists():
            d = json.loads((golden / f"full_{key}_digest.json").read_text())
            assert d["workload"] == s["workload"] and d["n"] == w.n and len(d["perm_head"]) == 64
        depth = O.tree_depth(w.n, w.leaf_size)
        begin, end = O.node_ranges(w.n, depth)
        first_leaf = (1 << depth) - 1
        g = s["subtree_root"]
        assert sorted(int(k) for k in s["nodes"]) == sorted([g, 2 * g + 1, 2 * g + 2] + [4 * g + 3 + j for j in range(4)])
        for node, rec in s["nodes"].items():
            i = int(node)
            idx = np.asarray(rec["indices"])
            assert 0 < idx.size <= w.max_rank and np.unique(idx).size == idx.size
            assert idx.min() >= begin[i] and idx.max() < end[i] and rec["rows"] >= w.samples
            if i < first_leaf:
                kids = set(s["nodes"][str(2 * i + 1)]["indices"]) | set(s["nodes"][str(2 * i + 2)]["indices"])
                assert set(rec["indices"]) <= kids
        z = np.load(golden / f"full_{key}_factor.npz")
        assert float(z["lam"]) == w.lam
        assert all(np.all(np.isfinite(z[k])) for k in z.files)
        assert z["theta_root_sketch"].shape[1] == 8 and z["upward_root"].shape == (len(s["nodes"][str(g)]["indices"]),)
