"""Subtree-sharded path (paper_1701_02324_b200/sharded.py)
against the unsharded one on the same seed.

P ranks run as P processes sharing cuda:0 and meeting only in gloo
collectives staged through host memory (tests/sharded_worker.py); no
kernel waits on another rank.  With the same seed the sharded run must give
the unsharded run's kNN rows and skeleton index sets exactly, and its
solution / matvec to roundoff (the subtree and top plans issue the same
per-node descriptors as the full plan)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
import sharded_worker as W  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(tmp_path, world, **kw):
    port = _port()
    args = [f"--{k}={v}" for k, v in kw.items()]
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=str(ROOT))
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tests" / "sharded_worker.py"),
                                       f"--out={tmp_path}", *args], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]


def _reference(n, d, leaf, s, kappa, tau, h, lam, seed):
    import paper_1701_02324_b200 as hk
    x, b = W.instance(n, d, seed)
    tree = hk.build_tree(hk.PointSet(x), leaf, seed=seed)
    knn = hk.knn_bruteforce(tree.points, kappa)
    kern = hk.KernelSpec("gaussian", h=h, regularization=lam)
    cfg = hk.SkeletonConfig(tau=tau, max_rank=s, samples=4 * s, sample_mode="knn_augmented", seed=seed)
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    op = hk.build_operator(tree, sk, kern)
    f = hk.factorize(op, lam)
    bt = b[np.asarray(tree.perm)]
    xs = hk.solve_multi(f, bt, in_tree_order=True)
    u = np.stack([hk.hmatvec(op, bt[:, j], lam) for j in range(bt.shape[1])], axis=1)
    xh, rep = hk.hybrid_solve(op, f, bt[:, 0], tol=1e-9, max_iter=40, restart=5)
    xq = np.random.default_rng([seed, 99]).random((300, d))  # the worker's KRR test points
    return dict(tree=tree, knn=np.asarray(knn), sk=sk, x=xs, u=u, zc=f.z_cond_per_level(), xh=xh, rep=rep,
                predict=lambda w: hk.cross_predict(kern, xq, tree.points, w))


CASES = {
    # P = 2: shard roots at level 1, the top plan is the root alone
    "p1": dict(world=2, n=4096, d=5, leaf=128, s=32, kappa=8, tau=1e-300, h=0.9, lam=1e-2, seed=3),
    # P = 4: a skeletonized top level (row bitmaps OR-ed across shards)
    "p2": dict(world=4, n=6000, d=4, leaf=100, s=24, kappa=8, tau=1e-300, h=0.8, lam=1e-2, seed=5),
    # P = 4 with every shard a single leaf (subtree depth 0), adaptive ranks
    "leafshards": dict(world=4, n=1000, d=3, leaf=256, s=40, kappa=6, tau=1e-6, h=0.7, lam=1e-3, seed=7),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_matches_unsharded(tmp_path, case):
    cfg = dict(CASES[case])
    world = cfg.pop("world")
    ranks = _run(tmp_path, world, **cfg)
    ref = _reference(**cfg)
    tree, sk = ref["tree"], ref["sk"]
    nn = (1 << (tree.depth + 1)) - 1
    p = world.bit_length() - 1
    seen = set()
    for r, res in enumerate(ranks):
        b, e = int(res["begin"]), int(res["end"])
        assert (b, e) == (int(tree._begin[(1 << p) - 1 + r]), int(tree._end[(1 << p) - 1 + r]))
        np.testing.assert_array_equal(res["knn"], ref["knn"][b:e])
        for i in range(1, nn):
            key = f"skel_{i}"
            if key not in res:
                continue
            seen.add(i)
            np.testing.assert_array_equal(res[key], sk[i].indices, err_msg=f"rank {r} node {i}")
            if f"interp_{i}" in res:
                np.testing.assert_allclose(res[f"interp_{i}"], sk[i].interp, rtol=0, atol=1e-9 * max(
                    1.0, np.abs(sk[i].interp).max()), err_msg=f"rank {r} node {i}")
        xr = ref["x"][b:e].T
        np.testing.assert_allclose(res["x"], xr, rtol=0, atol=1e-11 * np.abs(ref["x"]).max())
        np.testing.assert_array_equal(res["x"], res["x2"])
        np.testing.assert_allclose(res["u"], ref["u"][b:e].T, rtol=0, atol=1e-12 * np.abs(ref["u"]).max())
        np.testing.assert_allclose(res["xfull"], ref["x"].T, rtol=0, atol=1e-11 * np.abs(ref["x"]).max())
        # hybrid GMRES over the shards: same iterations, same solution
        assert int(res["h_iters"]) == ref["rep"].iterations
        # Givens estimates agree; the last entry is the recomputed true
        # residual (krylov.py:131-139), a roundoff-level number below the
        # 1e-9 tolerance in both runs
        np.testing.assert_allclose(res["h_res"][:-1], ref["rep"].residuals[:-1], rtol=0.5, atol=1e-13)
        assert res["h_res"][-1] <= 1e-9 and ref["rep"].residuals[-1] <= 1e-9
        np.testing.assert_allclose(res["xh"], ref["xh"][b:e], rtol=0, atol=1e-10 * np.abs(ref["xh"]).max())
        # per-level z_cond: top levels identical on every rank, shard levels bounded by the global max
        for lev, z in zip(res["zc_levels"], res["zc"]):
            assert z <= ref["zc"][int(lev)] * (1 + 1e-8) + 1e-12
            if lev < p:
                assert z == pytest.approx(ref["zc"][int(lev)], rel=1e-8)
        # KRR predict over the training shards (partials summed in rank order): identical on every
        # rank, equal to the unsharded prediction up to the summation order
        # (same weights: the gathered sharded solution; |K| <= 1, so the bound scales with sum |w|)
        w = ranks[0]["xfull"][0]
        np.testing.assert_array_equal(res["pred"], ranks[0]["pred"])
        np.testing.assert_allclose(res["pred"], ref["predict"](w), rtol=0, atol=1e-14 * np.abs(w).sum())
    assert seen == set(range(1, nn)), "some skeletons were produced by no rank"
