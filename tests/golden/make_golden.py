"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container only (it imports ``/root/reference/pkg/src``
read-only; nothing at test time needs the reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each instance is run through the reference's public API exactly as
``cli._build_stage`` / ``_factorize_stage`` do (cli.py:188-305) and the
results are frozen as ``tests/golden/<name>.npz``.  Large float arrays are
stored as sketches (projections on fixed Gaussian vectors) to keep the
fixtures small; integer structure (perm, kNN, skeleton indices, ranks, row
counts) is stored in full so the bit-exact claims are checked in full.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import hikersolve as hk  # noqa: E402  (the reference, read-only)
from hikersolve.data import PointSet  # noqa: E402

from paper_1701_02324_b200 import workloads  # noqa: E402


def sketch_vec(tag, node, n):
    return np.random.default_rng([tag, node]).standard_normal(n)


def coords_digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def run_instance(name, coords, kernel, leaf, tau, max_rank, samples, mode, seed,
                 kappa=None, nrhs=2, store_coords=True, hybrid=False):
    t0 = time.time()
    ps = PointSet(coords)
    tree = hk.build_tree(ps, leaf, seed=seed)
    knn = hk.knn_bruteforce(tree.points, kappa) if mode == "knn_augmented" else None
    cfg = hk.SkeletonConfig(tau=tau, max_rank=max_rank, samples=samples,
                            sample_mode=mode, seed=seed)
    skels = hk.build_skeletons(tree, kernel, cfg, knn=knn, threads=8)
    op = hk.build_operator(tree, skels, kernel)
    lam = kernel.regularization
    f = hk.factorize(op, lam, threads=8)
    n = tree.n
    rng = np.random.default_rng([seed, 1000])
    b = rng.standard_normal((n, nrhs))
    x = hk.solve_multi(f, b, in_tree_order=True)
    w = np.random.default_rng([seed, 78]).standard_normal(n)
    u = hk.hmatvec(op, w, lam)

    nn = len(tree.nodes)
    ranks = np.full(nn, -1, dtype=np.int64)
    rows_count = np.full(nn, -1, dtype=np.int64)
    skel_idx, skel_off = [], [0]
    interp_sk, theta_sk = [], []
    interp_fro = np.zeros(nn)
    theta_fro = np.zeros(nn)
    z_cond = np.zeros(nn)
    for nd in tree.nodes:
        i = nd.index
        fac = f.factors[i]
        if nd.level > 0:
            s = skels[i]
            ranks[i] = s.rank
            skel_idx.append(np.asarray(s.indices, dtype=np.int64))
            interp_sk.append(s.interp @ sketch_vec(77, i, s.interp.shape[1]))
            interp_fro[i] = np.linalg.norm(s.interp)
            rows_count[i] = hk.skeleton.sample_rows(
                tree, nd, samples, mode, seed, knn=knn).size
            theta_sk.append(fac.theta @ sketch_vec(78, i, fac.theta.shape[1]))
            theta_fro[i] = np.linalg.norm(fac.theta)
        else:
            skel_idx.append(np.zeros(0, dtype=np.int64))
        skel_off.append(skel_off[-1] + skel_idx[-1].size)
        if not nd.is_leaf:
            z_cond[i] = fac.z_cond
    out = {
        "perm": np.asarray(tree.perm, dtype=np.int64),
        "split_value": np.array([nd.split_value if nd.split_value is not None else np.nan
                                 for nd in tree.nodes]),
        "ranks": ranks,
        "rows_count": rows_count,
        "skel_idx": np.concatenate(skel_idx),
        "skel_off": np.asarray(skel_off, dtype=np.int64),
        "interp_sketch": np.concatenate(interp_sk) if interp_sk else np.zeros(0),
        "interp_fro": interp_fro,
        "theta_sketch": np.concatenate(theta_sk) if theta_sk else np.zeros(0),
        "theta_fro": theta_fro,
        "z_cond": z_cond,
        "x": x,
        "u": u,
        "coords_sha256": np.array(coords_digest(coords)),
    }
    if knn is not None:
        out["knn"] = np.asarray(knn, dtype=np.int64)
    if store_coords:
        out["coords"] = np.asarray(coords, dtype=np.float64)
    if hybrid:
        xb, rep = hk.hybrid_solve(op, f, b[:, 0], tol=1e-10, restart=50,
                                  operator_mode="compressed")
        out["hybrid_x"] = xb
        out["hybrid_iterations"] = np.array(rep.iterations)
        out["hybrid_final_residual"] = np.array(rep.final_residual)
    meta = {"name": name, "family": kernel.family, "h": kernel.h,
            "degree": kernel.degree, "shift": kernel.shift, "lam": lam,
            "leaf": leaf, "tau": tau, "max_rank": max_rank, "samples": samples,
            "mode": mode, "seed": seed, "kappa": kappa, "nrhs": nrhs, "n": n,
            "d": int(coords.shape[1]), "depth": tree.depth,
            "seconds": round(time.time() - t0, 2)}
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, meta["seconds"], "s; ranks", sorted(set(ranks.tolist())))


def workload_instance(key, n, nrhs=2, store_coords=False, hybrid=False):
    w = workloads.CONFIGS[key].scaled(n)
    coords = workloads.points(w, 0)
    kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    run_instance(f"{key.lower()}_n{n}", coords, kern, w.leaf_size, w.tau,
                 w.max_rank, w.samples, "knn_augmented", 0, kappa=w.kappa,
                 nrhs=nrhs, store_coords=store_coords, hybrid=hybrid)


def ladder_instance(key, n, hybrid=False):
    """Reduced-N ladder fixture (N = 16384 and 65536, the
    reference's kNN guard allows no more).  Integer structure in full
    (perm, skeleton indices, ranks) or as a SHA-256 of the full array plus
    its first rows (kNN); float outputs as norms / sketches / the reference's
    own accuracy metrics:
      relres_ktilde  ||(lam I + Ktilde) x - b|| / ||b|| through the
                     reference's hmatvec (treecode.py:92-128);
      sampled_*      256 rows R = default_rng([seed, 77]) of the exact
                     K + lam I from the reference's eval_block
                     (kernels.py:64-105) against all n columns: the matvec
                     error of its u = hmatvec(w), w = default_rng([seed, 78]),
                     and the true residual of its x (b column 0).
    The thread count (8) does not change any result (test_solver.py:211-219)."""
    t0 = time.time()
    w = workloads.CONFIGS[key].scaled(n)
    coords = workloads.points(w, 0)
    kernel = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
    seed, lam = 0, w.lam
    tree = hk.build_tree(PointSet(coords), w.leaf_size, seed=seed)
    t_tree = time.time()
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    t_knn = time.time()
    cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples,
                            sample_mode="knn_augmented", seed=seed)
    skels = hk.build_skeletons(tree, kernel, cfg, knn=knn, threads=8)
    t_sk = time.time()
    op = hk.build_operator(tree, skels, kernel)
    f = hk.factorize(op, lam, threads=8)
    t_f = time.time()
    b = np.random.default_rng([seed, 1000]).standard_normal((n, 2))
    x = hk.solve_multi(f, b, in_tree_order=True)
    t_s = time.time()
    wv = np.random.default_rng([seed, 78]).standard_normal(n)
    u = hk.hmatvec(op, wv, lam)
    relres = [float(np.linalg.norm(hk.hmatvec(op, x[:, j], lam) - b[:, j]) / np.linalg.norm(b[:, j]))
              for j in range(2)]
    xt = tree.points.coords
    R = np.sort(np.random.default_rng([seed, 77]).choice(n, size=256, replace=False))
    KR = hk.eval_block(kernel, xt[R], xt)
    kw = KR @ wv
    s_mv = float(np.linalg.norm((u[R] - lam * wv[R]) - kw) / np.linalg.norm(kw))
    s_res = float(np.linalg.norm(KR @ x[:, 0] + lam * x[R, 0] - b[R, 0]) / np.linalg.norm(b[R, 0]))
    nn = len(tree.nodes)
    ranks = np.full(nn, -1, dtype=np.int64)
    z_cond = np.zeros(nn)
    theta_fro = np.zeros(nn)
    skel_idx, skel_off = [], [0]
    for nd in tree.nodes:
        i = nd.index
        if nd.level > 0:
            ranks[i] = skels[i].rank
            skel_idx.append(np.asarray(skels[i].indices, dtype=np.int32))
            theta_fro[i] = np.linalg.norm(f.factors[i].theta)
        else:
            skel_idx.append(np.zeros(0, dtype=np.int32))
        skel_off.append(skel_off[-1] + skel_idx[-1].size)
        if not nd.is_leaf:
            z_cond[i] = f.factors[i].z_cond
    G = np.random.default_rng([seed, 4242]).standard_normal((8, n))
    knn64 = np.ascontiguousarray(np.asarray(knn, dtype=np.int64))
    out = {
        "perm": np.asarray(tree.perm, dtype=np.int32),
        "knn_sha256": np.array(hashlib.sha256(knn64.tobytes()).hexdigest()),
        "knn_head": knn64[:256],
        "ranks": ranks, "z_cond": z_cond, "theta_fro": theta_fro,
        "skel_idx": np.concatenate(skel_idx), "skel_off": np.asarray(skel_off, dtype=np.int64),
        "x_norm": np.linalg.norm(x, axis=0), "x_sketch": G @ x, "u_norm": np.array(np.linalg.norm(u)),
        "u_sketch": G @ u, "relres_ktilde": np.array(relres), "sampled_rows": R,
        "sampled_matvec_relerr": np.array(s_mv), "sampled_true_residual": np.array(s_res),
        "coords_sha256": np.array(coords_digest(coords)),
    }
    if n <= 16384:
        out["x0"] = x[:, 0].copy()
    if hybrid:
        xb, rep = hk.hybrid_solve(op, f, b[:, 0], tol=w.gmres_tol, restart=w.gmres_restart,
                                  operator_mode="compressed")
        out["hybrid_iterations"] = np.array(rep.iterations)
        out["hybrid_final_residual"] = np.array(rep.final_residual)
        out["hybrid_x_norm"] = np.array(np.linalg.norm(xb))
        out["hybrid_x_sketch"] = G @ xb
    meta = {"name": f"{key.lower()}_n{n}", "workload": key, "n": n, "lam": lam, "seed": seed,
            "depth": tree.depth, "threads": 8,
            "seconds": {"tree": round(t_tree - t0, 2), "knn": round(t_knn - t_tree, 2),
                        "skeletons": round(t_sk - t_knn, 2), "factorize": round(t_f - t_sk, 2),
                        "solve2": round(t_s - t_f, 2), "total": round(time.time() - t0, 2)}}
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(HERE / f"ladder_{key.lower()}_n{n}.npz", **out)
    print(meta["name"], meta["seconds"], "ranks", sorted(set(ranks.tolist()))[:3], "...",
          max(ranks.tolist()), "relres", relres, "sampled", s_mv, s_res, flush=True)


def main(which):
    if "frozen" in which:
        ps = hk.generate("uniform_cube", 1024, 3, d=3)
        kern = hk.KernelSpec("gaussian", h=0.3, regularization=1e-2)
        run_instance("frozen_n1024", ps.coords, kern, 256, 1e-7, 384, 256,
                     "exact", 3, hybrid=True)
    if "tiny" in which:
        ps = hk.generate("uniform_cube", 10, 0, d=2)
        run_instance("tiny_n10", ps.coords, hk.KernelSpec("gaussian", h=0.5),
                     5, 1e-7, 64, 256, "exact", 0)
        ps = hk.generate("uniform_cube", 128, 3, d=2)
        run_instance("rank0_n128", ps.coords,
                     hk.KernelSpec("gaussian", h=1e-9, regularization=1e-1),
                     32, 1e-4, 8, 256, "exact", 0)
    if "families" in which:
        base = hk.generate("uniform_cube", 1024, 11, d=3)
        run_instance("laplace_n1024", base.coords * 2.0,
                     hk.KernelSpec("laplace3d", regularization=1e-1), 128, 1e-8,
                     64, 256, "uniform", 11)
        run_instance("poly_n1024", base.coords * 0.05,
                     hk.KernelSpec("polynomial", degree=2, shift=0.02,
                                   regularization=1e-3), 128, 1e-8, 64, 256,
                     "uniform", 11)
        run_instance("gauss_uniform_n2000", hk.generate("uniform_cube", 2000, 5, d=4).coords,
                     hk.KernelSpec("gaussian", h=0.4, regularization=1e-2), 100, 1e-6,
                     48, 96, "uniform", 5)
    if "c1" in which:
        workload_instance("C1", 4096, nrhs=4, store_coords=True, hybrid=True)
    if "c2" in which:
        workload_instance("C2", 8192)
    if "c3" in which:
        workload_instance("C3", 8192)
    if "c4" in which:
        workload_instance("C4", 8192)
    if "c5" in which:
        workload_instance("C5", 2048, hybrid=True)
    for key, n in (("C2", 16384), ("C3", 16384), ("C4", 16384), ("C5", 16384),
                   ("C2", 65536), ("C3", 65536), ("C4", 65536)):
        if f"ladder_{key.lower()}_{n}" in which or "ladder" in which:
            ladder_instance(key, n, hybrid=key == "C5")
    if "report_schema" in which:
        import importlib.util  # the reference's own schema (tests/helpers.py:145-177)
        spec = importlib.util.spec_from_file_location("ref_helpers", "/root/reference/pkg/tests/helpers.py")
        mod = importlib.util.module_from_spec(spec)
        sys.modules["ref_helpers"] = mod
        spec.loader.exec_module(mod)
        (HERE / "report_schema.json").write_text(json.dumps(mod.REPORT_SCHEMA, indent=1) + "\n")
    if "knn_small" in which:
        rng = np.random.default_rng(0)
        pts = rng.random((200, 3))
        np.savez_compressed(HERE / "knn_n200.npz", coords=pts,
                            knn=hk.knn_bruteforce(PointSet(pts), 5))
    if "gmres" in which:
        ps = hk.generate("uniform_cube", 512, 3, d=3)
        kern = hk.KernelSpec("gaussian", h=0.5, regularization=1e-6)
        tree = hk.build_tree(ps, 512, seed=3)
        from hikersolve import oracle as ref_oracle
        dense = ref_oracle.dense_kernel_matrix(kern, tree.points, 1e-6)
        b = np.random.default_rng([3, 41]).standard_normal(512)
        x, rep = hk.gmres(lambda v: dense @ v, lambda v: v, b, tol=1e-8,
                          max_iter=500, restart=50)
        np.savez_compressed(HERE / "gmres_n512.npz", x=x,
                            iterations=np.array(rep.iterations),
                            converged=np.array(rep.converged),
                            final_residual=np.array(rep.final_residual),
                            residuals=np.array(rep.residuals))
    if "qr" in which:
        rng = np.random.default_rng(1)
        cases = {}
        for t in range(12):
            m, n = int(rng.integers(5, 60)), int(rng.integers(5, 60))
            u, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
            v, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
            a = (u * 0.6 ** np.arange(min(m, n))) @ v.T
            tol, mr = [1e-3, 1e-8, 1e-12][t % 3], int(rng.integers(1, 40))
            cols, p = hk.interpolative_decomposition(a, tol, mr)
            cases[f"a{t}"] = a
            cases[f"cols{t}"] = np.asarray(cols, dtype=np.int64)
            cases[f"p{t}"] = p
            cases[f"tol{t}"] = np.array([tol, mr])
        np.savez_compressed(HERE / "id_cases.npz", **cases)


if __name__ == "__main__":
    main(sys.argv[1:] or ["frozen", "tiny", "families", "c1", "c2", "c3", "c4",
                          "c5", "knn_small", "qr", "gmres"])
