"""One rank of a sharded run (tests/test_gpu_sharded.py launches P of these
on one GPU with the gloo backend: the ranks only meet in host-side
collectives, no kernel waits on another rank).  Writes the rank's results
to <out>/rank<r>.npz for the parent to compare with the unsharded path."""

import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def instance(n, d, seed):
    rng = np.random.default_rng([seed, 0])
    centers = rng.standard_normal((4, d))
    lab = rng.integers(0, 4, n)
    x = centers[lab] + 0.4 * rng.standard_normal((n, d))
    b = np.random.default_rng([seed, 1]).standard_normal((n, 3))
    return x, b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--d", type=int, default=5)
    ap.add_argument("--leaf", type=int, default=128)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--kappa", type=int, default=8)
    ap.add_argument("--tau", type=float, default=1e-300)
    ap.add_argument("--h", type=float, default=0.9)
    ap.add_argument("--lam", type=float, default=1e-2)
    ap.add_argument("--seed", type=int, default=3)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist
    import paper_1701_02324_b200 as hk
    from paper_1701_02324_b200 import sharded as S

    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    comm = S.ShardComm()
    x, b = instance(a.n, a.d, a.seed)
    tree = hk.build_tree(hk.PointSet(x), a.leaf, seed=a.seed)
    spec = S.ShardSpec(a.n, tree.depth, comm.world, comm.rank)
    knn = S.knn_shard(tree, a.kappa, spec)
    kern = hk.KernelSpec("gaussian", h=a.h, regularization=a.lam)
    cfg = hk.SkeletonConfig(tau=a.tau, max_rank=a.s, samples=4 * a.s, sample_mode="knn_augmented", seed=a.seed)
    sk = S.build_skeletons_sharded(tree, kern, cfg, knn, spec, comm)
    op = S.build_operator_sharded(tree, sk, kern, comm)
    res = {"knn": knn.cpu().numpy(), "begin": spec.begin, "end": spec.end}
    try:
        f = S.factorize_sharded(op, a.lam)
    except Exception as exc:  # noqa: BLE001 -- reported to the parent
        res["error"] = f"{type(exc).__name__}: {exc}"
        np.savez(os.path.join(a.out, f"rank{comm.rank}.npz"), **res)
        dist.destroy_process_group()
        return
    bt = b[np.asarray(tree.perm)]
    B = torch.from_numpy(np.ascontiguousarray(bt[spec.begin: spec.end].T)).cuda()
    X = S.solve_sharded(f, B)
    X2 = S.solve_sharded(f, B)  # graph replay
    U = S.hmatvec_sharded(op, B, a.lam)
    full = S.gather_rows(comm, spec, X)
    from paper_1701_02324_b200.krylov import hybrid_solve_sharded
    xh, rep = hybrid_solve_sharded(op, f, B[0], tol=1e-9, max_iter=40, restart=5)
    res.update(xh=xh.cpu().numpy(), h_iters=rep.iterations, h_res=np.array(rep.residuals),
               h_final=rep.final_residual)
    xq = np.random.default_rng([a.seed, 99]).random((300, a.d))  # KRR test points
    res["pred"] = S.cross_predict_sharded(kern, xq, op, X[0]).cpu().numpy()
    res.update(x=X.cpu().numpy(), x2=X2.cpu().numpy(), u=U.cpu().numpy(), xfull=full.cpu().numpy())
    for i in range(1, (1 << (tree.depth + 1)) - 1):
        if i in sk:
            s_ = sk[i]
            res[f"skel_{i}"] = s_.indices
            if s_.interp.size:
                res[f"interp_{i}"] = s_.interp
    zc = f.z_cond_per_level()
    res["zc_levels"] = np.array(sorted(zc))
    res["zc"] = np.array([zc[k] for k in sorted(zc)])
    res["level_seconds"] = np.array([f.level_seconds[k] for k in sorted(f.level_seconds)])
    np.savez(os.path.join(a.out, f"rank{comm.rank}.npz"), **{k: np.asarray(v) for k, v in res.items()})
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
