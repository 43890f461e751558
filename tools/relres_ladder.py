"""Residual growth with N: the GPU's ||(lam I + Ktilde) x - b|| / ||b|| and
sampled-row metrics for one configuration's generator / kernel / ranks at
N = 16384 ... full N, beside the reference's own values at the N it can run
(tests/golden/ladder_*.npz).  Prints one JSON line per N.

    python tools/relres_ladder.py C3 16384 65536 262144 1048576
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1701_02324_b200 as hk  # noqa: E402
from paper_1701_02324_b200 import metrics as M, workloads as W  # noqa: E402


def main(key, sizes):
    for n in sizes:
        w = W.CONFIGS[key].scaled(n)
        t0 = time.time()
        x = W.points(w, 0)
        kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
        tree = hk.build_tree(hk.PointSet(x), w.leaf_size, seed=0)
        knn = hk.knn_bruteforce(tree.points, w.kappa)
        cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented",
                                seed=0)
        sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
        op = hk.build_operator(tree, sk, kern)
        f = hk.factorize(op, w.lam)
        b = np.random.default_rng([0, 1000]).standard_normal((n, 2))
        rep = M.sampled_error_report(op, f, b=b[:, 0], rows=256, seed=0)
        zc = f.z_cond_per_level()
        out = {"workload": key, "n": n, "gpu": rep, "z_cond_max": max(zc.values()) if zc else None,
               "ranks_max": int(sk.ranks[1:].max()), "seconds": round(time.time() - t0, 1)}
        g = ROOT / "tests" / "golden" / f"ladder_{key.lower()}_n{n}.npz"
        if g.exists():
            z = np.load(g)
            out["reference"] = {"matvec_relerr_vs_K": float(z["sampled_matvec_relerr"]),
                                "true_residual": float(z["sampled_true_residual"]),
                                "residual_vs_Ktilde": float(z["relres_ktilde"][0]),
                                "z_cond_max": float(z["z_cond"].max())}
        print(json.dumps(out), flush=True)
        del f, op, sk, tree


if __name__ == "__main__":
    main(sys.argv[1], [int(v) for v in sys.argv[2:]] or [16384, 65536])
