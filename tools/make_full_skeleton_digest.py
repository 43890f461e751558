"""Full-size skeleton fixtures from the CPU oracle (test infrastructure): the
skeleton index sets of one depth-2 subtree (4 leaves, their 2 parents and
the grandparent) of a BASELINE configuration at its full N, for
tests/test_gpu_full_structure.py.  Only the kNN rows those nodes sample from
are computed (oracle knn_rows), so C3 at N = 1,048,576 takes minutes.  The
oracle's skeletonization (oracle/hks_oracle.py, skeleton.py:84-182 and
linalg.py:43-136 restated) pivots on the sampled blocks themselves; the GPU
path runs them through the tall-skinny QR pre-reduction first.

    OPENBLAS_NUM_THREADS=8 python tools/make_full_skeleton_digest.py C3 123
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import hks_oracle as O  # noqa: E402
from paper_1701_02324_b200 import workloads as W  # noqa: E402


class KnnRows:
    """knn_lists[begin:end] on demand, cached per slice."""

    def __init__(self, coords, k):
        self.coords, self.k, self.cache = coords, k, {}

    def __getitem__(self, sl):
        key = (sl.start, sl.stop)
        if key not in self.cache:
            self.cache[key] = O.knn_rows(self.coords, self.k, np.arange(sl.start, sl.stop))
        return self.cache[key]


def main(key, which):
    w = W.CONFIGS[key]
    x = W.points(w, 0)
    t0 = time.time()
    tree = O.build_tree(x, w.leaf_size, 0)
    kern = {"family": "gaussian", "h": w.h}
    knn = KnnRows(tree.coords, w.kappa)
    depth = tree.depth
    g = (1 << (depth - 2)) - 1 + which  # a node two levels above the leaves
    order = [4 * g + 3, 4 * g + 4, 4 * g + 5, 4 * g + 6, 2 * g + 1, 2 * g + 2, g]
    skel, interp, out = {}, {}, {}
    for i in order:
        b, e = int(tree.begin[i]), int(tree.end[i])
        rows = O.sample_rows(tree.n, b, e, i, w.samples, "knn_augmented", 0, knn)
        cands = np.arange(b, e) if tree.is_leaf(i) else np.concatenate([skel[2 * i + 1], skel[2 * i + 2]])
        blk = O.kernel_block("gaussian", tree.coords[rows], tree.coords[cands], h=w.h)
        tau = w.tau if w.tau else 1e-300
        cols, p_i = O.interp_decomp(blk, tau, w.max_rank)
        skel[i] = cands[cols]
        interp[i] = p_i
        out[str(i)] = {"rows": int(rows.size), "indices": skel[i].tolist()}
        print(i, "rows", rows.size, "rank", cols.size, f"{time.time() - t0:.0f} s", flush=True)
    # the subtree's factorization (solver.py:111-186 restated in the oracle):
    # theta of every node, push / z_cond of the internal ones -- the subtree
    # depends on nothing outside it
    lam = w.lam
    fac, facts = {}, {}
    for i in order:
        if tree.is_leaf(i):
            b, e = int(tree.begin[i]), int(tree.end[i])
            a = O.kernel_block("gaussian", tree.coords[b:e], tree.coords[b:e], h=w.h) + lam * np.eye(e - b)
            phi = O.lu_solve(O.lu(a), interp[i].T)
            fac[i] = {"theta": interp[i] @ phi}
        else:
            tl, tr = fac[2 * i + 1]["theta"], fac[2 * i + 2]["theta"]
            rl, rr = tl.shape[0], tr.shape[0]
            c = O.kernel_block("gaussian", tree.coords[skel[2 * i + 1]], tree.coords[skel[2 * i + 2]], h=w.h)
            z = np.eye(rl + rr)
            z[:rl, rl:] += tl @ c
            z[rl:, :rl] += tr @ c.T
            zf, cond = O.factor_z(z, i, tree.level_of(i))
            th = np.zeros((rl + rr, rl + rr))
            th[:rl, :rl] = tl
            th[rl:, rl:] = tr
            folded = O._couple(c, O.lu_solve(zf, th))
            fac[i] = {"theta": interp[i] @ (th - th @ folded) @ interp[i].T, "push": interp[i].T - folded @ interp[i].T,
                      "z_cond": cond}
        facts[f"theta_norm_{i}"] = np.linalg.norm(fac[i]["theta"])
        if "z_cond" in fac[i]:
            facts[f"z_cond_{i}"] = fac[i]["z_cond"]
            facts[f"push_norm_{i}"] = np.linalg.norm(fac[i]["push"])
    # the subtree root's theta and push as 8 seeded Gaussian sketches (the test regenerates G)
    gs = np.random.default_rng([29, int(g)]).standard_normal((fac[g]["theta"].shape[1], 8))
    facts["theta_root_sketch"] = fac[g]["theta"] @ gs
    facts["push_root_sketch"] = fac[g]["push"] @ gs
    # upward pass of a seeded weight vector supported on the subtree
    # (treecode.py:65-89): the subtree root's skeleton weights
    b0, e0 = int(tree.begin[g]), int(tree.end[g])
    wv = np.random.default_rng([31, int(g)]).standard_normal(e0 - b0)
    up = {}
    for i in order:
        if tree.is_leaf(i):
            up[i] = interp[i] @ wv[int(tree.begin[i]) - b0: int(tree.end[i]) - b0]
        else:
            up[i] = interp[i] @ np.concatenate([up[2 * i + 1], up[2 * i + 2]])
    facts["upward_root"] = up[g]
    facts["lam"] = lam
    np.savez_compressed(ROOT / "tests" / "golden" / f"full_{key.lower()}_factor.npz", **facts)
    print("factor fixtures", f"{time.time() - t0:.0f} s", {k: float(v) for k, v in facts.items() if np.ndim(v) == 0})
    res = {"workload": key, "n": w.n, "subtree_root": int(g), "nodes": out,
           "seconds": round(time.time() - t0, 1)}
    (ROOT / "tests" / "golden" / f"full_{key.lower()}_skeletons.json").write_text(json.dumps(res) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else 123)
