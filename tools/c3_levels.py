"""Per-level structure (node count, mean / max R and r) and device times of
one workload's factorize.  Usage: python tools/c3_levels.py [C3]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
depth = int(np.log2(w.n // w.leaf_size))
rank = {i: int(v) for i, v in enumerate(sk.ranks)}
for lev in range(depth, -1, -1):
    ids = range(2 ** lev - 1, 2 ** (lev + 1) - 1)
    r = np.array([rank.get(i, 0) for i in ids])
    R = np.array([rank.get(2 * i + 1, 0) + rank.get(2 * i + 2, 0) for i in ids]) if lev < depth else np.zeros(1)
    print(f"level {lev:2d} nodes {len(ids):5d} r mean {r.mean():6.1f} max {int(r.max()):4d}  R mean {R.mean():6.1f} max {int(R.max()):4d}")
for cond in (False, True):
    for _ in range(3):
        f = hk.factorize(op, w.lam, with_cond=cond)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f = hk.factorize(op, w.lam, with_cond=cond)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"with_cond={cond}: factorize ms {np.round(ts, 3)} levels",
          {k: round(v * 1e3, 3) for k, v in sorted(f.level_seconds.items())})
