import sys, time, json, os
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W, _native as N
w = W.CONFIGS["C2"]
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
for cond in (False, True):
    for _ in range(3):
        f = hk.factorize(op, w.lam, with_cond=cond)
    torch.cuda.synchronize()
    dev, wall = [], []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(); f = hk.factorize(op, w.lam, with_cond=cond); e1.record(); torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3); dev.append(e0.elapsed_time(e1))
    print("cond", cond, "dev ms", [round(t, 1) for t in dev], "wall", [round(t, 1) for t in wall])
    print("   levels", {k: round(v * 1e3, 2) for k, v in f.level_seconds.items()})
