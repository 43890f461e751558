import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
w = W.CONFIGS["C2"].scaled(n)
x = W.points(w, 0)
def log(*a):
    print(f"[{time.perf_counter():.2f}]", *a, flush=True)
log("points", x.shape)
ps = hk.PointSet(x)
tree = hk.build_tree(ps, w.leaf_size, seed=0); torch.cuda.synchronize(); log("tree", tree.depth)
knn = hk.knn_bruteforce(tree.points, w.kappa); torch.cuda.synchronize(); log("knn")
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
from paper_1701_02324_b200 import skeleton as S
skels = hk.build_skeletons(tree, kern, cfg, knn=knn); torch.cuda.synchronize(); log("skel", skels.ranks[:8], skels.rows_count[:8])
op = hk.build_operator(tree, skels, kern); torch.cuda.synchronize(); log("op")
f = hk.factorize(op, w.lam); torch.cuda.synchronize(); log("fact")
b = W.rhs(w, 0)
xs = hk.solve_multi(f, b); log("solve")
