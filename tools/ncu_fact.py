import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W
w = W.CONFIGS["C2"]
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
f = hk.factorize(op, w.lam)
torch.cuda.synchronize()
torch.cuda.profiler.start()
f = hk.factorize(op, w.lam)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
