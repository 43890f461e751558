"""Per-step device times of back-to-back C2 factorize+solve steps (looking
for intermittent slow steps).  Usage: python tools/spikes.py [cond] [steps]"""
import gc
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W
from paper_1701_02324_b200.solver import solve_device
w = W.CONFIGS["C2"]
cond = len(sys.argv) > 1 and sys.argv[1] == "1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
B = torch.from_numpy(np.ascontiguousarray(W.rhs(w, 0).T)).cuda()
keep = None
for _ in range(3):
    f = hk.factorize(op, w.lam, with_cond=cond)
    keep = (f, solve_device(f, B))
torch.cuda.synchronize()
gc.disable()
ts = []
for i in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f = hk.factorize(op, w.lam, with_cond=cond)
    X = solve_device(f, B)
    e1.record()
    keep = (f, X)
    ts.append((e0, e1))
torch.cuda.synchronize()
print("cond" if cond else "nocond", [round(a.elapsed_time(b), 2) for a, b in ts])
