"""Standalone cost of the dgecon estimates: with HKS_COND_START_LEVEL=0 every
estimate chain starts after the root, so the interval from the end of the
factorization (main stream) to the end of the estimates (join_cond) is the
estimates' run time with the GPU otherwise idle.  Usage:
HKS_COND_START_LEVEL=0 python tools/gecon_alone.py C3"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W
assert os.environ.get("HKS_COND_START_LEVEL") == "0"
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
res = []
for it in range(6):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    f = hk.factorize(op, w.lam, with_cond=True)
    e1.record()
    f.join_cond()
    e2.record()
    torch.cuda.synchronize()
    res.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    zc = f.z_cond_per_level()
print("factorize ms / estimate tail ms:", [(round(a, 2), round(b, 2)) for a, b in res[2:]])
print("z_cond per level", {k: f"{v:.3e}" for k, v in zc.items()})
