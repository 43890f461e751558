"""Per-step device times of one C2 factorize (hks_profile with HKS_TRACE=1;
graphs off).  Usage: HKS_TRACE=1 python tools/trace_fact.py 2> trace.txt"""
import sys
sys.path.insert(0, ".")
import torch
import numpy as np
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W, _native as N
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
COND = len(sys.argv) > 2 and sys.argv[2] == "cond"
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
for _ in range(3):
    f = hk.factorize(op, w.lam, with_cond=COND)
torch.cuda.synchronize()
N.profile(True)
f = hk.factorize(op, w.lam, with_cond=COND)
torch.cuda.synchronize()
print("MARK", file=sys.stderr, flush=True)
res = N.profile(False)
print({k: round(v["ms"], 3) for k, v in res.items() if v["launches"]})

# the solve of the bench step (nrhs right-hand sides, device resident)
from paper_1701_02324_b200 import solver as S
B = torch.from_numpy(np.ascontiguousarray(W.rhs(w, 0).T)).cuda()
for _ in range(3):
    S.solve_device(f, B)
torch.cuda.synchronize()
print("MARK SOLVE", file=sys.stderr, flush=True)
N.profile(True)
S.solve_device(f, B)
torch.cuda.synchronize()
res = N.profile(False)
print("solve", {k: round(v["ms"], 3) for k, v in res.items() if v["launches"]})
