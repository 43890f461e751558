"""Per-level device times of the C2 factorize (graphs on) and the per-step
trace (graphs off).  Usage: HKS_TRACE=1 python tools/level_times.py [C2] 2> trace.txt"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W, _native as N
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
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
N.profile(True)
f = hk.factorize(op, w.lam, with_cond=True)
torch.cuda.synchronize()
res = N.profile(False)
print({k: round(v["ms"], 3) for k, v in res.items() if v["launches"]})

# the bench step's solve (nrhs device-resident right-hand sides), per step
from paper_1701_02324_b200 import solver as S
B = torch.from_numpy(np.ascontiguousarray(W.rhs(w, 0).T)).cuda()
for _ in range(3):
    S.solve_device(f, B)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.solve_device(f, B)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("solve ms (graph)", np.round(ts, 3))
print("MARK SOLVE", file=sys.stderr, flush=True)
N.profile(True)
S.solve_device(f, B)
torch.cuda.synchronize()
res = N.profile(False)
print("solve", {k: round(v["ms"], 3) for k, v in res.items() if v["launches"]})
