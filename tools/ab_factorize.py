import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W, _native as N
from paper_1701_02324_b200.solver import solve_device
w = W.CONFIGS["C2"].scaled(int(sys.argv[1]) if len(sys.argv) > 1 else 262144)
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
op = hk.build_operator(tree, sk, kern)
for _ in range(3):
    f = hk.factorize(op, w.lam)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f = hk.factorize(op, w.lam); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("factorize ms", [round(t, 2) for t in ts])
print("level ms", {k: round(v * 1e3, 2) for k, v in f.level_seconds.items()})
N.profile(True)
f = hk.factorize(op, w.lam)
k = N.profile(False)
print("profile", json.dumps({a: round(b["ms"], 2) for a, b in k.items() if b["launches"]}))
t0 = time.perf_counter(); f = hk.factorize(op, w.lam, with_cond=False); torch.cuda.synchronize(); print("no-cond factorize wall ms", (time.perf_counter()-t0)*1e3)
