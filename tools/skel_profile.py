"""Where build_skeletons spends its time (C2 by default): per-level host
sampling vs device skeletonize (ID) time, and the kernel-kind profile."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import workloads as W, _native as N, skeleton as S
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
if len(sys.argv) > 2:
    w = w.scaled(int(sys.argv[2]))
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
torch.cuda.synchronize()
orig_rows, orig_call = S._level_rows, N.fn
tr = {"rows": 0.0}
def timed_rows(*a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = orig_rows(*a, **k); torch.cuda.synchronize()
    tr["rows"] += time.perf_counter() - t0
    return out
S._level_rows = timed_rows
t0 = time.perf_counter()
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"build_skeletons {tot:.3f} s, of which row sampling {tr['rows']:.3f} s")
N.profile(True)
sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
torch.cuda.synchronize()
print({k: round(v["ms"], 1) for k, v in N.profile(False).items() if v["launches"]})
