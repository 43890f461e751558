"""Repeated build_skeletons at C2: wall time per call and per level (host
wall around each hks_skeletonize_level, device drained), then a CUDA
kernel profile of one more call.  python tools/skel_times.py [C2]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1701_02324_b200 as hk  # noqa: E402
from paper_1701_02324_b200 import _native as N  # noqa: E402
from paper_1701_02324_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
orig = N.fn
per = []


def fn(name):
    f = orig(name)
    if name != "hks_skeletonize_level":
        return f

    def wrapped(*a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = f(*a)
        torch.cuda.synchronize()
        per.append(round(time.perf_counter() - t0, 3))
        return rc
    return wrapped


N.fn = fn
for i in range(3):
    per.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    torch.cuda.synchronize()
    print("build_skeletons", round(time.perf_counter() - t0, 3), "levels", per,
          "free GB", round(torch.cuda.mem_get_info()[0] / 2**30, 1),
          "torch reserved GB", round(torch.cuda.memory_reserved() / 2**30, 1))
    del sk
