"""Exact kNN wall time on a workload's points: python tools/knn_time.py [C3] [N]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1701_02324_b200 as hk  # noqa: E402
from paper_1701_02324_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
if len(sys.argv) > 2:
    w = w.scaled(int(sys.argv[2]))
x = W.points(w, 0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    knn = hk.knn_bruteforce(tree.points, w.kappa)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{w.name} n={w.n} d={x.shape[1]} k={w.kappa}: kNN {dt:.3f} s, {2.0 * w.n * w.n * x.shape[1] / dt / 1e12:.2f} TFLOP/s (2 n^2 d)")
