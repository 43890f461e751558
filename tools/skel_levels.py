"""Per-level shape and time of build_skeletons: node count, sampled rows
(mean / max), candidate columns, ranks, host row sampling and device
skeletonize wall time.  Usage: python tools/skel_levels.py [C3] [N]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_02324_b200 as hk  # noqa: E402
from paper_1701_02324_b200 import _native as N  # noqa: E402
from paper_1701_02324_b200 import skeleton as S  # noqa: E402
from paper_1701_02324_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
if len(sys.argv) > 2:
    w = w.scaled(int(sys.argv[2]))
x = W.points(w, 0)
kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples, sample_mode="knn_augmented", seed=0)
tree = hk.build_tree(hk.PointSet(x), w.leaf_size)
knn = hk.knn_bruteforce(tree.points, w.kappa)
torch.cuda.synchronize()
orig_rows, orig_fn = S._level_rows, N.fn
t_rows, t_dev = [], []


def timed_rows(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = orig_rows(*a, **k)
    torch.cuda.synchronize()
    t_rows.append(time.perf_counter() - t0)
    return out


def fn(name):
    f = orig_fn(name)
    if name != "hks_skeletonize_level":
        return f

    def wrapped(*a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = f(*a)
        torch.cuda.synchronize()
        t_dev.append(time.perf_counter() - t0)
        return rc
    return wrapped


S._level_rows = timed_rows
N.fn = fn
for rep in range(2):
    t_rows.clear()
    t_dev.clear()
    t0 = time.perf_counter()
    sk = hk.build_skeletons(tree, kern, cfg, knn=knn)
    torch.cuda.synchronize()
    print(f"build_skeletons {time.perf_counter() - t0:.3f} s (rows {sum(t_rows):.3f}, device {sum(t_dev):.3f})")
depth = tree.depth
for j, lev in enumerate(range(depth, 0, -1)):
    first, count = (1 << lev) - 1, 1 << lev
    rc = sk.rows_count[first:first + count]
    r = sk.ranks[first:first + count]
    if lev == depth:
        c = np.full(count, w.leaf_size)
    else:
        c = np.array([sk.ranks[2 * i + 1] + sk.ranks[2 * i + 2] for i in range(first, first + count)])
    gb = float((rc * c).sum()) * 8 / 1e9
    print(f"level {lev:2d} nodes {count:5d} rows mean {rc.mean():9.1f} max {rc.max():8d} cols mean {c.mean():6.1f} "
          f"rank mean {r.mean():6.1f} max {r.max():4d}  block GB {gb:7.2f}  rows_s {t_rows[j]:.3f} dev_s {t_dev[j]:.3f}")
