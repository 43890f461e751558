import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import skeleton as S, _native as N
from golden_cases import load, coords_for, skel_list
g = load("c4_n8192"); m = g["meta"]
x = coords_for("c4_n8192")
tree = hk.build_tree(hk.PointSet(x), m["leaf"], seed=0)
knn = hk.knn_bruteforce(tree.points, m["kappa"])
cfg = hk.SkeletonConfig(tau=m["tau"], max_rank=m["max_rank"], samples=m["samples"], sample_mode=m["mode"], seed=0)
kern = hk.KernelSpec("gaussian", h=m["h"], regularization=m["lam"])
rows, roff = S._level_rows(tree, 3, cfg, knn.device.contiguous())
rows2, roff2 = S._level_rows(tree, 3, cfg, knn.device.contiguous())
print("rows deterministic", torch.equal(rows, rows2), roff)
X = tree.device_points()
for j, node in enumerate(range(7, 15)):
    r = rows[roff[j]:roff[j+1]]
    b0, e0 = int(tree._begin[node]), int(tree._end[node])
    A = hk.kernels.eval_block_device(kern, X, rows=r, cols=torch.arange(b0, e0, device=X.device), row_major=True).cpu().numpy()
    cols, p = hk.interpolative_decomposition(A, m["tau"], m["max_rank"])
    ref = skel_list(g, node)
    print(node, "single-node ID matches golden:", np.array_equal(cols + b0, ref), "rows", A.shape)
