import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_1701_02324_b200 as hk
from golden_cases import load, coords_for, skel_list
g = load("c4_n8192"); m = g["meta"]
x = coords_for("c4_n8192")
tree = hk.build_tree(hk.PointSet(x), m["leaf"], seed=0)
knn = hk.knn_bruteforce(tree.points, m["kappa"])
cfg = hk.SkeletonConfig(tau=m["tau"], max_rank=m["max_rank"], samples=m["samples"], sample_mode=m["mode"], seed=0)
kern = hk.KernelSpec("gaussian", h=m["h"], regularization=m["lam"])
s1 = hk.build_skeletons(tree, kern, cfg, knn=knn)
s2 = hk.build_skeletons(tree, kern, cfg, knn=knn)
for i in range(1, 31):
    a, b, ref = s1[i].indices, s2[i].indices, skel_list(g, i)
    same_run = np.array_equal(a, b)
    eq = np.array_equal(a, ref)
    first = int(np.argmax(a != ref)) if not eq and a.size == ref.size else -1
    print(i, "deterministic" if same_run else "NONDETERMINISTIC", "match" if eq else f"differs from position {first} of {a.size}",
          "setdiff", len(set(a) ^ set(ref)))
