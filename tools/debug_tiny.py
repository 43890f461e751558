import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_1701_02324_b200 as hk
from golden_cases import oracle_instance, load
from oracle import hks_oracle as O
inst = oracle_instance("tiny_n10")
t = inst["tree"]
x = t.coords
A = O.kernel_block("gaussian", x[5:10], x[0:5], h=0.5)
print("oracle", O.qrcp(A, 1e-7, 64)[0])
cols, p = hk.interpolative_decomposition(A, 1e-7, 64)
print("gpu id cols", cols)
qr = hk.pivoted_qr(A, 1e-7, 64)
print("gpu qr", qr.pivots, qr.rank)
g = load("tiny_n10")
tree = hk.build_tree(hk.PointSet(inst["coords_in"]), 5, seed=0)
cfg = hk.SkeletonConfig(tau=1e-7, max_rank=64, samples=256, sample_mode="exact", seed=0)
sk = hk.build_skeletons(tree, hk.KernelSpec("gaussian", h=0.5), cfg)
print("gpu skel", sk[1].indices, sk[2].indices, sk.ranks)
Ad = hk.kernels.eval_block_device(hk.KernelSpec("gaussian", h=0.5), tree.device_points(), rows=hk._native.to_device(np.arange(5, 10)), cols=hk._native.to_device(np.arange(0, 5)), row_major=True)
print("gpu eval row-major\n", Ad.cpu().numpy() - A)
z = np.load("tests/golden/id_cases.npz")
bad = 0
for tt in range(12):
    tol, mr = z[f"tol{tt}"]
    c, pp = hk.interpolative_decomposition(z[f"a{tt}"], tol, int(mr))
    if not np.array_equal(c, z[f"cols{tt}"]):
        bad += 1
        print("id case", tt, c[:8], z[f"cols{tt}"][:8], z[f"a{tt}"].shape, tol, mr)
print("bad id cases", bad)
