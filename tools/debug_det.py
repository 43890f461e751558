import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
rng = np.random.default_rng(0)
m, n = 4000, 1024
u, _ = np.linalg.qr(rng.standard_normal((m, 300)))
v, _ = np.linalg.qr(rng.standard_normal((n, 300)))
a = (u * 0.9 ** np.arange(300)) @ v.T
res = [hk.interpolative_decomposition(a, 1e-300, 256) for _ in range(3)]
print("ID cols equal:", all(np.array_equal(res[0][0], r[0]) for r in res), "P equal:", all(np.array_equal(res[0][1], r[1]) for r in res))
x = rng.random((3000, 18))
k = hk.KernelSpec("gaussian", h=0.6)
X = hk._native.to_device(x)
rows = hk._native.to_device(rng.integers(0, 3000, 2500))
cols = hk._native.to_device(np.arange(1024))
e = [hk.kernels.eval_block_device(k, X, rows=rows, cols=cols, row_major=True).cpu().numpy() for _ in range(3)]
print("eval equal:", all(np.array_equal(e[0], z) for z in e))
