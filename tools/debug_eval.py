import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1701_02324_b200 as hk
from paper_1701_02324_b200 import _native as N
x = np.random.default_rng(0).random((10, 2))
X = N.to_device(x)
k = hk.KernelSpec("gaussian", h=0.5)
rows = N.to_device(np.arange(5, 10)); cols = N.to_device(np.arange(0, 5))
print("rows ptr", hex(rows.data_ptr()), "cols ptr", hex(cols.data_ptr()))
for rm in (True, False):
    A = hk.kernels.eval_block_device(k, X, rows=rows, cols=cols, row_major=rm).cpu().numpy()
    ref = np.exp(((x[5:10, None, :] - x[None, 0:5, :]) ** 2).sum(-1) / (-2 * 0.25))
    print(rm, np.abs(A - ref).max(), np.diag(A))
torch.cuda.synchronize()
