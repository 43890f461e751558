"""One pre-reduced pivoted QR of a tall random block on the device (the
tsqr_absorb_kernel workload for ncu): python tools/tsqr_prof.py [rows] [cols]"""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1701_02324_b200 import _native as N  # noqa: E402
from paper_1701_02324_b200 import linalg  # noqa: F401,E402  (registers the signatures)

m = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
torch.manual_seed(0)
for rep in range(2):
    A = torch.rand(m, n, dtype=torch.float64, device="cuda")
    piv = torch.empty(n, dtype=torch.int64, device="cuda")
    P = torch.zeros(8 * n, dtype=torch.float64, device="cuda")
    rank = ctypes.c_int64(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    N.call("hks_interp_decomp", N.ptr(A), m, n, n, 1e-300, 8, N.ptr(piv), N.ptr(P), ctypes.byref(rank), N.stream_ptr())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rows {m} cols {n}: {dt * 1e3:.1f} ms, {2.0 * m * n * n / dt / 1e12:.2f} TFLOP/s (2 m n^2), rank {rank.value}")
