import os
import sys
from pathlib import Path

# The oracle's last bits follow the BLAS reduction order; pin one BLAS thread
# so the CPU checks against tests/golden are reproducible (and, on a loaded
# 8-core host, several times faster than oversubscribed OpenBLAS).
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")
try:
    from threadpoolctl import threadpool_limits as _tpl
    _tpl(1, user_api="blas")
except Exception:  # pragma: no cover - threadpoolctl is optional
    pass

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(Path(__file__).resolve().parent)):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhks.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
