"""Full-size structure digests from the CPU oracle (test infrastructure):
tree permutation and exact kNN lists of a BASELINE configuration at its
full N, as SHA-256 digests of the int64 arrays plus their first rows, for
tests/test_gpu_full_structure.py.  The oracle (oracle/hks_oracle.py) is the
reference's algorithm restated (tree.py:87-144, 163-188) and pinned
bit-exactly against the unmodified reference's outputs up to N = 65536
(tests/test_oracle_golden.py, tests/golden/ladder_*.npz); the reference
itself refuses kNN above 65536 points (tree.py:170-171).

    OPENBLAS_NUM_THREADS=8 python tools/make_full_digests.py C2
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import hks_oracle as O  # noqa: E402
from paper_1701_02324_b200 import workloads as W  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def main(key, with_knn=True, knn_rows=0):
    """with_knn: the whole kNN table (hours of CPU at N = 1M); knn_rows > 0
    instead digests the lists of that many seeded sample rows, each against
    all N points (minutes)."""
    w = W.CONFIGS[key]
    x = W.points(w, 0)
    t0 = time.time()
    tree = O.build_tree(x, w.leaf_size, 0)
    t1 = time.time()
    out = {"workload": key, "n": w.n, "leaf": w.leaf_size, "kappa": w.kappa,
           "coords_sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
           "perm_sha256": sha(tree.perm), "perm_head": tree.perm[:64].tolist()}
    secs = {"tree": round(t1 - t0, 1)}
    if with_knn:
        nl = O.knn(tree.coords, w.kappa)
        out.update(knn_sha256=sha(nl), knn_head=nl[:64].tolist())
        secs["knn"] = round(time.time() - t1, 1)
    elif knn_rows > 0:
        rows = np.sort(np.random.default_rng([17, w.n]).choice(w.n, size=knn_rows, replace=False))
        nl = O.knn_rows(tree.coords, w.kappa, rows)
        out.update(knn_sample_rows=rows.tolist(), knn_sample_sha256=sha(nl), knn_sample_head=nl[:8].tolist())
        secs["knn_sample"] = round(time.time() - t1, 1)
    out["seconds"] = secs
    (ROOT / "tests" / "golden" / f"full_{key.lower()}_digest.json").write_text(json.dumps(out) + "\n")
    print(key, out["seconds"])


if __name__ == "__main__":
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    mode = sys.argv[2] if len(sys.argv) > 2 else "full"
    main(key, with_knn=mode == "full", knn_rows=int(sys.argv[3]) if mode == "sample" and len(sys.argv) > 3 else 0)
