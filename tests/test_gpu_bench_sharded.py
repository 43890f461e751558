"""bench.py's fixed-N multi-GPU mode (the default for N > 1): the
configuration's instance split across 2 ranks by subtree gives the
single-GPU solution.  The 2 ranks run as 2 processes of bench.py sharing
cuda:0 with gloo collectives (HKS_BENCH_BACKEND=gloo; no kernel waits on
another rank); the C3 generator / kernel / adaptive ranks at N = 32768."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
ARGS = ["--config", "C3", "--points", "32768", "--steps", "1", "--warmup", "1", "--no-cpu-baseline",
        "--no-clocks", "--no-accuracy"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(tmp, world):
    port, procs = _port(), []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), HKS_BENCH_BACKEND="gloo")
        if world == 1:
            for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
                env.pop(k)
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "bench.py"), *ARGS, "--dump-x", str(tmp)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (out, err) in zip(procs, outs):
        assert p.returncode == 0, err[-3000:]
    return json.loads(outs[0][0].strip().splitlines()[-1])


def test_fixed_n_split_matches_single_gpu(tmp_path):
    one, two = tmp_path / "p1", tmp_path / "p2"
    one.mkdir()
    two.mkdir()
    line1 = _bench(one, 1)
    line2 = _bench(two, 2)
    assert line1["config"]["n_global"] == line2["config"]["n_global"] == 32768
    assert line2["scaling"] == "strong" and line2["n_gpus"] == 2
    x1 = np.load(one / "x_rank0.npz")["x"]
    parts = sorted((np.load(two / f"x_rank{r}.npz") for r in range(2)), key=lambda z: int(z["begin"]))
    x2 = np.concatenate([z["x"] for z in parts], axis=1)
    assert x2.shape == x1.shape
    err = np.linalg.norm(x2 - x1) / np.linalg.norm(x1)
    assert err <= 1e-11, err
    assert line2["relres_vs_ktilde"] <= 10 * max(line1["relres_vs_ktilde"], 1e-14)
