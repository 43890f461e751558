"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE.json names no dataset; every input is synthetic (SURVEY.md section
8(d)).  All generators are host numpy with keyed
streams ``default_rng([seed, stream])`` so the oracle and the device path see
identical bits.  C1 is exactly the reference's
``generate("uniform_cube", N, seed, d=8)`` (data.py:94-95).

Choices BASELINE.json leaves open, fixed here once and echoed in every report:
  * seed 0;
  * ``samples`` (the row-sample target ell) = max(4 s, 128);
  * "fixed rank s" = tau 1e-300 with max_rank s;
  * C3 noise is N(0, 1e-6) read as *variance* 1e-6 (sigma 1e-3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    h: float
    lam: float
    leaf_size: int
    max_rank: int
    tau: float
    kappa: int
    nrhs: int
    generator: str
    method: str = "direct"          # or "hybrid"
    gmres_tol: float = 1e-6
    gmres_restart: int = 50

    @property
    def samples(self):
        return max(4 * self.max_rank, 128)

    def scaled(self, n):
        """Same generator / kernel / tree / rank parameters at another N."""
        return Workload(**{**self.__dict__, "n": int(n)})

    def echo(self):
        out = dict(self.__dict__)
        out["samples"] = self.samples
        out["sample_mode"] = "knn_augmented"
        return out


FIXED = 1e-300

CONFIGS = {
    "C1": Workload("C1", 16384, 8, 0.5, 1.0, 256, 64, FIXED, 16, 4, "uniform_cube"),
    "C2": Workload("C2", 262144, 18, 0.8, 1e-2, 512, 128, FIXED, 32, 16, "mixture8"),
    "C3": Workload("C3", 1048576, 28, 0.5, 1e-3, 512, 256, 1e-5, 32, 16, "subspace6"),
    "C4": Workload("C4", 4194304, 18, 0.6, 1e-2, 1024, 256, FIXED, 32, 64, "mixture8"),
    "C5": Workload("C5", 1048576, 784, 1.0, 1e-5, 512, 512, 1e-4, 32, 8, "sparse784",
                   method="hybrid"),
}

_STREAM = {"mixture8": 902, "subspace6": 903, "sparse784": 905}


def points(w: Workload, seed: int = 0) -> np.ndarray:
    """(n, d) float64 points for workload ``w``."""
    n, d = w.n, w.d
    if w.generator == "uniform_cube":
        return np.random.default_rng([seed, 0, 0]).random((n, d))
    g = np.random.default_rng([seed, _STREAM[w.generator]])
    if w.generator == "mixture8":
        centres = g.standard_normal((8, d))
        label = g.integers(8, size=n)
        x = centres[label] + 0.3 * g.standard_normal((n, d))
        return (x - x.mean(axis=0)) / x.std(axis=0)
    if w.generator == "subspace6":
        q, _ = np.linalg.qr(g.standard_normal((d, 6)))
        return g.standard_normal((n, 6)) @ q.T + np.sqrt(1e-6) * g.standard_normal((n, d))
    if w.generator == "sparse784":
        x = np.where(g.random((n, d)) < 0.8, 0.0, 1.0 - g.random((n, d)))
        bad = ~x.any(axis=1)
        while bad.any():
            k = int(bad.sum())
            x[bad] = np.where(g.random((k, d)) < 0.8, 0.0, 1.0 - g.random((k, d)))
            bad = ~x.any(axis=1)
        return x / np.linalg.norm(x, axis=1)[:, None]
    raise ValueError(f"unknown generator {w.generator!r}")


def rhs(w: Workload, seed: int = 0, k: int | None = None) -> np.ndarray:
    """(n, k) iid N(0, 1) right-hand sides."""
    return np.random.default_rng([seed, 1000]).standard_normal((w.n, k or w.nrhs))
