"""Point sets and the reference's synthetic generators (host side).

Point-set I/O is outside the accelerated path (data.py
is host I/O kept for the harness); ``PointSet`` and ``generate`` are kept
so callers of the reference find the same constructors (data.py:32-114).
The device copy of a point set is cached on first use.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SHAPES = ("uniform_cube", "sphere_surface", "gaussian_mixture")
_MIX_STD, _MIX_SEP, _MIX_BOX = 0.5, 6.0, 10.0


@dataclass(frozen=True)
class PointSet:
    coords: np.ndarray
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        c = np.asarray(self.coords, dtype=np.float64)
        if c.ndim != 2:
            raise ValueError("coords must be 2-D")
        if c.shape[0] < 1 or c.shape[1] < 1:
            raise ValueError("point set needs n >= 1 and d >= 1")
        if not np.all(np.isfinite(c)):
            raise ValueError("coordinates must be finite")
        c = c.copy()
        c.flags.writeable = False
        object.__setattr__(self, "coords", c)

    @property
    def n(self):
        return self.coords.shape[0]

    @property
    def d(self):
        return self.coords.shape[1]

    def device(self):
        """(n, d) float64 CUDA tensor (cached)."""
        if "x" not in self._dev:
            from . import _native as N
            self._dev["x"] = N.to_device(self.coords)
        return self._dev["x"]


def _rng(seed, *stream):
    return np.random.default_rng([int(seed), *map(int, stream)])


def mixture_centers(d, k_clusters, seed, max_draws=1_000_000):
    """Rejection-sampled centres >= 12 sigma apart (data.py:63-80); bounded
    so an infeasible draw sequence raises instead of looping forever."""
    rng = _rng(seed, 2, 0)
    centers = np.empty((k_clusters, d))
    count = 0
    for _ in range(max_draws):
        if count == k_clusters:
            break
        cand = rng.uniform(0.0, _MIX_BOX, size=d)
        if count == 0 or np.min(np.linalg.norm(centers[:count] - cand, axis=1)) >= _MIX_SEP:
            centers[count] = cand
            count += 1
    if count < k_clusters:
        raise ValueError("could not place mixture centres; lower k_clusters or raise d")
    return centers


def generate(shape, n, seed, d=3, k_clusters=4):
    """Deterministic synthetic point sets (data.py:83-114)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if d < 1:
        raise ValueError("d must be >= 1")
    if shape == "uniform_cube":
        coords = _rng(seed, 0, 0).random((n, d))
    elif shape == "sphere_surface":
        rng = _rng(seed, 1, 0)
        coords = rng.standard_normal((n, d))
        norms = np.linalg.norm(coords, axis=1)
        while np.any(norms == 0.0):
            bad = norms == 0.0
            coords[bad] = rng.standard_normal((int(bad.sum()), d))
            norms = np.linalg.norm(coords, axis=1)
        coords /= norms[:, None]
    elif shape == "gaussian_mixture":
        if k_clusters < 1:
            raise ValueError("k_clusters must be >= 1")
        centers = mixture_centers(d, k_clusters, seed)
        rng = _rng(seed, 2, 1)
        which = rng.integers(k_clusters, size=n)
        coords = centers[which] + _MIX_STD * rng.standard_normal((n, d))
    else:
        raise ValueError(f"unknown shape {shape!r}")
    return PointSet(coords)
