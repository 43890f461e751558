"""Balanced binary partition + exact kNN on the GPU (tree.py of the reference).

``build_tree`` runs the level-synchronous sm_100a build (csrc/tree.cu):
per node the centred second-moment power iteration from the reference's
own start vector ``default_rng([seed, level, begin])`` (drawn here with host
numpy so the bits match), the projection, a segmented stable radix sort and
the physical permutation -- tree.py:70-144.  ``knn_bruteforce`` is the tiled
DMMA distance kernel with a per-query (d^2, index) top-k (tree.py:163-188),
without the reference's 65536-point guard.

Objects mirror the reference: PartitionTree.points / perm / inv_perm /
nodes / depth / leaf_size, TreeNode fields, levels().  Host views are
materialised lazily from device tensors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .data import PointSet

_POWER_STEPS = 10
KNN_MAX_POINTS = None  # the reference guards n <= 65536 (tree.py:159); the GPU path has no guard


@dataclass(frozen=True)
class TreeNode:
    index: int
    level: int
    begin: int
    end: int
    left: int | None = None
    right: int | None = None
    split_direction: np.ndarray | None = None
    split_value: float | None = None

    @property
    def is_leaf(self):
        return self.left is None

    @property
    def size(self):
        return self.end - self.begin


def tree_depth(n, leaf_size):
    """Smallest L with ceil(n / 2^L) <= leaf_size (tree.py:100-102)."""
    depth = 0
    while -(n // -(1 << depth)) > leaf_size:
        depth += 1
    return depth


def node_ranges(n, depth):
    """Heap-ordered begin / end (left child takes ceil(size / 2))."""
    count = (1 << (depth + 1)) - 1
    begin = np.zeros(count, dtype=np.int64)
    end = np.zeros(count, dtype=np.int64)
    end[0] = n
    for i in range((1 << depth) - 1):
        cut = begin[i] + (end[i] - begin[i] + 1) // 2
        begin[2 * i + 1], end[2 * i + 1] = begin[i], cut
        begin[2 * i + 2], end[2 * i + 2] = cut, end[i]
    return begin, end


class PartitionTree:
    """Tree-ordered points on the device plus the reference's host views."""

    def __init__(self, x_dev, perm_dev, depth, leaf_size, split_dirs=None, split_vals=None,
                 host_coords=None):
        self._x = x_dev
        self._perm_dev = perm_dev
        self.depth = int(depth)
        self.leaf_size = int(leaf_size)
        self._begin, self._end = node_ranges(int(x_dev.shape[0]), self.depth)
        self._split_dirs = split_dirs
        self._split_vals = split_vals
        self._host_coords = host_coords
        self._cache = {}

    # --- reference surface ---------------------------------------------------
    @property
    def n(self):
        return int(self._x.shape[0])

    @property
    def d(self):
        return int(self._x.shape[1])

    @property
    def points(self):
        if "points" not in self._cache:
            coords = self._host_coords if self._host_coords is not None else self._x.cpu().numpy()
            ps = PointSet(coords)
            ps._dev["x"] = self._x
            self._cache["points"] = ps
        return self._cache["points"]

    @property
    def perm(self):
        if "perm" not in self._cache:
            p = self._perm_dev.cpu().numpy().astype(np.int64)
            p.flags.writeable = False
            self._cache["perm"] = p
        return self._cache["perm"]

    @property
    def inv_perm(self):
        if "inv" not in self._cache:
            inv = np.empty(self.n, dtype=np.int64)
            inv[self.perm] = np.arange(self.n)
            inv.flags.writeable = False
            self._cache["inv"] = inv
        return self._cache["inv"]

    @property
    def nodes(self):
        if "nodes" not in self._cache:
            out = []
            first_leaf = (1 << self.depth) - 1
            for i in range((1 << (self.depth + 1)) - 1):
                lev = int(np.floor(np.log2(i + 1)))
                if i >= first_leaf:
                    out.append(TreeNode(i, lev, int(self._begin[i]), int(self._end[i])))
                else:
                    sd = None if self._split_dirs is None else np.array(self._split_dirs[i])
                    sv = None if self._split_vals is None else float(self._split_vals[i])
                    out.append(TreeNode(i, lev, int(self._begin[i]), int(self._end[i]),
                                        left=2 * i + 1, right=2 * i + 2,
                                        split_direction=sd, split_value=sv))
            self._cache["nodes"] = out
        return self._cache["nodes"]

    @property
    def root(self):
        return self.nodes[0]

    def children(self, node):
        return self.nodes[node.left], self.nodes[node.right]

    def leaves(self):
        return self.nodes[(1 << self.depth) - 1:]

    # --- device surface ------------------------------------------------------
    def device_points(self):
        return self._x

    def device_perm(self):
        return self._perm_dev

    @classmethod
    def from_host(cls, coords_tree_order, perm, leaf_size, split_dirs=None, split_vals=None):
        """Wrap an externally built tree (tests feed the oracle's tree)."""
        coords = np.ascontiguousarray(coords_tree_order, dtype=np.float64)
        depth = tree_depth(coords.shape[0], leaf_size)
        return cls(N.to_device(coords), N.to_device(np.asarray(perm, dtype=np.int64)), depth,
                   leaf_size, split_dirs, split_vals, host_coords=coords)


def levels(tree, bottom_up=True):
    """Each level's nodes ordered by range (tree.py:147-156)."""
    ks = range(tree.depth, -1, -1) if bottom_up else range(tree.depth + 1)
    for k in ks:
        first = (1 << k) - 1
        yield tree.nodes[first: 2 * first + 1]


def _start_vectors(seed, n, depth, d):
    """The reference's per-node power-method start vectors
    default_rng([seed, level, begin]).standard_normal(d), normalised
    (tree.py:76-77, 114), for every internal node in heap order."""
    begin, _ = node_ranges(n, depth)
    out = np.zeros(((1 << depth) - 1, d))
    for i in range((1 << depth) - 1):
        level = int(np.floor(np.log2(i + 1)))
        v = np.random.default_rng([seed, level, int(begin[i])]).standard_normal(d)
        out[i] = v / np.linalg.norm(v)
    return out


def build_tree(ps, leaf_size, seed=0):
    """Balanced spatial partition, built on the GPU (tree.py:87-144)."""
    if leaf_size < 2:
        raise ValueError("leaf_size must be >= 2")
    if not isinstance(ps, PointSet):
        ps = PointSet(ps)
    n, d = ps.n, ps.d
    depth = tree_depth(n, leaf_size)
    t = N.torch()
    x_in = ps.device()
    x_out = t.empty((n, d), dtype=t.float64, device=x_in.device)
    perm = t.empty(n, dtype=t.int64, device=x_in.device)
    nint = (1 << depth) - 1
    starts = N.to_device(_start_vectors(seed, n, depth, d)) if nint else t.zeros(1, dtype=t.float64,
                                                                                 device=x_in.device)
    dirs = t.zeros((max(nint, 1), d), dtype=t.float64, device=x_in.device)
    vals = t.zeros(max(nint, 1), dtype=t.float64, device=x_in.device)
    N.call("hks_build_tree", N.ptr(x_in), n, d, depth, _POWER_STEPS, N.ptr(starts), N.ptr(x_out), N.ptr(perm),
           N.ptr(dirs), N.ptr(vals), N.stream_ptr())
    return PartitionTree(x_out, perm, depth, leaf_size, dirs.cpu().numpy()[:nint], vals.cpu().numpy()[:nint])


class DeviceArray:
    """A device-resident result with numpy semantics on demand (``np.asarray``,
    indexing, ``shape``); ``.device`` is the CUDA tensor."""

    def __init__(self, dev):
        self.device = dev
        self._host = None

    def __array__(self, dtype=None, copy=None):
        if self._host is None:
            self._host = self.device.cpu().numpy()
        return self._host if dtype is None else self._host.astype(dtype)

    @property
    def shape(self):
        return tuple(self.device.shape)

    @property
    def dtype(self):
        return np.asarray(self).dtype

    def __len__(self):
        return int(self.device.shape[0])

    def __getitem__(self, item):
        return np.asarray(self)[item]

    def ravel(self):
        return np.asarray(self).ravel()


def knn_bruteforce(ps, k):
    """Exact k nearest neighbours per point, self excluded, ordered by
    (GEMM-form d^2, index) -- tree.py:163-188 -- on the GPU (csrc/knn.cu).
    Returns an (n, k) int64 array-like backed by device memory."""
    if not isinstance(ps, PointSet):
        ps = PointSet(ps)
    n = ps.n
    if not 1 <= k <= n - 1:
        raise ValueError("need 1 <= k <= n - 1")
    t = N.torch()
    x = ps.device()
    out = t.empty((n, k), dtype=t.int64, device=x.device)
    N.call("hks_knn", N.ptr(x), n, ps.d, k, N.ptr(out), N.stream_ptr())
    return DeviceArray(out)


def knn_approx(ps, k, trees=8, leaf_size=1024, seed=0):
    """Approximate k nearest neighbours (the
    reference has only the brute force of tree.py:163-188): the union, over
    `trees` random-projection trees (the partition of build_tree with random
    directions and no power steps), of the exact neighbours inside each
    leaf, merged per point by (GEMM-form d^2, index) with duplicates
    dropped.  Distances are computed exactly as knn_bruteforce computes
    them, so every neighbour it returns is ranked as the exact search ranks
    it.  Work is trees x n x leaf_size pairs instead of n^2.  With one leaf
    (leaf_size >= n) it is the exact search."""
    if not isinstance(ps, PointSet):
        ps = PointSet(ps)
    n, d = ps.n, ps.d
    if not 1 <= k <= n - 1:
        raise ValueError("need 1 <= k <= n - 1")
    if trees < 1:
        raise ValueError("trees must be >= 1")
    t = N.torch()
    x = ps.device()
    depth = tree_depth(n, max(int(leaf_size), 2))
    while depth > 0 and n >> depth < k + 1:  # every leaf must hold k + 1 points
        depth -= 1
    begin, end = node_ranges(n, depth)
    leaves = begin[(1 << depth) - 1:]
    seg = np.concatenate([leaves, [n]]).astype(np.int64)
    nint = (1 << depth) - 1
    best_i = best_d = None
    for tr in range(trees):
        rng = np.random.default_rng([int(seed), 101, tr])
        starts = rng.standard_normal((max(nint, 1), d))
        starts /= np.linalg.norm(starts, axis=1, keepdims=True)
        xt = t.empty_like(x)
        perm = t.empty(n, dtype=t.int64, device=x.device)
        dirs = t.zeros((max(nint, 1), d), dtype=t.float64, device=x.device)
        vals = t.zeros(max(nint, 1), dtype=t.float64, device=x.device)
        N.call("hks_build_tree", N.ptr(x), n, d, depth, 0, N.ptr(N.to_device(starts)), N.ptr(xt), N.ptr(perm),
               N.ptr(dirs), N.ptr(vals), N.stream_ptr())
        ip = t.empty((n, k), dtype=t.int64, device=x.device)
        dp = t.empty((n, k), dtype=t.float64, device=x.device)
        N.call("hks_knn_segments", N.ptr(xt), n, d, k, seg.ctypes.data_as(N._I64P), len(seg) - 1, N.ptr(perm),
               N.ptr(ip), N.ptr(dp), N.stream_ptr())
        ti = t.empty_like(ip)
        td = t.empty_like(dp)
        ti[perm] = ip  # rows back to the point set's order
        td[perm] = dp
        if best_i is None:
            best_i, best_d = ti, td
            continue
        oi, od = t.empty_like(ti), t.empty_like(td)
        N.call("hks_knn_merge", N.ptr(best_i), N.ptr(best_d), N.ptr(ti), N.ptr(td), n, k, N.ptr(oi), N.ptr(od),
               N.stream_ptr())
        best_i, best_d = oi, od
    return DeviceArray(best_i)
