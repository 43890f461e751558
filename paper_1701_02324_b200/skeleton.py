"""Nested skeletonization on the GPU (skeleton.py of the reference).

Per tree level (bottom-up, root excluded; skeleton.py:171-181) every node's
row sample, the sampled kernel block K(X[rows], X[cands]), the truncated
column-pivoted QR and the interpolative decomposition run as one batched
level program in libhks (csrc/sample.cu, csrc/qrcp.cu).  Random draws stay
host numpy with the reference's keyed streams ``default_rng([seed, 3,
node])`` (skeleton.py:106) so they are bit-identical; the kNN union /
complement bookkeeping is a device bitmap.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .tree import PartitionTree, levels

SAMPLE_MODES = ("uniform", "knn_augmented", "exact")


@dataclass(frozen=True)
class Skeleton:
    node: int
    indices: np.ndarray
    interp: np.ndarray

    @property
    def rank(self):
        return self.indices.shape[0]


@dataclass(frozen=True)
class SkeletonConfig:
    tau: float = 1e-5
    max_rank: int = 64
    samples: int = 256
    sample_mode: str = "uniform"
    seed: int = 0

    def __post_init__(self):
        if self.tau <= 0:
            raise ValueError("tau must be positive")
        if self.max_rank < 1:
            raise ValueError("max_rank must be >= 1")
        if self.samples < 1:
            raise ValueError("samples must be >= 1")
        if self.sample_mode not in SAMPLE_MODES:
            raise ValueError(f"unknown sample mode {self.sample_mode!r}")


class SkeletonSet:
    """Skeletons of every non-root node, stored in the flat device layout
    (HKS_BUF_INTERP / HKS_BUF_SKEL); ``skels[i]`` materialises the host view."""

    def __init__(self, tree, config, layout, interp, skel, ranks, rows_count=None):
        self.tree = tree
        self.config = config
        self.layout = layout
        self.interp_buf = interp
        self.skel_buf = skel
        self.ranks = np.asarray(ranks, dtype=np.int64)
        self.rows_count = rows_count
        self._cache = {}

    @property
    def skeletons(self):
        return {i: self[i] for i in range(1, self.layout.nn)}

    def _interp_dev(self, i):
        r = int(self.ranks[i])
        c = self.candidates_count(i)
        off = int(self.layout.off[N.BUF_INTERP, i])
        return self.interp_buf[off: off + r * c].view(c, r).t() if r and c else None

    def candidates_count(self, i):
        if i >= (1 << self.layout.depth) - 1:
            return int(self.tree._end[i] - self.tree._begin[i])
        return int(self.ranks[2 * i + 1] + self.ranks[2 * i + 2])

    def __getitem__(self, i):
        i = int(i)
        if i not in self:
            raise KeyError(i)
        if i not in self._cache:
            r, c = int(self.ranks[i]), self.candidates_count(i)
            so = int(self.layout.off[N.BUF_SKEL, i])
            idx = self.skel_buf[so: so + r].cpu().numpy().astype(np.int64)
            p = self._interp_dev(i)
            p = p.cpu().numpy() if p is not None else np.zeros((r, c))
            self._cache[i] = Skeleton(node=i, indices=idx, interp=np.ascontiguousarray(p))
        return self._cache[i]

    def __len__(self):
        return self.layout.nn - 1

    def __contains__(self, i):
        return 1 <= int(i) < self.layout.nn

    def max_rank_per_level(self, tree=None):
        out = {}
        for lev in range(1, self.layout.depth + 1):
            first = (1 << lev) - 1
            out[lev] = int(self.ranks[first: 2 * first + 1].max())
        return out

    @classmethod
    def from_host(cls, tree, skel_dict, config):
        """Upload externally computed skeletons {node: (indices, interp)}
        (tests feed the oracle's skeletons to isolate the factorization)."""
        lay = N.Layout(tree.n, tree.depth, config.max_rank)
        interp = lay.alloc(N.BUF_INTERP)
        skel = lay.alloc(N.BUF_SKEL)
        ranks = np.zeros(lay.nn, dtype=np.int64)
        hi = np.zeros(int(lay.sizes[N.BUF_INTERP]) or 1)
        hs = np.zeros(int(lay.sizes[N.BUF_SKEL]) or 1, dtype=np.int64)
        for i, (idx, p) in skel_dict.items():
            p = np.asarray(p, dtype=np.float64)
            r = p.shape[0]
            ranks[i] = r
            oi, os_ = int(lay.off[N.BUF_INTERP, i]), int(lay.off[N.BUF_SKEL, i])
            hi[oi: oi + p.size] = p.T.ravel()  # column-major, ld r
            hs[os_: os_ + r] = idx
        interp.copy_(N.torch().from_numpy(hi).to(interp.device))
        skel.copy_(N.torch().from_numpy(hs).to(skel.device))
        return cls(tree, config, lay, interp, skel, ranks)


# ----------------------------------------------------------------- sampling

def sample_rows(tree, node, ell, mode, seed, knn=None):
    """Row indices for skeletonizing ``node`` (skeleton.py:84-122), host
    semantics; the level-batched device version lives in build_skeletons."""
    if ell < 1:
        raise ValueError("ell must be >= 1")
    n = tree.n
    begin, end = node.begin, node.end
    size = end - begin
    comp = n - size
    if comp == 0:
        raise ValueError("node covers the whole point set; no rows to sample")
    if mode == "exact":
        return np.concatenate([np.arange(begin), np.arange(end, n)])
    ell = min(ell, comp)
    rng = np.random.default_rng([int(seed), 3, int(node.index)])
    if mode == "uniform":
        draw = rng.choice(comp, size=ell, replace=False)
        draw[draw >= begin] += size
        return np.sort(draw)
    if mode == "knn_augmented":
        if knn is None:
            raise ValueError("knn_augmented sampling needs precomputed kNN lists")
        nb = np.unique(np.asarray(knn[begin:end]).ravel())
        base = nb[(nb < begin) | (nb >= end)]
        if base.size >= ell:
            return base
        rest = np.setdiff1d(np.concatenate([np.arange(begin), np.arange(end, n)]), base,
                            assume_unique=True)
        extra = rng.choice(rest.size, size=ell - base.size, replace=False)
        return np.sort(np.concatenate([base, rest[extra]]))
    raise ValueError(f"unknown sample mode {mode!r}")


def _level_rows(tree, level, config, knn_dev):
    """Device row lists for every node of one level: flat int64 tensor + host
    offsets.  knn_augmented: device bitmap union of the nodes' neighbour lists
    minus the node range, host RNG top-up when short (skeleton.py:111-121)."""
    t = N.torch()
    first, count = (1 << level) - 1, 1 << level
    n = tree.n
    begin, end = tree._begin[first:first + count], tree._end[first:first + count]
    mode, ell, seed = config.sample_mode, config.samples, config.seed
    if mode in ("exact", "uniform"):
        lists = []
        for j in range(count):
            b, e = int(begin[j]), int(end[j])
            size, comp = e - b, n - (e - b)
            if comp == 0:
                raise ValueError("node covers the whole point set; no rows to sample")
            if mode == "exact":
                lists.append(np.concatenate([np.arange(b), np.arange(e, n)]))
            else:
                rng = np.random.default_rng([int(seed), 3, first + j])
                draw = rng.choice(comp, size=min(ell, comp), replace=False)
                draw[draw >= b] += size
                lists.append(np.sort(draw))
        off = np.zeros(count + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(x) for x in lists])
        return N.to_device(np.concatenate(lists).astype(np.int64)), off
    # knn_augmented on the device
    kappa = int(knn_dev.shape[1])
    words = (n + 31) // 32
    bitmap = t.zeros(count * words, dtype=t.int32, device=knn_dev.device)
    counts = np.zeros(count, dtype=np.int64)
    N.call("hks_knn_rows_mark", N.ptr(knn_dev), n, kappa, level, tree.depth, N.ptr(bitmap),
           counts.ctypes.data_as(N._I64P), N.stream_ptr())
    extra_lists, extra_off = [], np.zeros(count + 1, dtype=np.int64)
    final = counts.copy()
    for j in range(count):
        size = int(end[j] - begin[j])
        comp = n - size
        if comp == 0:
            raise ValueError("node covers the whole point set; no rows to sample")
        want = min(ell, comp)
        if counts[j] < want:
            rng = np.random.default_rng([int(seed), 3, first + j])
            extra = rng.choice(comp - int(counts[j]), size=want - int(counts[j]), replace=False)
            extra_lists.append(np.asarray(extra, dtype=np.int64))
            final[j] = want
        else:
            extra_lists.append(np.zeros(0, dtype=np.int64))
        extra_off[j + 1] = extra_off[j] + extra_lists[-1].size
    off = np.zeros(count + 1, dtype=np.int64)
    off[1:] = np.cumsum(final)
    rows = t.empty(max(int(off[-1]), 1), dtype=t.int64, device=knn_dev.device)
    extra = N.to_device(np.concatenate(extra_lists) if extra_off[-1] else np.zeros(1, dtype=np.int64))
    N.call("hks_knn_rows_fill", n, level, tree.depth, N.ptr(bitmap), N.ptr(extra),
           extra_off.ctypes.data_as(N._I64P), N.ptr(rows), off.ctypes.data_as(N._I64P), N.stream_ptr())
    return rows, off


def build_skeletons(tree, kernel, config=None, knn=None, threads=1):
    """Skeletonize every non-root node, leaves first (skeleton.py:143-182).
    ``threads`` is accepted for API parity; the GPU batches each level."""
    config = config or SkeletonConfig()
    if config.sample_mode == "knn_augmented" and knn is None:
        raise ValueError("knn_augmented sampling needs precomputed kNN lists")
    t = N.torch()
    lay = N.Layout(tree.n, tree.depth, config.max_rank)
    interp = lay.alloc(N.BUF_INTERP)
    skel = lay.alloc(N.BUF_SKEL)
    ranks = np.zeros(lay.nn, dtype=np.int64)
    rows_count = np.zeros(lay.nn, dtype=np.int64)
    x = tree.device_points()
    knn_dev = None
    if config.sample_mode == "knn_augmented":
        knn_dev = knn.device if hasattr(knn, "device") and not isinstance(knn, np.ndarray) else \
            N.to_device(np.asarray(knn, dtype=np.int64))
        knn_dev = knn_dev.contiguous()
    kern = N.kernel_struct(kernel)
    for level in range(tree.depth, 0, -1):
        first, count = (1 << level) - 1, 1 << level
        rows, roff = _level_rows(tree, level, config, knn_dev)
        rows_count[first:first + count] = np.diff(roff)
        if level == tree.depth:
            cands = t.arange(tree.n, dtype=t.int64, device=x.device)
            coff = np.concatenate([tree._begin[first:first + count], [tree.n]]).astype(np.int64)
        else:
            parts, coff = [], np.zeros(count + 1, dtype=np.int64)
            for j in range(count):
                i = first + j
                for ch in (2 * i + 1, 2 * i + 2):
                    so, r = int(lay.off[N.BUF_SKEL, ch]), int(ranks[ch])
                    parts.append(skel[so: so + r])
                coff[j + 1] = coff[j] + ranks[2 * i + 1] + ranks[2 * i + 2]
            cands = t.cat(parts) if coff[-1] else t.zeros(1, dtype=t.int64, device=x.device)
        out_ranks = np.zeros(count, dtype=np.int64)
        rc = N.fn("hks_skeletonize_level")(
            N.ptr(x), tree.d, ctypes.byref(kern), count, first,
            N.ptr(rows), roff.ctypes.data_as(N._I64P), N.ptr(cands), coff.ctypes.data_as(N._I64P),
            float(config.tau), int(config.max_rank),
            N.ptr(skel), np.ascontiguousarray(lay.off[N.BUF_SKEL, first:first + count]).ctypes.data_as(N._I64P),
            N.ptr(interp), np.ascontiguousarray(lay.off[N.BUF_INTERP, first:first + count]).ctypes.data_as(N._I64P),
            out_ranks.ctypes.data_as(N._I64P), N.stream_ptr())
        if rc != N.HKS_OK:
            msg = N.last_error()
            node = int(msg.split("node ")[1].split()[0]) if "node " in msg else first
            raise RuntimeError(f"skeletonization failed at node {node} (level {level})") from \
                N.HksError(rc, msg)
        ranks[first:first + count] = out_ranks
    N.call("hks_skeleton_workspace_release", N.stream_ptr())
    return SkeletonSet(tree, config, lay, interp, skel, ranks, rows_count)


N.SIGNATURES.update({
    "hks_knn_rows_mark": [N._P, N._I64, N._I64, N._I64, N._I64, N._P, N._I64P, N._P],
    "hks_knn_rows_fill": [N._I64, N._I64, N._I64, N._P, N._P, N._I64P, N._P, N._I64P, N._P],
    "hks_skeletonize_level": [N._P, N._I64, N._KP, N._I64, N._I64, N._P, N._I64P, N._P, N._I64P,
                              N._D, N._I64, N._P, N._I64P, N._P, N._I64P, N._I64P, N._P],
    "hks_skeleton_workspace_release": [N._P],
})
