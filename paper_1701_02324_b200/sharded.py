"""Subtree-sharded setup, factorization, solve and matvec over P = 2^p ranks
(SURVEY.md section 8(e)).  One process per GPU; the collectives go through
``torch.distributed`` (NCCL over NVLink between B200s).

The global tree is split at level p: rank q owns the subtree rooted at heap
node 2^p - 1 + q (a contiguous block of tree-ordered points).  Everything at
levels >= p is rank-local -- kNN rows of the shard's points, row sampling,
skeletonization, leaf / internal factorization, the up and down sweeps --
and runs through a HKS_PLAN_SUBTREE plan whose root keeps its skeleton,
Theta and push.  Levels 0..p-1 (2^p - 1 nodes) are computed redundantly on
every rank by a HKS_PLAN_TOP plan whose leaves are the shard roots.  The
only data exchanged (all-gathers, the shard roots' blocks landing straight
in the top plan's layout):

  * setup: shard-root ranks and skeleton indices; for each top node the OR
    of the ranks' knn_augmented row bitmaps (skeleton.py:111-121 over a node
    that spans several shards);
  * factorize: the shard roots' Theta (s x s each), solver.py:139-143;
  * solve / hmatvec: the shard roots' psi / skeleton weights going up and
    nothing coming down -- every rank evaluates the top levels itself and
    keeps its own root's correction (solver.py:219-253, treecode.py:83-123).

The reference (pkg/src/hikersolve) is single-process; with the same seed
the sharded path produces the same tree, kNN lists, skeletons and
factors as the unsharded one, node for node (tests/test_gpu_sharded.py).
The tree itself (tree.py:87-144) is built redundantly on every rank: each
rank needs every point anyway (kNN candidates, sampled rows and skeleton
columns are global indices).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native as N
from .linalg import SingularMatrixError
from .skeleton import Skeleton
from .solver import FactorizationError, _FACTOR_BUFS
from .tree import node_ranges


# ------------------------------------------------------------ collectives

class ShardComm:
    """The sharded path's collectives over a torch.distributed group
    (NCCL for CUDA tensors between GPUs; gloo, staged through host memory,
    for tests).  Without an initialised process group it is a one-rank
    group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, None

    def all_gather(self, out, inp):
        """out (flat, world * inp.numel()) <- every rank's inp in rank order."""
        inp = inp.reshape(-1)
        if out.numel() != self.world * inp.numel():
            raise ValueError("all_gather: output must hold world * input elements")
        if self.world == 1:
            out.copy_(inp)
        elif self.backend == "nccl":
            self._dist.all_gather_into_tensor(out, inp.contiguous(), group=self.group)
        else:
            h = inp.detach().cpu()
            parts = [N.torch().empty_like(h) for _ in range(self.world)]
            self._dist.all_gather(parts, h, group=self.group)
            out.copy_(N.torch().cat(parts).to(out.device))
        return out

    def all_reduce_max(self, value):
        """Max over ranks of a host integer (error flags)."""
        if self.world == 1:
            return int(value)
        t = N.torch()
        dev = N.device() if self.backend == "nccl" else "cpu"
        v = t.tensor([int(value)], dtype=t.int64, device=dev)
        self._dist.all_reduce(v, op=self._dist.ReduceOp.MAX, group=self.group)
        return int(v.item())

    def all_reduce_sum_(self, tensor):
        """In-place sum over ranks (the sharded GMRES inner products)."""
        if self.world == 1:
            return tensor
        if self.backend == "nccl":
            self._dist.all_reduce(tensor, group=self.group)
        else:
            h = tensor.detach().cpu()
            self._dist.all_reduce(h, group=self.group)
            tensor.copy_(h.to(tensor.device))
        return tensor


# ------------------------------------------------------------ geometry

def _level(i):
    return int(i + 1).bit_length() - 1


class ShardSpec:
    """Which part of the global tree (n points, depth) rank `rank` of
    `world` owns.  Host-only arithmetic (tests/test_multiproc.py)."""

    def __init__(self, n, depth, world, rank):
        world, rank = int(world), int(rank)
        if world < 2 or world & (world - 1):
            raise ValueError(f"subtree sharding needs a power-of-two number of ranks >= 2 (got {world})")
        p = world.bit_length() - 1
        if p > depth:
            raise ValueError(f"{world} shards need a tree of depth >= {p} (got depth {depth})")
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside [0, {world})")
        self.n, self.depth, self.world, self.rank, self.p = int(n), int(depth), world, rank, p
        self.begins, self.ends = node_ranges(self.n, self.depth)
        self.root = (1 << p) - 1 + rank
        self.begin, self.end = int(self.begins[self.root]), int(self.ends[self.root])
        self.local_depth = self.depth - p
        self.shard_sizes = (self.ends - self.begins)[(1 << p) - 1: (1 << (p + 1)) - 1]

    @property
    def size(self):
        return self.end - self.begin

    def global_node(self, j):
        """Local heap index j of this shard's subtree -> global heap index."""
        ell = _level(j)
        return (1 << (self.p + ell)) - 1 + (self.rank << ell) + (j - ((1 << ell) - 1))

    def local_node(self, i):
        """Global heap index -> local heap index (None outside the shard)."""
        lev = _level(i)
        if lev < self.p:
            return None
        ell = lev - self.p
        pos = i - ((1 << lev) - 1)
        if pos >> ell != self.rank:
            return None
        return (1 << ell) - 1 + (pos - (self.rank << ell))

    def owner(self, i):
        """Rank owning global node i (None for the replicated top levels)."""
        lev = _level(i)
        if lev < self.p:
            return None
        return (i - ((1 << lev) - 1)) >> (lev - self.p)


def or_reduce_bitmaps(gathered, world):
    """OR of `world` equal-length int32 bitmaps stacked in `gathered`."""
    parts = gathered.view(world, -1)
    out = parts[0].clone()
    for q in range(1, world):
        out.bitwise_or_(parts[q])
    return out


# ------------------------------------------------------------ setup

def knn_shard(tree, k, spec):
    """kNN lists (tree.py:163-188) of the shard's points against all n
    points, global indices: (n_shard, k) int64 on the device."""
    t = N.torch()
    n = tree.n
    if not 1 <= k <= n - 1:
        raise ValueError("need 1 <= k <= n - 1")
    x = tree.device_points()
    out = t.empty((spec.size, k), dtype=t.int64, device=x.device)
    N.call("hks_knn_rows", N.ptr(x), n, tree.d, k, spec.begin, spec.size, N.ptr(out), N.stream_ptr())
    return out


def _rows(spec, level, node0, count, config, knn_local, comm, combine):
    """Sampled rows (skeleton.py:84-122) of the nodes [node0, node0 + count)
    of `level`: flat device int64 list + host offsets.  combine: the nodes
    span several shards, so the knn_augmented bitmaps are OR-ed over ranks."""
    t = N.torch()
    n = spec.n
    first = (1 << level) - 1
    ids = first + node0 + np.arange(count)
    begin, end = spec.begins[ids], spec.ends[ids]
    mode, ell, seed = config.sample_mode, config.samples, config.seed
    if mode in ("exact", "uniform"):
        lists = []
        for j in range(count):
            b, e = int(begin[j]), int(end[j])
            size, comp = e - b, n - (e - b)
            if mode == "exact":
                lists.append(np.concatenate([np.arange(b), np.arange(e, n)]))
            else:
                rng = np.random.default_rng([int(seed), 3, int(ids[j])])
                draw = rng.choice(comp, size=min(ell, comp), replace=False)
                draw[draw >= b] += size
                lists.append(np.sort(draw))
        off = np.zeros(count + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(x) for x in lists])
        return N.to_device(np.concatenate(lists).astype(np.int64)), off
    kappa = int(knn_local.shape[1])
    words = (n + 31) // 32
    bitmap = t.zeros(count * words, dtype=t.int32, device=knn_local.device)
    counts = np.zeros(count, dtype=np.int64)
    N.call("hks_knn_rows_mark_ex", N.ptr(knn_local), spec.begin, spec.size, n, kappa, level, node0, count,
           N.ptr(bitmap), counts.ctypes.data_as(N._I64P), N.stream_ptr())
    if combine and comm.world > 1:
        gathered = t.empty(comm.world * bitmap.numel(), dtype=t.int32, device=bitmap.device)
        comm.all_gather(gathered, bitmap)
        bitmap = or_reduce_bitmaps(gathered, comm.world)
        N.call("hks_bitmap_count", N.ptr(bitmap), n, count, counts.ctypes.data_as(N._I64P), N.stream_ptr())
    extra_lists, extra_off = [], np.zeros(count + 1, dtype=np.int64)
    final = counts.copy()
    for j in range(count):
        comp = n - int(end[j] - begin[j])
        want = min(ell, comp)
        if counts[j] < want:
            rng = np.random.default_rng([int(seed), 3, int(ids[j])])
            extra = rng.choice(comp - int(counts[j]), size=want - int(counts[j]), replace=False)
            extra_lists.append(np.asarray(extra, dtype=np.int64))
            final[j] = want
        else:
            extra_lists.append(np.zeros(0, dtype=np.int64))
        extra_off[j + 1] = extra_off[j] + extra_lists[-1].size
    off = np.zeros(count + 1, dtype=np.int64)
    off[1:] = np.cumsum(final)
    rows = t.empty(max(int(off[-1]), 1), dtype=t.int64, device=knn_local.device)
    extra = N.to_device(np.concatenate(extra_lists) if extra_off[-1] else np.zeros(1, dtype=np.int64))
    N.call("hks_knn_rows_fill_ex", n, level, node0, count, N.ptr(bitmap), N.ptr(extra),
           extra_off.ctypes.data_as(N._I64P), N.ptr(rows), off.ctypes.data_as(N._I64P), N.stream_ptr())
    return rows, off


def _skeletonize(x, d, kern, level, first_global, rows, roff, cands, coff, config, skel, interp, lay, local_ids):
    count = len(local_ids)
    out_ranks = np.zeros(count, dtype=np.int64)
    rc = N.fn("hks_skeletonize_level")(
        N.ptr(x), d, ctypes.byref(kern), count, first_global,
        N.ptr(rows), roff.ctypes.data_as(N._I64P), N.ptr(cands), coff.ctypes.data_as(N._I64P),
        float(config.tau), int(config.max_rank),
        N.ptr(skel), np.ascontiguousarray(lay.off[N.BUF_SKEL, local_ids]).ctypes.data_as(N._I64P),
        N.ptr(interp), np.ascontiguousarray(lay.off[N.BUF_INTERP, local_ids]).ctypes.data_as(N._I64P),
        out_ranks.ctypes.data_as(N._I64P), N.stream_ptr())
    if rc != N.HKS_OK:
        msg = N.last_error()
        node = int(msg.split("node ")[1].split()[0]) if "node " in msg else first_global
        raise RuntimeError(f"skeletonization failed at node {node} (level {level})") from N.HksError(rc, msg)
    return out_ranks


def _candidates(skel, lay, ranks, local_ids, device):
    t = N.torch()
    parts, coff = [], np.zeros(len(local_ids) + 1, dtype=np.int64)
    for j, i in enumerate(local_ids):
        for ch in (2 * i + 1, 2 * i + 2):
            so, r = int(lay.off[N.BUF_SKEL, ch]), int(ranks[ch])
            parts.append(skel[so: so + r])
        coff[j + 1] = coff[j] + ranks[2 * i + 1] + ranks[2 * i + 2]
    cands = t.cat(parts) if coff[-1] else t.zeros(1, dtype=t.int64, device=device)
    return cands, coff


class ShardedSkeletons:
    """Skeletons of one rank's subtree (HKS_PLAN_SUBTREE layout, indices
    local to the shard) and of the replicated top levels (HKS_PLAN_TOP
    layout, global indices).  ``sk[i]`` (global heap index) materialises a
    Skeleton with global indices for every node this rank holds."""

    def __init__(self, spec, config, local_layout, local_interp, local_skel, local_skel_global, local_ranks,
                 top_layout, top_interp, top_skel, top_ranks):
        self.spec, self.config = spec, config
        self.local_layout, self.local_interp = local_layout, local_interp
        self.local_skel, self.local_skel_global = local_skel, local_skel_global
        self.local_ranks = np.asarray(local_ranks, dtype=np.int64)
        self.top_layout, self.top_interp, self.top_skel = top_layout, top_interp, top_skel
        self.top_ranks = np.asarray(top_ranks, dtype=np.int64)

    def rank_of(self, i):
        j = self.spec.local_node(i)
        if j is not None:
            return int(self.local_ranks[j])
        if _level(i) < self.spec.p:
            return int(self.top_ranks[i])
        if _level(i) == self.spec.p:
            return int(self.top_ranks[i])
        raise KeyError(i)

    def __contains__(self, i):
        i = int(i)
        return i >= 1 and (_level(i) <= self.spec.p or self.spec.local_node(i) is not None) and \
            i < (1 << (self.spec.depth + 1)) - 1

    def __getitem__(self, i):
        i = int(i)
        if i not in self:
            raise KeyError(i)
        j = self.spec.local_node(i)
        if j is not None:
            lay, ranks, skel, interp, ii = self.local_layout, self.local_ranks, self.local_skel_global, \
                self.local_interp, j
        elif _level(i) < self.spec.p:
            lay, ranks, skel, interp, ii = self.top_layout, self.top_ranks, self.top_skel, self.top_interp, i
        else:  # another rank's shard root: indices only
            r = int(self.top_ranks[i])
            so = int(self.top_layout.off[N.BUF_SKEL, i])
            return Skeleton(node=i, indices=self.top_skel[so: so + r].cpu().numpy().astype(np.int64),
                            interp=np.zeros((r, 0)))
        r = int(ranks[ii])
        if lay.mode == N.PLAN_SUBTREE and ii >= (1 << lay.depth) - 1:
            b, e = node_ranges(lay.n, lay.depth)
            c = int(e[ii] - b[ii])
        else:
            c = int(ranks[2 * ii + 1] + ranks[2 * ii + 2])
        so, io = int(lay.off[N.BUF_SKEL, ii]), int(lay.off[N.BUF_INTERP, ii])
        idx = skel[so: so + r].cpu().numpy().astype(np.int64)
        p = interp[io: io + r * c].view(c, r).t().cpu().numpy() if r and c else np.zeros((r, c))
        return Skeleton(node=i, indices=idx, interp=np.ascontiguousarray(p))


def agree_on_failure(comm, local_error, message):
    """Collective error agreement before a rank's next collective: every
    rank learns whether any rank failed (max over ranks of 1 + the failing
    rank), so none blocks in an all-gather while another raises.  The
    failing rank re-raises its own exception; the others raise
    RuntimeError(message.format(rank=<failing rank>))."""
    worst = comm.all_reduce_max(0 if local_error is None else 1 + comm.rank)
    if local_error is not None:
        raise local_error
    if worst:
        raise RuntimeError(message.format(rank=worst - 1))


def build_skeletons_sharded(tree, kernel, config, knn_local, spec, comm):
    """build_skeletons (skeleton.py:143-182) over a sharded tree: the shard's
    levels locally, the shard roots' ranks / indices all-gathered, the top
    levels redundantly on every rank."""
    if config.sample_mode == "knn_augmented" and knn_local is None:
        raise ValueError("knn_augmented sampling needs precomputed kNN lists")
    t = N.torch()
    x = tree.device_points()
    kern = N.kernel_struct(kernel)
    s = int(config.max_rank)
    lay = N.Layout(spec.size, spec.local_depth, s, N.PLAN_SUBTREE)
    interp = lay.alloc(N.BUF_INTERP)
    skel = lay.alloc(N.BUF_SKEL, min_elems=s)
    skel.zero_()
    ranks = np.zeros(lay.nn, dtype=np.int64)
    lbeg, _ = node_ranges(spec.size, spec.local_depth)
    local_error = None
    try:  # shard levels: no collective inside, so a failure is agreed on below before the first one
        for ell in range(spec.local_depth, -1, -1):
            level = spec.p + ell
            node0, count = spec.rank << ell, 1 << ell
            local_ids = np.arange((1 << ell) - 1, (1 << (ell + 1)) - 1)
            rows, roff = _rows(spec, level, node0, count, config, knn_local, comm, combine=False)
            if ell == spec.local_depth:
                cands = t.arange(spec.begin, spec.end, dtype=t.int64, device=x.device)
                coff = np.concatenate([lbeg[local_ids], [spec.size]]).astype(np.int64)
            else:
                cands, coff = _candidates(skel, lay, ranks, local_ids, x.device)
            ranks[local_ids] = _skeletonize(x, tree.d, kern, level, (1 << level) - 1 + node0, rows, roff, cands,
                                            coff, config, skel, interp, lay, local_ids)
    except (RuntimeError, ValueError) as exc:
        local_error = exc
    agree_on_failure(comm, local_error, f"skeletonization failed on rank {{rank}} (shard levels {spec.p}..{spec.depth})")
    # shard roots -> the top plan's leaves (ranks, then s-padded index blocks)
    P = comm.world
    root_ranks = t.empty(P, dtype=t.int64, device=x.device)
    comm.all_gather(root_ranks, t.tensor([int(ranks[0])], dtype=t.int64, device=x.device))
    top = N.Layout(spec.n, spec.p, s, N.PLAN_TOP)
    top_interp = top.alloc(N.BUF_INTERP)
    top_skel = top.alloc(N.BUF_SKEL)
    comm.all_gather(top_skel[: P * s], skel[:s])
    top_ranks = np.zeros(top.nn, dtype=np.int64)
    top_ranks[(1 << spec.p) - 1:] = root_ranks.cpu().numpy()
    for level in range(spec.p - 1, 0, -1):
        count = 1 << level
        ids = np.arange((1 << level) - 1, (1 << (level + 1)) - 1)
        rows, roff = _rows(spec, level, 0, count, config, knn_local, comm, combine=True)
        cands, coff = _candidates(top_skel, top, top_ranks, ids, x.device)
        top_ranks[ids] = _skeletonize(x, tree.d, kern, level, int(ids[0]), rows, roff, cands, coff, config,
                                      top_skel, top_interp, top, ids)
    N.call("hks_skeleton_workspace_release", N.stream_ptr())
    local_skel = skel - spec.begin  # the subtree plan evaluates on the shard's own points
    return ShardedSkeletons(spec, config, lay, interp, local_skel, skel, ranks, top, top_interp, top_skel,
                            top_ranks)


# ------------------------------------------------------------ operator

class _ModePlan:
    """Owner of one hks_plan* of a given mode, with its dgecon stream."""

    def __init__(self, x, n, d, depth, s, ranks, kern_struct, mode):
        self.kern = kern_struct
        self.handle = ctypes.c_void_p()
        self._x = x
        r = np.ascontiguousarray(ranks, dtype=np.int64)
        N.call("hks_plan_create_ex", ctypes.byref(self.handle), N.ptr(x), n, d, depth, s,
               r.ctypes.data_as(N._I64P), ctypes.byref(self.kern), mode)
        self.cond_stream = N.torch().cuda.Stream(device=N.device(), priority=0)
        N.call("hks_set_cond_stream", self.handle, ctypes.c_void_p(self.cond_stream.cuda_stream))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and N._lib is not None:
            N._lib.hks_plan_destroy(h)
            self.handle = None


def _bufs(extra):
    b = [None] * N.NBUF
    for k, v in extra.items():
        b[k] = v
    return N.buffers_array(b)


class ShardedOperator:
    """build_operator (treecode.py:41-62) of a sharded tree: the subtree
    plan's couplings from the shard's skeletons, the top plan's from the
    replicated top skeletons."""

    def __init__(self, tree, skeletons, kernel, comm):
        sk = skeletons
        spec = sk.spec
        self.tree, self.skeletons, self.kernel, self.comm, self.spec = tree, sk, kernel, comm, spec
        s = int(sk.config.max_rank)
        self.s = s
        x = tree.device_points()
        self._x_local = x[spec.begin: spec.end]
        kern = N.kernel_struct(kernel)
        self.local = _ModePlan(self._x_local, spec.size, tree.d, spec.local_depth, s, sk.local_ranks, kern,
                               N.PLAN_SUBTREE)
        self.top = _ModePlan(x, spec.n, tree.d, spec.p, s, sk.top_ranks, kern, N.PLAN_TOP)
        self.local_coup = sk.local_layout.alloc(N.BUF_COUP)
        self.top_coup = sk.top_layout.alloc(N.BUF_COUP)
        N.call("hks_build_operator", self.local.handle, self.local_buffers(), N.stream_ptr())
        from .treecode import cache_leaf_blocks
        self.leaf_cache = cache_leaf_blocks(self.local.handle, spec.size, int(tree._end[-1] - tree._begin[-1]))
        N.call("hks_build_operator", self.top.handle, self.top_buffers(), N.stream_ptr())

    @property
    def n(self):
        return self.tree.n

    def local_buffers(self, extra=None):
        sk = self.skeletons
        return _bufs({N.BUF_INTERP: sk.local_interp, N.BUF_SKEL: sk.local_skel, N.BUF_COUP: self.local_coup,
                      **(extra or {})})

    def top_buffers(self, extra=None):
        sk = self.skeletons
        return _bufs({N.BUF_INTERP: sk.top_interp, N.BUF_SKEL: sk.top_skel, N.BUF_COUP: self.top_coup,
                      **(extra or {})})

    def matvec_local(self, W, lam):
        return hmatvec_sharded(self, W, lam)


def build_operator_sharded(tree, skeletons, kernel, comm):
    return ShardedOperator(tree, skeletons, kernel, comm)


# ------------------------------------------------------------ factorize / solve / matvec

def _raise_factor(rc, node_map):
    msg = N.last_error()
    if rc == N.HKS_ERR_SINGULAR:
        raise SingularMatrixError(msg)
    if rc == N.HKS_ERR_REDUCED_SINGULAR:
        raise FactorizationError(node_map(msg))
    raise N.HksError(rc, msg)


class ShardedFactorization:
    """One rank's part of factorize (solver.py:111-186) on a sharded tree:
    the shard's factors plus the replicated top levels."""

    def __init__(self, op, lam, local_bufs, top_bufs, level_seconds):
        self.op, self.lam = op, float(lam)
        self.local_bufs, self.top_bufs = local_bufs, top_bufs
        self.level_seconds = level_seconds
        self._zc = None

    def z_cond_per_level(self):
        """Max z_cond per level; levels >= p over this rank's shard only."""
        op, spec = self.op, self.op.spec
        zl = np.zeros(op.skeletons.local_layout.nn)
        zt = np.zeros(op.skeletons.top_layout.nn)
        N.call("hks_factor_stats", op.local.handle, op.local_buffers(self.local_bufs), zl.ctypes.data_as(N._DP),
               None, N.stream_ptr())
        N.call("hks_factor_stats", op.top.handle, op.top_buffers(self.top_bufs), zt.ctypes.data_as(N._DP), None,
               N.stream_ptr())
        out = {}
        for lev in range(spec.p):
            out[lev] = float(zt[(1 << lev) - 1: (1 << (lev + 1)) - 1].max())
        for ell in range(spec.local_depth):
            out[spec.p + ell] = float(zl[(1 << ell) - 1: (1 << (ell + 1)) - 1].max())
        return out

    def solve_local(self, B):
        return solve_sharded(self, B)

    def join_cond(self):
        """The current stream waits for both plans' dgecon estimates."""
        N.call("hks_cond_wait", self.op.local.handle, N.stream_ptr())
        N.call("hks_cond_wait", self.op.top.handle, N.stream_ptr())


def factorize_sharded(op, lam, with_cond=True):
    """Shard levels on this rank, shard-root Theta all-gathered, top levels
    on every rank.  A singular block on any rank raises on every rank."""
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    sk, spec, comm, s = op.skeletons, op.spec, op.comm, op.s
    P = comm.world
    ll, tl = sk.local_layout, sk.top_layout
    if getattr(op, "_factor_pools", None) is None:  # reusable storage (solver.FactorStorage)
        from .solver import FactorStorage
        op._factor_pools = (FactorStorage(ll, op.local.cond_stream, {N.BUF_THETA: s * s}),
                            FactorStorage(tl, op.top.cond_stream))
    lease_l, lease_t = op._factor_pools[0].lease(), op._factor_pools[1].lease()
    lb, tb = lease_l.bufs, lease_t.bufs
    bad = ctypes.c_int64(-1)
    rc = N.fn("hks_factorize")(op.local.handle, op.local_buffers(lb), float(lam), int(bool(with_cond)),
                               ctypes.byref(bad), N.stream_ptr())
    local_msg = N.last_error() if rc != N.HKS_OK else ""
    worst = comm.all_reduce_max(rc)
    if rc != N.HKS_OK:
        def glob(msg):
            j = int(bad.value)
            if j >= 0 and "at node" in msg:
                i = spec.global_node(j)
                lev = _level(i)
                head, tail = msg.split("at node", 1)
                rest = tail.split(")", 1)[1] if ")" in tail else ""
                return f"{head}at node {i} (level {lev}){rest}"
            return msg
        msg = glob(local_msg)
        if rc == N.HKS_ERR_SINGULAR:
            raise SingularMatrixError(msg)
        if rc == N.HKS_ERR_REDUCED_SINGULAR:
            raise FactorizationError(msg)
        raise N.HksError(rc, msg)
    if worst != N.HKS_OK:
        raise FactorizationError(f"factorization failed on another rank (status {worst})")
    comm.all_gather(tb[N.BUF_THETA][: P * s * s], lb[N.BUF_THETA][: s * s])
    rc = N.fn("hks_factorize")(op.top.handle, op.top_buffers(tb), float(lam), int(bool(with_cond)),
                               ctypes.byref(bad), N.stream_ptr())
    if rc != N.HKS_OK:
        _raise_factor(rc, lambda m: m)
    ms_l = np.zeros(spec.local_depth + 1)
    ms_t = np.zeros(spec.p + 1)
    N.call("hks_factor_level_ms", op.local.handle, ms_l.ctypes.data_as(N._DP))
    N.call("hks_factor_level_ms", op.top.handle, ms_t.ctypes.data_as(N._DP))
    level_seconds = {lev: float(ms_t[lev]) * 1e-3 for lev in range(spec.p)}
    for ell in range(spec.local_depth + 1):
        level_seconds[spec.p + ell] = float(ms_l[ell]) * 1e-3
    fac = ShardedFactorization(op, lam, lb, tb, level_seconds)
    fac._leases = (lease_l, lease_t)  # the storage returns to the operator's pools with the factorization
    return fac


def _exchange_blocks(op, k):
    t = N.torch()
    P, s = op.comm.world, op.s
    xo = t.zeros(s * k, dtype=t.float64, device=N.device())
    tin = t.empty(P * s * k, dtype=t.float64, device=N.device())
    tout = t.empty(P * s * k, dtype=t.float64, device=N.device())
    return xo, tin, tout


def solve_sharded(f, B):
    """solve / solve_multi (solver.py:189-270) for this rank's rows: B is the
    (k, n_shard) device block of the shard's right-hand sides (tree order,
    column-major n_shard x k); returns the shard's rows of x, same layout."""
    op = f.op
    t = N.torch()
    B = B.reshape(-1, op.spec.size) if B.dim() == 1 else B
    if B.shape[1] != op.spec.size:
        raise ValueError(f"right-hand side block must have {op.spec.size} rows per column")
    B = B.to(t.float64).contiguous()
    k = B.shape[0]
    X = t.empty_like(B)
    xo, tin, tout = _exchange_blocks(op, k)
    lbufs, tbufs = op.local_buffers(f.local_bufs), op.top_buffers(f.top_bufs)
    N.call("hks_solve_part", op.local.handle, lbufs, N.ptr(B), N.ptr(X), k, 1, N.ptr(xo), N.stream_ptr())
    op.comm.all_gather(tin, xo)
    N.call("hks_solve_part", op.top.handle, tbufs, N.ptr(tin), N.ptr(tout), k, 0, None, N.stream_ptr())
    mine = tout[op.spec.rank * op.s * k:]
    N.call("hks_solve_part", op.local.handle, lbufs, N.ptr(B), N.ptr(X), k, 2, N.ptr(mine), N.stream_ptr())
    return X


def hmatvec_sharded(op, W, lam):
    """hmatvec (treecode.py:92-128) for this rank's rows: W (k, n_shard)
    device block -> U = rows of (Ktilde + lam I) w owned by this rank."""
    t = N.torch()
    W = W.reshape(-1, op.spec.size) if W.dim() == 1 else W
    if W.shape[1] != op.spec.size:
        raise ValueError(f"weight block must have {op.spec.size} rows per column")
    W = W.to(t.float64).contiguous()
    k = W.shape[0]
    U = t.empty_like(W)
    xo, tin, tout = _exchange_blocks(op, k)
    lbufs, tbufs = op.local_buffers(), op.top_buffers()
    N.call("hks_hmatvec_part", op.local.handle, lbufs, N.ptr(W), N.ptr(U), k, float(lam), 1, N.ptr(xo),
           N.stream_ptr())
    op.comm.all_gather(tin, xo)
    N.call("hks_hmatvec_part", op.top.handle, tbufs, N.ptr(tin), N.ptr(tout), k, float(lam), 0, None,
           N.stream_ptr())
    mine = tout[op.spec.rank * op.s * k:]
    N.call("hks_hmatvec_part", op.local.handle, lbufs, N.ptr(W), N.ptr(U), k, float(lam), 2, N.ptr(mine),
           N.stream_ptr())
    return U


def gather_rows(comm, spec, X):
    """All shards' (k, n_shard) blocks -> the full (k, n) block on every
    rank (shards may differ in size by one point: padded exchange)."""
    t = N.torch()
    k = X.shape[0]
    m = int(spec.shard_sizes.max())
    pad = t.zeros((k, m), dtype=X.dtype, device=X.device)
    pad[:, : X.shape[1]] = X
    out = t.empty(comm.world * k * m, dtype=X.dtype, device=X.device)
    comm.all_gather(out, pad)
    blocks = out.view(comm.world, k, m)
    return t.cat([blocks[q, :, : int(spec.shard_sizes[q])] for q in range(comm.world)], dim=1)


def cross_predict_sharded(kernel, test, op, w_local):
    """KRR prediction K(test, train) w (cli.py:415-422) over training
    points sharded by subtree: each rank sums its own shard's sources
    (``metrics.cross_sum`` on the shard's tree-ordered points, never storing
    K), then the P partial sums are all-gathered and added in rank order, so
    every rank returns the same (nq,) device vector, independent of the
    collective's reduction order.  ``w_local`` is this rank's slice of the
    tree-ordered weights (e.g. a row of ``solve_sharded``'s result)."""
    from .metrics import cross_sum
    from .tree import PointSet
    t = N.torch()
    spec, comm = op.spec, op.comm
    w = w_local.to(t.float64).reshape(1, -1).contiguous()
    if w.shape[1] != spec.size:
        raise ValueError(f"weights must have length {spec.size} on rank {spec.rank}")
    test = test if isinstance(test, PointSet) else PointSet(np.asarray(test, dtype=np.float64))
    xs = op._x_local.contiguous()
    return sum_in_rank_order(comm, cross_sum(kernel, test.device(), xs, w)[0])


def sum_in_rank_order(comm, part):
    """Every rank's `part` added in rank order ((p0 + p1) + p2 ...), the
    same bits on every rank whatever the backend's reduction order."""
    t = N.torch()
    part = part.contiguous()
    if comm.world == 1:
        return part
    out = t.empty(comm.world * part.numel(), dtype=part.dtype, device=part.device)
    comm.all_gather(out, part)
    blocks = out.view(comm.world, *part.shape)
    acc = blocks[0].clone()
    for q in range(1, comm.world):
        acc += blocks[q]
    return acc


def timed_setup(fn):
    t0 = time.perf_counter()
    out = fn()
    N.torch().cuda.synchronize()
    return out, time.perf_counter() - t0
