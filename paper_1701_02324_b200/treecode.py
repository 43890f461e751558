"""Compressed operator and the treecode matvec on the GPU (treecode.py of
the reference).

``build_operator`` evaluates the sibling couplings K(q_l, q_r) into the
flat layout (one batched launch) and creates the level program (hks_plan)
that ``hmatvec`` / ``upward_pass`` / ``factorize`` replay.  Leaf blocks are
not stored: hmatvec's leaf level is the fused kernel-summation kernel and
factorize re-evaluates K_aa + lam I straight into its LU storage;
``op.leaf_blocks`` materialises them on demand for diagnostics.
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping

import numpy as np

from . import _native as N

MATERIALIZE_MAX_POINTS = 4096


class Plan:
    """Owner of one hks_plan* (destroyed with the Python object)."""

    def __init__(self, tree, skeletons, kernel):
        self.kern = N.kernel_struct(kernel)
        self.handle = ctypes.c_void_p()
        ranks = np.ascontiguousarray(skeletons.ranks, dtype=np.int64)
        self._x = tree.device_points()
        N.call("hks_plan_create", ctypes.byref(self.handle), N.ptr(self._x), tree.n, tree.d, tree.depth,
               skeletons.layout.max_rank, ranks.ctypes.data_as(N._I64P), ctypes.byref(self.kern))
        # dgecon estimates run here, off the factorization's critical path;
        # factor storage they read is marked in use on this stream
        self.cond_stream = N.torch().cuda.Stream(device=N.device(), priority=0)
        N.call("hks_set_cond_stream", self.handle, ctypes.c_void_p(self.cond_stream.cuda_stream))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and N._lib is not None:
            N._lib.hks_plan_destroy(h)
            self.handle = None


class _LazyBlocks(Mapping):
    def __init__(self, keys, fetch):
        self._keys = list(keys)
        self._fetch = fetch
        self._cache = {}

    def __getitem__(self, k):
        if k not in self._keys:
            raise KeyError(k)
        if k not in self._cache:
            self._cache[k] = self._fetch(k)
        return self._cache[k]

    def __iter__(self):
        return iter(self._keys)

    def __len__(self):
        return len(self._keys)


class HierarchicalOperator:
    """tree, skeletons, kernel, leaf_blocks, couplings, n, matvec
    (treecode.py:25-38)."""

    def __init__(self, tree, skeletons, kernel):
        self.tree = tree
        self.skeletons = skeletons
        self.kernel = kernel
        lay = skeletons.layout
        self.layout = lay
        self.plan = Plan(tree, skeletons, kernel)
        self.coup_buf = lay.alloc(N.BUF_COUP)
        N.call("hks_build_operator", self.plan.handle, self.buffers(), N.stream_ptr())
        self.leaf_cache = cache_leaf_blocks(self.plan.handle, tree.n, int(tree._end[-1] - tree._begin[-1])
                                            if tree.depth else tree.n)
        nint = (1 << tree.depth) - 1
        self.leaf_blocks = _LazyBlocks(range(nint, lay.nn), self._leaf_block)
        self.couplings = _LazyBlocks(range(nint), self._coupling)

    @property
    def n(self):
        return self.tree.n

    def matvec(self, w, lam):
        return hmatvec(self, w, lam)

    def buffers(self, extra=None):
        bufs = [None] * N.NBUF
        bufs[N.BUF_INTERP] = self.skeletons.interp_buf
        bufs[N.BUF_SKEL] = self.skeletons.skel_buf
        if hasattr(self, "coup_buf"):
            bufs[N.BUF_COUP] = self.coup_buf
        for k, v in (extra or {}).items():
            bufs[k] = v
        return N.buffers_array(bufs)

    def _leaf_block(self, i):
        m = int(self.tree._end[i] - self.tree._begin[i])
        t = N.torch()
        out = t.empty(m * m, dtype=t.float64, device=N.device())
        N.call("hks_leaf_block", self.plan.handle, i, N.ptr(out), N.stream_ptr())
        return out.view(m, m).t().cpu().numpy().copy()

    def coupling_device(self, i):
        rl, rr = int(self.skeletons.ranks[2 * i + 1]), int(self.skeletons.ranks[2 * i + 2])
        off = int(self.layout.off[N.BUF_COUP, i])
        return self.coup_buf[off: off + rl * rr].view(rr, rl).t()

    def _coupling(self, i):
        return self.coupling_device(i).cpu().numpy().copy()


def cache_leaf_blocks(plan_handle, n, leaf_size):
    """Keep the plan's leaf blocks K_aa on the device (the reference's
    build_operator caches leaf_blocks too, treecode.py:48-51) when they take
    at most 8% of the device's memory -- C2, C3, C5 (1-4.3 GB); not C4
    (34 GB beside its 67 GB factor sets).  HKS_LEAF_CACHE=0/1 forces it.
    Returns whether the blocks are cached."""
    import os
    env = os.environ.get("HKS_LEAF_CACHE")
    t = N.torch()
    if env is not None:
        want = env != "0"
    else:
        want = 8.0 * n * leaf_size <= 0.08 * t.cuda.get_device_properties(N.device()).total_memory
    if want:
        N.call("hks_plan_cache_leaves", plan_handle, N.stream_ptr())
    return want


def build_operator(tree, skeletons, kernel):
    """Evaluate the sibling couplings and build the level program
    (treecode.py:41-62)."""
    return HierarchicalOperator(tree, skeletons, kernel)


def _as_device_cols(v, n, what):
    """1-D / 2-D host or device input -> (k, n) contiguous device tensor
    (column-major n x k) and a flag for returning the caller's kind."""
    t = N.torch()
    if isinstance(v, t.Tensor) and v.is_cuda:
        dev = True
        a = v.to(t.float64)
    else:
        dev = False
        a = np.asarray(v, dtype=np.float64)
    if a.shape[0] != n:
        raise ValueError(f"{what} must have length {n}")
    return N.col_major(a), dev


def hmatvec_device(op, W, lam):
    """(k, n) column-major device block -> (k, n) result (no host traffic)."""
    t = N.torch()
    U = t.empty_like(W)
    N.call("hks_hmatvec", op.plan.handle, op.buffers(), N.ptr(W), N.ptr(U), W.shape[0], float(lam),
           N.stream_ptr())
    return U


def hmatvec(op, w, lam):
    """u = (Ktilde + lam I) w in tree order (treecode.py:92-128); 1-D like the
    reference (a CUDA tensor input stays on the device)."""
    t = N.torch()
    is_dev = isinstance(w, t.Tensor) and w.is_cuda
    shape = tuple(w.shape) if is_dev else np.asarray(w).shape
    if shape != (op.n,):
        raise ValueError(f"weight vector must have length {op.n}")
    W, dev = _as_device_cols(w, op.n, "weight vector")
    U = hmatvec_device(op, W, lam)
    return U[0] if dev else U[0].cpu().numpy()


def upward_pass(op, w):
    """Skeleton weights of every non-root node (treecode.py:65-89)."""
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (op.n,):
        raise ValueError(f"weight vector must have length {op.n}")
    t = N.torch()
    nn = op.layout.nn
    offs = np.zeros(nn, dtype=np.int64)
    lds = np.zeros(nn, dtype=np.int64)
    total = ctypes.c_int64(0)
    N.call("hks_upward_offsets", op.plan.handle, 1, offs.ctypes.data_as(N._I64P), lds.ctypes.data_as(N._I64P),
           ctypes.byref(total))
    out = t.zeros(max(total.value, 1), dtype=t.float64, device=N.device())
    if op.tree.depth > 0:
        W = N.to_device(w)
        N.call("hks_upward", op.plan.handle, op.buffers(), N.ptr(W), 1, N.ptr(out), N.stream_ptr())
    host = out.cpu().numpy()
    res = {}
    for i in range(1, nn):
        r = int(op.skeletons.ranks[i])
        res[i] = host[offs[i]: offs[i] + r].copy()
    return res


def materialize_ktilde(op, lam):
    """Explicit dense Ktilde + lam I, all n columns in one batched matvec
    (diagnostic only, treecode.py:131-144)."""
    n = op.n
    if n > MATERIALIZE_MAX_POINTS:
        raise ValueError(f"materialize_ktilde is limited to n <= {MATERIALIZE_MAX_POINTS}")
    t = N.torch()
    eye = t.eye(n, dtype=t.float64, device=N.device()).contiguous()
    U = hmatvec_device(op, eye, lam)  # row j of U = column j of Ktilde + lam I
    return U.t().cpu().numpy().copy()
