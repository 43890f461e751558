"""ctypes binding of libhks.so (include/hks.h) and device-memory plumbing.

This module is the only place the package touches the C ABI.  There is no
CPU fallback: importing the package on a machine without the built library
raises, and every compute entry point raises when CUDA is unavailable.
PyTorch is used only as the device allocator and stream provider.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

# HKS_LIB_NAME selects a variant build in _lib/ (A/B experiments); default libhks.so
LIB_PATH = Path(__file__).resolve().parent / "_lib" / os.environ.get("HKS_LIB_NAME", "libhks.so")

HKS_OK = 0
HKS_ERR_INVALID = 1
HKS_ERR_CUDA = 2
HKS_ERR_SINGULAR = 3
HKS_ERR_REDUCED_SINGULAR = 4
HKS_ERR_SKELETON = 5
HKS_ERR_NOT_SUPPORTED = 6

FAMILY_CODE = {"gaussian": 0, "laplace3d": 1, "polynomial": 2}

(BUF_INTERP, BUF_SKEL, BUF_THETA, BUF_LEAF_LU, BUF_LEAF_PIV, BUF_PHI, BUF_Z_LU,
 BUF_Z_PIV, BUF_PUSH, BUF_COUP, BUF_STATS) = range(11)
NBUF = 11
BUF_DTYPE = {BUF_SKEL: np.int64, BUF_LEAF_PIV: np.int32, BUF_Z_PIV: np.int32}


class HksKernel(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("h", ctypes.c_double), ("shift", ctypes.c_double),
                ("regularization", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)
_DP = ctypes.POINTER(ctypes.c_double)
_KP = ctypes.POINTER(HksKernel)
_BUFS = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (restype is int unless noted); mirrors include/hks.h
SIGNATURES = {
    "hks_abi_version": [],
    "hks_layout": [_I64, _I64, _I64, _I64P, _I64P],
    "hks_eval_block": [_P, _I64, _KP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I32, _D, _P],
    "hks_kernel_sum": [_P, _I64, _KP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _D, _D, _P],
    "hks_lu_factor": [_P, _I64, _I64, _P, _I32P, _P],
    "hks_lu_solve": [_P, _P, _I64, _I64, _P, _I64, _I64, _P],
    "hks_interp_decomp": [_P, _I64, _I64, _I64, _D, _I64, _P, _P, _I64P, _P],
    "hks_plan_create": [ctypes.POINTER(_P), _P, _I64, _I64, _I64, _I64, _I64P, _KP],
    "hks_plan_destroy": [_P],
    "hks_build_operator": [_P, _BUFS, _P],
    "hks_leaf_block": [_P, _I64, _P, _P],
    "hks_plan_cache_leaves": [_P, _P],
    "hks_factorize": [_P, _BUFS, _D, _I32, _I64P, _P],
    "hks_factor_stats": [_P, _BUFS, _DP, _I32P, _P],
    "hks_solve": [_P, _BUFS, _P, _P, _I64, _P],
    "hks_hmatvec": [_P, _BUFS, _P, _P, _I64, _D, _P],
    "hks_upward_offsets": [_P, _I64, _I64P, _I64P, _I64P],
    "hks_upward": [_P, _BUFS, _P, _I64, _P, _P],
    "hks_build_tree": [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P],
    "hks_knn": [_P, _I64, _I64, _I64, _P, _P],
    "hks_vdots": [_P, _I64, _I64, _P, _I64, _P, _D, _I32, _P, _P],
    "hks_vaxpys": [_P, _I64, _I64, _P, _D, _P, _I64, _P],
    "hks_profile": [_I32, _DP],
    "hks_factor_level_ms": [_P, _DP],
    "hks_set_cond_stream": [_P, _P],
    "hks_cond_wait": [_P, _P],
    # subtree sharding (include/hks.h, "subtree sharding")
    "hks_layout_ex": [_I64, _I64, _I64, _I32, _I64P, _I64P],
    "hks_plan_create_ex": [ctypes.POINTER(_P), _P, _I64, _I64, _I64, _I64, _I64P, _KP, _I32],
    "hks_solve_part": [_P, _BUFS, _P, _P, _I64, _I32, _P, _P],
    "hks_hmatvec_part": [_P, _BUFS, _P, _P, _I64, _D, _I32, _P, _P],
    "hks_knn_rows": [_P, _I64, _I64, _I64, _I64, _I64, _P, _P],
    "hks_knn_rows_mark_ex": [_P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64P, _P],
    "hks_bitmap_count": [_P, _I64, _I64, _I64P, _P],
    "hks_knn_segments": [_P, _I64, _I64, _I64, _I64P, _I64, _P, _P, _P, _P],
    "hks_knn_merge": [_P, _P, _P, _P, _I64, _I64, _P, _P, _P],
    "hks_cross_sum": [_P, _I64, _P, _I64, _I64, _KP, _P, _P, _I64, _I64, _P, _I64, _D, _P],
    "hks_knn_rows_fill_ex": [_I64, _I64, _I64, _I64, _P, _P, _I64P, _P, _I64P, _P],
}

PLAN_FULL, PLAN_SUBTREE, PLAN_TOP = 0, 1, 2

KIND_NAMES = ("gemm", "copy", "getrf", "getrs", "gecon", "eval", "eval_rm", "ksum", "panel", "swap",
              "trsm_l", "trsm_u", "norm1", "lu_fused", "gather", "getrs_fused")  # plan.h StepKind order (kNumKinds)


def profile(enable):
    """Start (True) / stop (False) per-kind CUDA-event timing of plan steps;
    returns {kind: {launches, ms, flops, bytes}} accumulated so far."""
    out = (ctypes.c_double * (4 * 64))()  # >= 4 * kNumKinds (tests/test_cpu_abi.py checks the names)
    call("hks_profile", int(bool(enable)), out)
    return {k: {"launches": out[4 * i], "ms": out[4 * i + 1], "flops": out[4 * i + 2],
                "bytes": out[4 * i + 3]} for i, k in enumerate(KIND_NAMES)}


def launch_count():
    f = lib().hks_launch_count
    f.restype = ctypes.c_longlong
    f.argtypes = []
    return int(f())


class HksError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


_lib = None


def lib():
    """The loaded libhks.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        L.hks_last_error.restype = ctypes.c_char_p
        L.hks_last_error.argtypes = []
        _lib = L
    return _lib


def fn(name):
    """The typed ctypes function for an hks_* entry point."""
    f = getattr(lib(), name)
    if name not in _configured:
        f.argtypes = SIGNATURES[name]
        f.restype = ctypes.c_int
        _configured.add(name)
    return f


_configured = set()


def last_error():
    return lib().hks_last_error().decode()


def call(name, *args):
    """Call an hks_* entry point; raise HksError on a non-zero status."""
    rc = fn(name)(*args)
    if rc != HKS_OK:
        raise HksError(rc, last_error())
    return rc


# ----------------------------------------------------------------- devices

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1701_02324_b200 needs a CUDA device (B200); there is no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def to_device(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy when already there)."""
    t = torch()
    if isinstance(a, t.Tensor):
        out = a.to(device=device(), dtype=dtype or a.dtype)
        return out.contiguous()
    arr = np.ascontiguousarray(a, dtype=dtype and _np_dtype(dtype))
    if not arr.flags.writeable:  # e.g. tree.perm: torch wants a writable source
        arr = arr.copy()
    return t.from_numpy(arr).to(device())


def _np_dtype(tdtype):
    t = torch()
    return {t.float64: np.float64, t.int64: np.int64, t.int32: np.int32}[tdtype]


def empty(n, dtype):
    t = torch()
    return t.empty(int(n), dtype=dtype, device=device())


def kernel_struct(kern):
    return HksKernel(FAMILY_CODE[kern.family], int(kern.degree), float(kern.h),
                     float(kern.shift), float(kern.regularization))


def buffers_array(bufs):
    """Python list of torch tensors / None -> void*[NBUF] for the ABI."""
    arr = (ctypes.c_void_p * NBUF)()
    for i, t in enumerate(bufs):
        arr[i] = t.data_ptr() if t is not None and t.numel() > 0 else None
    return arr


def col_major(mat):
    """(n, k) host or device matrix -> device tensor laid out column-major
    (returned as a (k, n) contiguous tensor whose rows are the columns)."""
    t = torch()
    if isinstance(mat, t.Tensor):
        m = mat.to(device=device(), dtype=t.float64)
    else:
        m = t.from_numpy(np.ascontiguousarray(mat, dtype=np.float64)).to(device())
    return m.t().contiguous() if m.dim() == 2 else m.reshape(1, -1).contiguous()


class Layout:
    """Flat per-node buffer layout of a complete tree (hks_layout_ex); mode
    PLAN_SUBTREE / PLAN_TOP for the two halves of a sharded tree."""

    def __init__(self, n, depth, max_rank, mode=PLAN_FULL):
        self.n, self.depth, self.max_rank, self.mode = int(n), int(depth), int(max_rank), int(mode)
        self.nn = (1 << (self.depth + 1)) - 1
        sizes = (ctypes.c_int64 * NBUF)()
        offs = np.zeros(NBUF * self.nn, dtype=np.int64)
        call("hks_layout_ex", self.n, self.depth, self.max_rank, self.mode, sizes,
             offs.ctypes.data_as(_I64P))
        self.sizes = np.array(list(sizes), dtype=np.int64)
        self.off = offs.reshape(NBUF, self.nn)

    def alloc(self, buf, min_elems=1):
        t = torch()
        dt = {np.int64: t.int64, np.int32: t.int32}.get(BUF_DTYPE.get(buf), t.float64)
        return t.empty(max(int(self.sizes[buf]), int(min_elems), 1), dtype=dt, device=device())
