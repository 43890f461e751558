"""Restarted, right-preconditioned GMRES with device-resident vectors
(krylov.py of the reference).

The Krylov basis, the Arnoldi products and the residual updates live on the
GPU; the modified Gram-Schmidt dots / updates are libhks vector kernels
(csrc/vec.cu) and the (restart+1) x restart Hessenberg least-squares problem
with its Givens rotations is host scalar work, as in krylov.py:40-143.
``hybrid_solve`` wires hmatvec (compressed) or a dense kernel matrix
(dense_oracle, n <= 4096) as A and the factorization's solve as M^-1
(krylov.py:155-188).

Deliberate difference: the Arnoldi vector is a fresh buffer, so an
operator returning its input cannot alias basis[0] (the reference's
in-place ``w -= ...`` bug).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from . import _native as N
from . import treecode

_REORTH_THRESHOLD = 1e-8
OPERATOR_MODES = ("compressed", "dense_oracle")
_VG = 296


@dataclass
class KrylovReport:
    iterations: int = 0
    restarts: int = 0
    residuals: list = field(default_factory=list)
    converged: bool = False
    wall_time: float = 0.0
    final_residual: float = 0.0


class _Vec:
    """Device BLAS-1 helpers over libhks.  With a ShardComm of several ranks
    the vectors are the ranks' row blocks and every inner product is summed
    over the ranks (one all-reduce of m doubles per call)."""

    def __init__(self, n, cap, comm=None):
        t = N.torch()
        self.n = n
        self.comm = comm if comm is not None and comm.world > 1 else None
        self.part = t.empty(max(cap, 1) * _VG, dtype=t.float64, device=N.device())
        self.scal = t.empty(max(cap, 1), dtype=t.float64, device=N.device())

    def dots(self, V, m, w, out=None, scale=1.0, accumulate=False):
        out = self.scal if out is None else out
        if accumulate and self.comm is not None:
            raise ValueError("accumulating dots are not supported over several ranks")
        N.call("hks_vdots", N.ptr(V), V.stride(0), m, N.ptr(w), self.n, N.ptr(out), float(scale),
               int(accumulate), N.ptr(self.part), N.stream_ptr())
        if self.comm is not None:
            self.comm.all_reduce_sum_(out[:m])
        return out

    def norm(self, w):
        d = self.dots(w.view(1, -1), 1, w)
        return float(np.sqrt(d[:1].item()))

    def axpys(self, V, m, coef, scale, y):
        N.call("hks_vaxpys", N.ptr(V), V.stride(0), m, N.ptr(coef), float(scale), N.ptr(y), self.n,
               N.stream_ptr())


def _device_op(fn, n, host_callable, check):
    t = N.torch()

    def apply(v):
        arg = v.cpu().numpy() if host_callable else v
        out = fn(arg)
        if isinstance(out, t.Tensor):
            o = out.to(device=N.device(), dtype=t.float64)
            shape = tuple(o.shape)
        else:
            arr = np.asarray(out, dtype=np.float64)
            shape = arr.shape
            o = None if check and shape != (n,) else N.to_device(arr)
        if check and shape != (n,):
            raise ValueError(f"operator returned shape {shape}, expected ({n},)")
        return o.reshape(-1).contiguous()

    return apply


def gmres(apply_a, apply_minv, b, tol=1e-8, max_iter=500, restart=50, comm=None):
    """Solve A x = b with right-preconditioned restarted GMRES; x = M^-1 y
    (krylov.py:40-143).  b may be a numpy array (callables then receive and
    return numpy) or a CUDA tensor (callables see CUDA tensors).  comm (a
    sharded.ShardComm): b, x and the callables' vectors are this rank's
    rows of distributed vectors; inner products are all-reduced, so every
    rank takes the same Givens / restart / convergence decisions."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    if restart < 1:
        raise ValueError("restart must be >= 1")
    t = N.torch()
    host = not (isinstance(b, t.Tensor) and b.is_cuda)
    bd = (N.to_device(np.asarray(b, dtype=np.float64)) if host else b.to(t.float64)).reshape(-1).contiguous()
    n = bd.shape[0]
    A = _device_op(apply_a, n, host, True)
    M = _device_op(apply_minv, n, host, False)
    t0 = time.perf_counter()
    rep = KrylovReport()
    vec = _Vec(n, restart + 2, comm)
    bnorm = vec.norm(bd)
    out_of = (lambda x: x.cpu().numpy()) if host else (lambda x: x)
    if bnorm == 0.0:
        rep.converged = True
        rep.wall_time = time.perf_counter() - t0
        return out_of(t.zeros(n, dtype=t.float64, device=bd.device)), rep

    x = t.zeros(n, dtype=t.float64, device=bd.device)
    while rep.iterations < max_iter:
        r = bd - A(x)
        rnorm = vec.norm(r)
        if rnorm / bnorm <= tol:
            rep.converged = True
            break
        steps = min(restart, max_iter - rep.iterations)
        V = t.empty((steps + 1, n), dtype=t.float64, device=bd.device)
        V[0] = r / rnorm
        H = np.zeros((steps + 1, steps))
        cs, sn = np.empty(steps), np.empty(steps)
        g = np.zeros(steps + 1)
        g[0] = rnorm
        hcol = t.zeros(steps + 1, dtype=t.float64, device=bd.device)
        k, breakdown = 0, False
        while k < steps:
            w = A(M(V[k])).clone()  # fresh buffer: no aliasing of the basis
            win = vec.norm(w)
            hcol.zero_()
            for i in range(k + 1):  # modified Gram-Schmidt (krylov.py:84-86)
                vec.dots(V[i:i + 1], 1, w, out=hcol[i:i + 1])
                vec.axpys(V[i:i + 1], 1, hcol[i:i + 1], -1.0, w)
            ov = vec.dots(V, k + 1, w, out=t.empty(k + 1, dtype=t.float64, device=bd.device))
            ovh = ov.cpu().numpy()
            H[: k + 1, k] = hcol[: k + 1].cpu().numpy()
            if win > 0 and np.max(np.abs(ovh)) > _REORTH_THRESHOLD * win:  # krylov.py:89-92
                H[: k + 1, k] += ovh
                vec.axpys(V, k + 1, ov, -1.0, w)
            sub = vec.norm(w)
            H[k + 1, k] = sub
            for i in range(k):  # accumulated Givens rotations (krylov.py:98-101)
                hi, hj = H[i, k], H[i + 1, k]
                H[i, k] = cs[i] * hi + sn[i] * hj
                H[i + 1, k] = -sn[i] * hi + cs[i] * hj
            den = np.hypot(H[k, k], sub)
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = H[k, k] / den, sub / den
            H[k, k], H[k + 1, k] = den, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            est = abs(g[k + 1]) / bnorm
            rep.residuals.append(est)
            rep.iterations += 1
            breakdown = sub == 0.0
            if not breakdown:
                V[k + 1] = w / sub
            k += 1
            if breakdown or est <= tol:
                break
        if k > 0:
            y = scipy.linalg.solve_triangular(H[:k, :k], g[:k])  # k <= restart scalars
            yd = N.to_device(y)
            upd = t.zeros(n, dtype=t.float64, device=bd.device)
            vec.axpys(V, k, yd, 1.0, upd)
            x = x + M(upd)
            true_rel = vec.norm(bd - A(x)) / bnorm
            rep.residuals[-1] = true_rel
            if true_rel <= tol:
                rep.converged = True
                break
        if breakdown and not rep.converged:
            break
        if rep.iterations >= max_iter:
            break
        rep.restarts += 1
    rep.final_residual = vec.norm(bd - A(x)) / bnorm
    rep.wall_time = time.perf_counter() - t0
    return out_of(x), rep


def hybrid_solve(op, f, b, tol=1e-8, max_iter=500, restart=50, operator_mode="compressed"):
    """GMRES on the kernel system preconditioned by the factorization, all
    vectors in tree order (krylov.py:155-188)."""
    if operator_mode not in OPERATOR_MODES:
        raise ValueError(f"unknown operator mode {operator_mode!r}")
    lam = f.lam
    op_lam = op.kernel.regularization
    if op_lam != lam:
        raise ValueError(f"factorization lambda {lam} does not match operator lambda {op_lam}")
    t = N.torch()
    from .solver import solve_device
    if operator_mode == "compressed":
        def apply_a(v):
            return treecode.hmatvec_device(op, v.reshape(1, -1), lam)[0]
    else:
        n = op.n
        if n > treecode.MATERIALIZE_MAX_POINTS:
            raise ValueError(f"dense_oracle mode is limited to n <= {treecode.MATERIALIZE_MAX_POINTS}")
        x = op.tree.device_points()
        kern = N.kernel_struct(op.kernel)

        def apply_a(v):
            # true dense (K + lam I) v by fused kernel summation (K never stored)
            v = v.reshape(-1).contiguous()
            out = t.empty_like(v)
            N.call("hks_kernel_sum", N.ptr(x), x.shape[1], kern, None, 0, n, None, 0, n, N.ptr(v), n, 1,
                   N.ptr(out), n, 0.0, float(lam), N.stream_ptr())
            return out

    def apply_minv(v):
        return solve_device(f, v.reshape(1, -1).contiguous())[0]

    host = not (isinstance(b, t.Tensor) and b.is_cuda)
    bd = N.to_device(np.asarray(b, dtype=np.float64)) if host else b
    x, rep = gmres(apply_a, apply_minv, bd, tol=tol, max_iter=max_iter, restart=restart)
    return (x.cpu().numpy() if host else x), rep


def hybrid_solve_sharded(op, f, b, tol=1e-8, max_iter=500, restart=50):
    """hybrid_solve (krylov.py:155-188) on a subtree-sharded operator
    (sharded.py): b is this rank's rows (tree order, device or host), A the
    sharded hmatvec, M^-1 the sharded solve, inner products all-reduced over
    the ranks.  Returns this rank's rows of x and the (rank-identical)
    report."""
    from . import sharded as S
    lam = f.lam
    if op.kernel.regularization != lam:
        raise ValueError(f"factorization lambda {lam} does not match operator lambda {op.kernel.regularization}")
    t = N.torch()
    if (tuple(b.shape) if isinstance(b, t.Tensor) else np.shape(b)) != (op.spec.size,):
        raise ValueError(f"right-hand side must have this shard's {op.spec.size} rows")
    host = not (isinstance(b, t.Tensor) and b.is_cuda)
    bd = N.to_device(np.asarray(b, dtype=np.float64)) if host else b

    def apply_a(v):
        return S.hmatvec_sharded(op, v.reshape(1, -1), lam)[0]

    def apply_minv(v):
        return S.solve_sharded(f, v.reshape(1, -1))[0]

    x, rep = gmres(apply_a, apply_minv, bd, tol=tol, max_iter=max_iter, restart=restart, comm=op.comm)
    return (x.cpu().numpy() if host else x), rep


def gmres_multi(apply_a, apply_minv, B, tol=1e-8, max_iter=500, restart=50):
    """k independent restarted GMRES solves (krylov.py:40-143, one per
    column of the (k, n) device block B) run in lockstep, so every operator
    application is ONE batched call over the columns still iterating:
    apply_a / apply_minv map an (m, n) block to an (m, n) block.  Each
    column's recurrence, stopping tests and reports are its own; the
    batched hmatvec / solve give every column the bits a single-column call
    gives it (ksum and the DMMA products are column-independent), so each
    column equals gmres() on that column alone.  Returns (X, [reports])."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    if restart < 1:
        raise ValueError("restart must be >= 1")
    t = N.torch()
    B = B.to(t.float64).contiguous()
    k, n = B.shape
    vec = _Vec(n, restart + 2)
    t0 = time.perf_counter()
    reps = [KrylovReport() for _ in range(k)]
    X = t.zeros((k, n), dtype=t.float64, device=B.device)
    bnorm = [vec.norm(B[c]) for c in range(k)]
    live = []
    for c in range(k):
        if bnorm[c] == 0.0:
            reps[c].converged = True
        else:
            live.append(c)

    def A(cols, V):
        return apply_a(V.contiguous()) if cols else V

    def M(cols, V):
        return apply_minv(V.contiguous()) if cols else V

    stop = set()  # columns done (converged, broken down or out of iterations)
    while True:
        cols = [c for c in live if c not in stop and reps[c].iterations < max_iter]
        for c in live:
            if c not in cols:
                stop.add(c)
        if not cols:
            break
        R = B[cols] - A(cols, X[cols])
        st = {}
        for a, c in enumerate(cols):
            rnorm = vec.norm(R[a])
            if rnorm / bnorm[c] <= tol:
                reps[c].converged = True
                stop.add(c)
                continue
            steps = min(restart, max_iter - reps[c].iterations)
            V = t.empty((steps + 1, n), dtype=t.float64, device=B.device)
            V[0] = R[a] / rnorm
            g = np.zeros(steps + 1)
            g[0] = rnorm
            st[c] = dict(V=V, H=np.zeros((steps + 1, steps)), cs=np.empty(steps), sn=np.empty(steps), g=g,
                         steps=steps, k=0, breakdown=False, done=False,
                         hcol=t.zeros(steps + 1, dtype=t.float64, device=B.device))
        while True:  # the Arnoldi steps of this cycle, batched over the columns still in it
            act = [c for c in st if not st[c]["done"]]
            if not act:
                break
            Vk = t.stack([st[c]["V"][st[c]["k"]] for c in act])
            W = A(act, M(act, Vk)).clone()  # fresh buffer: no aliasing of the bases
            for a, c in enumerate(act):
                s = st[c]
                kk, V, H, hcol, w = s["k"], s["V"], s["H"], s["hcol"], W[a]
                win = vec.norm(w)
                hcol.zero_()
                for i in range(kk + 1):  # modified Gram-Schmidt (krylov.py:84-86)
                    vec.dots(V[i:i + 1], 1, w, out=hcol[i:i + 1])
                    vec.axpys(V[i:i + 1], 1, hcol[i:i + 1], -1.0, w)
                ov = vec.dots(V, kk + 1, w, out=t.empty(kk + 1, dtype=t.float64, device=B.device))
                ovh = ov.cpu().numpy()
                H[: kk + 1, kk] = hcol[: kk + 1].cpu().numpy()
                if win > 0 and np.max(np.abs(ovh)) > _REORTH_THRESHOLD * win:  # krylov.py:89-92
                    H[: kk + 1, kk] += ovh
                    vec.axpys(V, kk + 1, ov, -1.0, w)
                sub = vec.norm(w)
                H[kk + 1, kk] = sub
                cs, sn, g = s["cs"], s["sn"], s["g"]
                for i in range(kk):  # accumulated Givens rotations (krylov.py:98-101)
                    hi, hj = H[i, kk], H[i + 1, kk]
                    H[i, kk] = cs[i] * hi + sn[i] * hj
                    H[i + 1, kk] = -sn[i] * hi + cs[i] * hj
                den = np.hypot(H[kk, kk], sub)
                if den == 0.0:
                    cs[kk], sn[kk] = 1.0, 0.0
                else:
                    cs[kk], sn[kk] = H[kk, kk] / den, sub / den
                H[kk, kk], H[kk + 1, kk] = den, 0.0
                g[kk + 1] = -sn[kk] * g[kk]
                g[kk] = cs[kk] * g[kk]
                est = abs(g[kk + 1]) / bnorm[c]
                reps[c].residuals.append(est)
                reps[c].iterations += 1
                s["breakdown"] = sub == 0.0
                if not s["breakdown"]:
                    V[kk + 1] = w / sub
                s["k"] = kk + 1
                if s["breakdown"] or est <= tol or s["k"] >= s["steps"]:
                    s["done"] = True
        upd_cols = [c for c in st if st[c]["k"] > 0]
        if upd_cols:
            U = t.zeros((len(upd_cols), n), dtype=t.float64, device=B.device)
            for a, c in enumerate(upd_cols):
                s = st[c]
                y = scipy.linalg.solve_triangular(s["H"][: s["k"], : s["k"]], s["g"][: s["k"]])
                vec.axpys(s["V"], s["k"], N.to_device(y), 1.0, U[a])
            X[upd_cols] = X[upd_cols] + M(upd_cols, U)
            Rt = B[upd_cols] - A(upd_cols, X[upd_cols])
            for a, c in enumerate(upd_cols):
                true_rel = vec.norm(Rt[a]) / bnorm[c]
                reps[c].residuals[-1] = true_rel
                if true_rel <= tol:
                    reps[c].converged = True
                    stop.add(c)
                elif st[c]["breakdown"]:
                    stop.add(c)
        for c in st:
            if c not in stop and reps[c].iterations < max_iter:
                reps[c].restarts += 1
    if live:
        Rf = B[live] - A(live, X[live])
        for a, c in enumerate(live):
            reps[c].final_residual = vec.norm(Rf[a]) / bnorm[c]
    wall = time.perf_counter() - t0
    for r in reps:
        r.wall_time = wall
    return X, reps


def hybrid_solve_multi(op, f, B, tol=1e-8, max_iter=500, restart=50):
    """hybrid_solve (krylov.py:155-188) for an (n, k) block of right-hand
    sides (tree order, host or device): k GMRES solves in lockstep with
    batched matvecs / preconditioner solves (gmres_multi).  Returns X of the
    same kind and shape and one KrylovReport per column; column j equals
    hybrid_solve(op, f, B[:, j])."""
    lam = f.lam
    if op.kernel.regularization != lam:
        raise ValueError(f"factorization lambda {lam} does not match operator lambda {op.kernel.regularization}")
    t = N.torch()
    from .solver import solve_device
    dev = isinstance(B, t.Tensor) and B.is_cuda
    Bt = (B.to(t.float64) if dev else N.to_device(np.asarray(B, dtype=np.float64)))
    if Bt.dim() != 2 or Bt.shape[0] != op.n:
        raise ValueError(f"expected an ({op.n}, k) right-hand side block")
    X, reps = gmres_multi(lambda V: treecode.hmatvec_device(op, V, lam), lambda V: solve_device(f, V),
                          Bt.t().contiguous(), tol=tol, max_iter=max_iter, restart=restart)
    X = X.t()
    return (X if dev else X.cpu().numpy()), reps
