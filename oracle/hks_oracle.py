"""CPU oracle for the hierarchical kernel factorize / solve path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_1701_02324_b200/`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and there only as the
checker (or as the timed CPU reference arm), never as the product path.

It is a numpy/scipy restatement of the reference package ``hikersolve``
(``/root/reference/pkg/src/hikersolve``) written from its published algorithm;
every function cites the reference ``file:line`` range it follows.  The
restatement is *pinned*: ``tests/test_oracle_golden.py`` checks it against
golden vectors produced by importing the unmodified reference in the build
container (``tests/golden/make_golden.py``), bit-exactly for tree permutation,
kNN lists and skeleton index sets and to roundoff for the floating-point
arrays.

Differences from the reference that are deliberate:
  * ``gmres`` copies the Arnoldi vector before orthogonalising, so an
    operator that returns its own input does not corrupt ``basis[0]`` (the
    reference's aliasing bug; SPEC.md:462 asks for
    "1 iteration, x = b").
  * no size guards (``knn`` has no 65536 cap) -- the oracle is only ever run
    on bounded samples.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg
from scipy.linalg import lapack

POWER_STEPS = 10          # tree.py:22
REORTH_THRESHOLD = 1e-8   # krylov.py:25


# ----------------------------------------------------------------------------
# kernel blocks  (kernels.py:56-105)
# ----------------------------------------------------------------------------

def kernel_block(family, xt, xs, h=0.5, degree=2, shift=1.0):
    """Dense K(xt, xs); diff-form squared distances so K(x,y) == K(y,x)^T
    bit for bit (kernels.py:56-61), gaussian exp(sq / (-2 h^2)) with a true
    division (kernels.py:93-95), laplace 1/(4 pi r) with r=0 -> 0
    (kernels.py:96-101), polynomial (x.y + c)^p (kernels.py:102-104)."""
    xt = np.atleast_2d(np.asarray(xt, dtype=np.float64))
    xs = np.atleast_2d(np.asarray(xs, dtype=np.float64))
    if family == "polynomial":
        return (xt @ xs.T + shift) ** degree
    out = np.empty((xt.shape[0], xs.shape[0]))
    for lo in range(0, xt.shape[0], 512):
        d = xt[lo:lo + 512, None, :] - xs[None, :, :]
        sq = np.einsum("ijk,ijk->ij", d, d)
        if family == "gaussian":
            out[lo:lo + 512] = np.exp(sq / (-2.0 * h ** 2))
        else:
            with np.errstate(divide="ignore"):
                blk = 1.0 / (4.0 * np.pi * np.sqrt(sq))
            blk[sq == 0.0] = 0.0
            out[lo:lo + 512] = blk
    return out


# ----------------------------------------------------------------------------
# partition tree  (tree.py:70-156)
# ----------------------------------------------------------------------------

class Tree:
    """Complete binary partition in heap order.  Arrays: ``perm`` (tree pos
    -> input index), ``coords`` (tree order), ``begin``/``end`` per node,
    ``split_dir`` / ``split_val`` per internal node."""

    def __init__(self, coords, perm, begin, end, depth, split_dir, split_val,
                 leaf_size):
        self.coords, self.perm = coords, perm
        self.begin, self.end = begin, end
        self.depth, self.leaf_size = depth, leaf_size
        self.split_dir, self.split_val = split_dir, split_val
        self.inv_perm = np.empty_like(perm)
        self.inv_perm[perm] = np.arange(perm.size)

    @property
    def n(self):
        return self.coords.shape[0]

    @property
    def num_nodes(self):
        return (1 << (self.depth + 1)) - 1

    def level_nodes(self, level):
        return range((1 << level) - 1, (1 << (level + 1)) - 1)

    def is_leaf(self, i):
        return i >= (1 << self.depth) - 1

    def level_of(self, i):
        return int(math.floor(math.log2(i + 1)))


def tree_depth(n, leaf_size):
    """Smallest L with ceil(n / 2^L) <= leaf_size (tree.py:100-102)."""
    depth = 0
    while -(n // -(1 << depth)) > leaf_size:
        depth += 1
    return depth


def node_ranges(n, depth):
    """Heap-ordered [begin, end) ranges: left child takes ceil(size/2)
    (tree.py:117, 121)."""
    count = (1 << (depth + 1)) - 1
    begin = np.zeros(count, dtype=np.int64)
    end = np.zeros(count, dtype=np.int64)
    end[0] = n
    for i in range((1 << depth) - 1):
        b, e = begin[i], end[i]
        cut = b + (e - b + 1) // 2
        begin[2 * i + 1], end[2 * i + 1] = b, cut
        begin[2 * i + 2], end[2 * i + 2] = cut, e
    return begin, end


def split_direction(block, rng):
    """Seeded power iteration on the centred second moment (tree.py:70-84)."""
    d = block.shape[1]
    if d == 1:
        return np.ones(1)
    c = block - block.mean(axis=0)
    v = rng.standard_normal(d)
    v = v / np.linalg.norm(v)
    for _ in range(POWER_STEPS):
        w = c.T @ (c @ v)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            break
        v = w / nrm
    return v


def build_tree(coords, leaf_size, seed=0):
    """Recursive median split along the power-iteration direction, stable
    argsort, per-node RNG default_rng([seed, level, begin])
    (tree.py:87-144).  Iterative level sweep instead of recursion; nodes of
    one level touch disjoint ranges so the order is immaterial."""
    if leaf_size < 2:
        raise ValueError("leaf_size must be >= 2")
    x = np.array(coords, dtype=np.float64, copy=True)
    n = x.shape[0]
    depth = tree_depth(n, leaf_size)
    begin, end = node_ranges(n, depth)
    perm = np.arange(n, dtype=np.int64)
    split_dir, split_val = {}, {}
    for level in range(depth):
        for i in range((1 << level) - 1, (1 << (level + 1)) - 1):
            b, e = int(begin[i]), int(end[i])
            blk = x[b:e]
            direc = split_direction(blk, np.random.default_rng([seed, level, b]))
            proj = blk @ direc
            order = np.argsort(proj, kind="stable")
            x[b:e] = blk[order]
            perm[b:e] = perm[b:e][order]
            split_dir[i] = direc
            split_val[i] = float(proj[order[(e - b + 1) // 2 - 1]])
    return Tree(x, perm, begin, end, depth, split_dir, split_val, leaf_size)


def knn(coords, k, chunk=256):
    """Exact k-NN, GEMM-form d^2, self excluded, (d^2, index) order
    (tree.py:163-188)."""
    n = coords.shape[0]
    if not 1 <= k <= n - 1:
        raise ValueError("need 1 <= k <= n - 1")
    sq = np.einsum("ij,ij->i", coords, coords)
    out = np.empty((n, k), dtype=np.int64)
    for lo in range(0, n, chunk):
        hi = min(lo + chunk, n)
        d2 = sq[lo:hi, None] + sq[None, :] - 2.0 * (coords[lo:hi] @ coords.T)
        d2[np.arange(hi - lo), np.arange(lo, hi)] = np.inf
        kth = np.partition(d2, k - 1, axis=1)[:, k - 1]
        for r in range(hi - lo):
            cand = np.flatnonzero(d2[r] <= kth[r])
            cand = cand[np.lexsort((cand, d2[r, cand]))]
            out[lo + r] = cand[:k]
    return out


def knn_rows(coords, k, rows, chunk=256):
    """The lists of knn() for the query rows `rows` only (same formula, same
    (d^2, index) order; tree.py:163-188): full-size spot checks where the
    whole table would take hours of CPU."""
    n = coords.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    sq = np.einsum("ij,ij->i", coords, coords)
    out = np.empty((rows.size, k), dtype=np.int64)
    for lo in range(0, rows.size, chunk):
        q = rows[lo:lo + chunk]
        d2 = sq[q, None] + sq[None, :] - 2.0 * (coords[q] @ coords.T)
        d2[np.arange(q.size), q] = np.inf
        kth = np.partition(d2, k - 1, axis=1)[:, k - 1]
        for r in range(q.size):
            cand = np.flatnonzero(d2[r] <= kth[r])
            cand = cand[np.lexsort((cand, d2[r, cand]))]
            out[lo + r] = cand[:k]
    return out


# ----------------------------------------------------------------------------
# column-pivoted QR and interpolative decomposition  (linalg.py:43-136)
# ----------------------------------------------------------------------------

def qrcp(a, tol, max_rank):
    """Truncated Householder QR with column pivoting, norms recomputed from
    scratch every step, lowest index on ties, relative stop
    pivot <= tol * first pivot (linalg.py:43-104).  Returns
    (pivots, R[:rank], rank)."""
    r = np.array(a, dtype=np.float64, copy=True)
    m, n = r.shape
    piv = np.arange(n)
    if m == 0 or n == 0:
        return piv, np.zeros((0, n)), 0
    kmax = min(m, n, max_rank)
    rank, first = kmax, None
    for k in range(kmax):
        norms = np.sqrt(np.sum(r[k:, k:] ** 2, axis=0))
        j = k + int(np.argmax(norms))
        pn = norms[j - k]
        if first is None:
            first = pn
        if pn <= tol * first:
            rank = k
            break
        if j != k:
            r[:, [k, j]] = r[:, [j, k]]
            piv[[k, j]] = piv[[j, k]]
        x0 = r[k, k]
        alpha = -np.copysign(pn, x0) if x0 != 0 else -pn
        v = r[k:, k].copy()
        v[0] -= alpha
        vn = np.linalg.norm(v)
        if vn > 0:
            v /= vn
            r[k:, k:] -= 2.0 * np.outer(v, v @ r[k:, k:])
        r[k, k] = alpha
        r[k + 1:, k] = 0.0
    return piv, r[:rank].copy(), rank


def interp_decomp(a, tol, max_rank):
    """A ~= A[:, J] P with P[:, J] == I exactly (linalg.py:107-136)."""
    a = np.asarray(a, dtype=np.float64)
    piv, rf, r = qrcp(a, tol, max_rank)
    n = a.shape[1]
    p = np.zeros((r, n))
    if r == 0:
        return piv[:0].copy(), p
    coef = np.empty((r, n))
    coef[:, :r] = np.eye(r)
    if n > r:
        coef[:, r:] = scipy.linalg.solve_triangular(rf[:, :r], rf[:, r:])
    p[:, piv] = coef
    return piv[:r].copy(), p


# ----------------------------------------------------------------------------
# dense LU  (linalg.py:151-179)
# ----------------------------------------------------------------------------

class SingularMatrix(np.linalg.LinAlgError):
    pass


def lu(a):
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] == 0:
        return np.zeros((0, 0)), np.zeros(0, dtype=np.int32)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", scipy.linalg.LinAlgWarning)
        f, p = scipy.linalg.lu_factor(a)
    z = np.flatnonzero(np.abs(np.diag(f)) == 0.0)
    if z.size:
        raise SingularMatrix(f"singular matrix: zero pivot at elimination step {int(z[0])}")
    return f, p


def lu_solve(fac, b):
    if fac[0].shape[0] == 0:
        return np.array(b, dtype=np.float64, copy=True)
    return scipy.linalg.lu_solve(fac, b)


# ----------------------------------------------------------------------------
# row sampling and skeletonization  (skeleton.py:84-182)
# ----------------------------------------------------------------------------

def sample_rows(n, begin, end, node, ell, mode, seed, knn_lists=None):
    """skeleton.py:84-122: exact = whole complement; uniform = ell draws
    without replacement shifted past the node; knn_augmented = unique
    neighbours outside the node, all of them if >= ell, else topped up with
    uniform draws from the rest of the complement."""
    size = end - begin
    comp = n - size
    if comp == 0:
        raise ValueError("node covers the whole point set; no rows to sample")
    if mode == "exact":
        return np.concatenate([np.arange(begin), np.arange(end, n)])
    ell = min(ell, comp)
    rng = np.random.default_rng([int(seed), 3, int(node)])
    if mode == "uniform":
        draw = rng.choice(comp, size=ell, replace=False)
        draw[draw >= begin] += size
        return np.sort(draw)
    nb = np.unique(knn_lists[begin:end].ravel())
    base = nb[(nb < begin) | (nb >= end)]
    if base.size >= ell:
        return base
    rest = np.setdiff1d(np.concatenate([np.arange(begin), np.arange(end, n)]),
                        base, assume_unique=True)
    extra = rng.choice(rest.size, size=ell - base.size, replace=False)
    return np.sort(np.concatenate([base, rest[extra]]))


def build_skeletons(tree, kern, tau, max_rank, samples=256, mode="uniform",
                    seed=0, knn_lists=None, threads=1):
    """Bottom-up nested skeletons; leaf candidates = own points, internal =
    q_left ++ q_right (skeleton.py:125-182).  Returns
    {node: (indices, interp)} plus {node: rows} for diagnostics."""
    skel, rows_of = {}, {}
    x = tree.coords

    def one(i):
        b, e = int(tree.begin[i]), int(tree.end[i])
        rows = sample_rows(tree.n, b, e, i, samples, mode, seed, knn_lists)
        if tree.is_leaf(i):
            cands = np.arange(b, e)
        else:
            cands = np.concatenate([skel[2 * i + 1][0], skel[2 * i + 2][0]])
        blk = kernel_block(kern["family"], x[rows], x[cands], **_kp(kern))
        cols, p = interp_decomp(blk, tau, max_rank)
        return i, cands[cols], p, rows

    for level in range(tree.depth, 0, -1):
        work = list(tree.level_nodes(level))
        if threads > 1:
            with ThreadPoolExecutor(threads) as pool:
                res = list(pool.map(one, work))
        else:
            res = [one(i) for i in work]
        for i, idx, p, rows in res:
            skel[i] = (idx, p)
            rows_of[i] = rows
    return skel, rows_of


def _kp(kern):
    return {k: kern[k] for k in ("h", "degree", "shift") if k in kern}


# ----------------------------------------------------------------------------
# compressed operator and matvec  (treecode.py:41-128)
# ----------------------------------------------------------------------------

def build_operator(tree, skel, kern):
    x = tree.coords
    leaf, coup = {}, {}
    for i in range(tree.num_nodes):
        if tree.is_leaf(i):
            b, e = tree.begin[i], tree.end[i]
            leaf[i] = kernel_block(kern["family"], x[b:e], x[b:e], **_kp(kern))
        else:
            coup[i] = kernel_block(kern["family"], x[skel[2 * i + 1][0]],
                                   x[skel[2 * i + 2][0]], **_kp(kern))
    return leaf, coup


def upward(tree, skel, w):
    """treecode.py:65-89."""
    wt = {}
    for level in range(tree.depth, 0, -1):
        for i in tree.level_nodes(level):
            p = skel[i][1]
            if tree.is_leaf(i):
                wt[i] = p @ w[tree.begin[i]:tree.end[i]]
            else:
                wt[i] = p @ np.concatenate([wt[2 * i + 1], wt[2 * i + 2]])
    return wt


def matvec(tree, skel, leaf, coup, w, lam):
    """(Ktilde + lam I) w in tree order (treecode.py:92-128)."""
    w = np.asarray(w, dtype=np.float64)
    u = np.empty(tree.n)
    for i in tree.level_nodes(tree.depth):
        b, e = tree.begin[i], tree.end[i]
        u[b:e] = leaf[i] @ w[b:e] + lam * w[b:e]
    if tree.depth == 0:
        return u
    wt = upward(tree, skel, w)
    acc = {}
    for level in range(tree.depth):
        for i in tree.level_nodes(level):
            c = coup[i]
            tl = c @ wt[2 * i + 2]
            tr = c.T @ wt[2 * i + 1]
            if i in acc:
                push = skel[i][1].T @ acc[i]
                tl = tl + push[:tl.shape[0]]
                tr = tr + push[tl.shape[0]:]
            acc[2 * i + 1], acc[2 * i + 2] = tl, tr
    for i in tree.level_nodes(tree.depth):
        a = acc.get(i)
        if a is not None and a.size:
            u[tree.begin[i]:tree.end[i]] += skel[i][1].T @ a
    return u


# ----------------------------------------------------------------------------
# recursive SMW factorization and solve  (solver.py:86-270)
# ----------------------------------------------------------------------------

class ReducedSingular(RuntimeError):
    pass


def _couple(c, v):
    """B v for B = [[0, C], [C^T, 0]] (solver.py:86-89)."""
    rl = c.shape[0]
    return np.concatenate([c @ v[rl:], c.T @ v[:rl]], axis=0)


def factor_z(z, node, level):
    """LU of Z + 1-norm condition number from LAPACK dgecon
    (solver.py:92-108)."""
    if z.shape[0] == 0:
        return lu(z), 1.0
    anorm = np.linalg.norm(z, 1)
    try:
        f = lu(z)
    except SingularMatrix as exc:
        small = float(np.min(np.abs(np.diag(z)))) if z.size else 0.0
        raise ReducedSingular(
            f"reduced system singular at node {node} (level {level});"
            f" smallest pivot 0 (smallest |Z| diagonal {small:.3e});"
            " increase lambda or tighten tau") from exc
    rc, info = lapack.dgecon(f[0], anorm)
    return f, (float(1.0 / rc) if info == 0 and rc > 0 else np.inf)


def factorize(tree, skel, leaf, coup, lam, threads=1):
    """Bottom-up: leaves LU(K+lam I), phi = A^-1 P^T, theta = P phi;
    internal Z = I + [[0, th_l C], [th_r C^T, 0]], folded = B Z^-1 thhat,
    theta = P (thhat - thhat folded) P^T, push = P^T - folded P^T
    (solver.py:111-186)."""
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    fac = {}

    def do_leaf(i):
        a = leaf[i] + lam * np.eye(leaf[i].shape[0])
        f = lu(a)
        if i == 0:
            return {"lu": f}
        p = skel[i][1]
        phi = lu_solve(f, p.T)
        return {"lu": f, "phi": phi, "theta": p @ phi}

    def do_internal(i):
        tl, tr = fac[2 * i + 1]["theta"], fac[2 * i + 2]["theta"]
        rl, rr = tl.shape[0], tr.shape[0]
        c = coup[i]
        z = np.eye(rl + rr)
        z[:rl, rl:] += tl @ c
        z[rl:, :rl] += tr @ c.T
        zf, cond = factor_z(z, i, tree.level_of(i))
        if i == 0:
            return {"z_lu": zf, "z_cond": cond}
        th = np.zeros((rl + rr, rl + rr))
        th[:rl, :rl] = tl
        th[rl:, rl:] = tr
        p = skel[i][1]
        folded = _couple(c, lu_solve(zf, th))
        return {"z_lu": zf, "z_cond": cond,
                "theta": p @ (th - th @ folded) @ p.T,
                "push": p.T - folded @ p.T}

    for level in range(tree.depth, -1, -1):
        work = list(tree.level_nodes(level))
        fn = do_leaf if level == tree.depth else do_internal
        if threads > 1 and len(work) > 1:
            with ThreadPoolExecutor(threads) as pool:
                res = list(pool.map(fn, work))
        else:
            res = [fn(i) for i in work]
        fac.update(zip(work, res))
    return fac


def solve(tree, skel, coup, fac, b):
    """Upward leaf solves + psi projections, reduced solves g = B Z^-1 psi;
    downward child pushes; tree order in and out (solver.py:189-259)."""
    b = np.asarray(b, dtype=np.float64)
    y, psi, g = {}, {}, {}
    for level in range(tree.depth, -1, -1):
        for i in tree.level_nodes(level):
            f = fac[i]
            if tree.is_leaf(i):
                bl = b[tree.begin[i]:tree.end[i]]
                y[i] = lu_solve(f["lu"], bl)
                if i > 0:
                    psi[i] = f["phi"].T @ bl
            else:
                ph = np.concatenate([psi[2 * i + 1], psi[2 * i + 2]])
                g[i] = _couple(coup[i], lu_solve(f["z_lu"], ph))
                if i > 0:
                    rl = psi[2 * i + 1].shape[0]
                    thg = np.concatenate([fac[2 * i + 1]["theta"] @ g[i][:rl],
                                          fac[2 * i + 2]["theta"] @ g[i][rl:]])
                    psi[i] = skel[i][1] @ (ph - thg)
    x = np.empty(tree.n)
    corr = {}
    for level in range(tree.depth + 1):
        for i in tree.level_nodes(level):
            c = corr.get(i)
            if tree.is_leaf(i):
                xl = y[i]
                if c is not None and c.size:
                    xl = xl - fac[i]["phi"] @ c
                x[tree.begin[i]:tree.end[i]] = xl
            else:
                t = g[i]
                if c is not None and c.size:
                    t = t + fac[i]["push"] @ c
                rl = psi[2 * i + 1].shape[0]
                corr[2 * i + 1], corr[2 * i + 2] = t[:rl], t[rl:]
    return x


# ----------------------------------------------------------------------------
# GMRES  (krylov.py:40-188)
# ----------------------------------------------------------------------------

def gmres(apply_a, apply_minv, b, tol=1e-8, max_iter=500, restart=50):
    """Right-preconditioned restarted GMRES, MGS + one conditional
    reorthogonalisation, Givens rotations, true residual recomputed at every
    cycle end (krylov.py:40-143).  Returns (x, report dict)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    rep = {"iterations": 0, "restarts": 0, "residuals": [], "converged": False}
    bn = np.linalg.norm(b)
    if bn == 0.0:
        rep["converged"] = True
        rep["final_residual"] = 0.0
        return np.zeros(n), rep
    x = np.zeros(n)
    while rep["iterations"] < max_iter:
        r = b - apply_a(x)
        rn = np.linalg.norm(r)
        if rn / bn <= tol:
            rep["converged"] = True
            break
        steps = min(restart, max_iter - rep["iterations"])
        V = np.empty((steps + 1, n))
        V[0] = r / rn
        H = np.zeros((steps + 1, steps))
        cs, sn = np.empty(steps), np.empty(steps)
        g = np.zeros(steps + 1)
        g[0] = rn
        k, brk = 0, False
        while k < steps:
            w = np.array(apply_a(apply_minv(V[k])), dtype=np.float64, copy=True)
            win = np.linalg.norm(w)
            for i in range(k + 1):
                H[i, k] = V[i] @ w
                w -= H[i, k] * V[i]
            ov = V[:k + 1] @ w
            if win > 0 and np.max(np.abs(ov)) > REORTH_THRESHOLD * win:
                H[:k + 1, k] += ov
                w -= ov @ V[:k + 1]
            sub = np.linalg.norm(w)
            H[k + 1, k] = sub
            for i in range(k):
                a0, a1 = H[i, k], H[i + 1, k]
                H[i, k] = cs[i] * a0 + sn[i] * a1
                H[i + 1, k] = -sn[i] * a0 + cs[i] * a1
            den = np.hypot(H[k, k], sub)
            cs[k], sn[k] = (1.0, 0.0) if den == 0.0 else (H[k, k] / den, sub / den)
            H[k, k], H[k + 1, k] = den, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            est = abs(g[k + 1]) / bn
            rep["residuals"].append(est)
            rep["iterations"] += 1
            brk = sub == 0.0
            if not brk:
                V[k + 1] = w / sub
            k += 1
            if brk or est <= tol:
                break
        if k > 0:
            yv = scipy.linalg.solve_triangular(H[:k, :k], g[:k])
            x = x + apply_minv(yv @ V[:k])
            tr = np.linalg.norm(b - apply_a(x)) / bn
            rep["residuals"][-1] = tr
            if tr <= tol:
                rep["converged"] = True
                break
        if brk and not rep["converged"]:
            break
        if rep["iterations"] >= max_iter:
            break
        rep["restarts"] += 1
    rep["final_residual"] = float(np.linalg.norm(b - apply_a(x)) / bn)
    return x, rep


# ----------------------------------------------------------------------------
# convenience: the whole pipeline on one instance
# ----------------------------------------------------------------------------

def pipeline(coords, kern, leaf_size, tau, max_rank, samples, mode, seed,
             kappa=None, threads=1):
    """build_tree -> [knn] -> build_skeletons -> build_operator, mirroring
    cli.py:188-212.  Returns a dict of every intermediate."""
    tree = build_tree(coords, leaf_size, seed)
    nl = knn(tree.coords, kappa) if mode == "knn_augmented" else None
    skel, rows = build_skeletons(tree, kern, tau, max_rank, samples, mode,
                                 seed, nl, threads)
    leaf, coup = build_operator(tree, skel, kern)
    return {"tree": tree, "knn": nl, "skel": skel, "rows": rows,
            "leaf": leaf, "coup": coup}
