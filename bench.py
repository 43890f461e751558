#!/usr/bin/env python
"""Benchmark: factorize + k-RHS solve of (lambda I + Ktilde) on the BASELINE
workload (default C3: N=1048576, d=28, m=512, adaptive rank tau=1e-5 capped
at s=256, kappa=32, 16 RHS -- the configuration BASELINE.json quotes across
1/2/4/8 GPUs; ``--config C2`` etc. for the others).

One *step* = ``factorize(op, lam)`` + ``solve_multi(f, B)`` on a resident
operator (tree, kNN, skeletons and couplings are built once, untimed, and
reported under ``setup``).  ``value`` = N / device step time with B resident
in HBM; ``e2e`` = the same step through the public API from a pinned host B
to a host x (H2D + D2H inside the timed region).  ``--impl reference`` times
the CPU oracle (oracle/hks_oracle.py, the reference algorithm restated) on a
bounded sample of the same workload.  See DESIGN.md for the definitions.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hks|reference] [--config C3]

Multi-GPU (torchrun, one rank per GPU): the configuration's N is split
across the ranks by subtree (strong scaling, BASELINE's fixed-N runs);
``--weak`` instead gives every rank the configuration's N.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_DMMA_PEAK_TFLOPS = 37.1  # measured, profiles/fp64_peaks_r01.jsonl (mma.sync m8n8k4 f64)
FP64_DFMA_PEAK_TFLOPS = 34.2  # measured, same file


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["hks", "reference"], default="hks")
    p.add_argument("--config", default="C3")
    p.add_argument("--weak", action="store_true",
                   help="N > 1 GPUs: every rank holds the config's N (default: the config's N split across ranks)")
    p.add_argument("--no-accuracy", action="store_true", help="skip the full-N sampled-row accuracy metrics")
    p.add_argument("--points", type=int, default=None, help="override N per GPU (same generator / kernel / ranks)")
    p.add_argument("--cpu-sample-n", type=int, default=16384)
    p.add_argument("--cpu-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-clocks", action="store_true", help="skip the nvidia-smi clock sampler (diagnostics)")
    p.add_argument("--dump-x", default=None,
                   help="directory: each rank saves its block of the timed solution (tree order) as x_rank<r>.npz")
    p.add_argument("--knn-trees", type=int, default=0,
                   help="setup only: approximate kNN from this many random-projection trees (0 = exact)")
    return p.parse_args()


def max_over_ranks(value, world, device):
    """The slowest rank's value (timings are reported as the max over ranks);
    NCCL on the GPU box, gloo in the CPU tests."""
    if world <= 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], device=device, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU arm

def oracle_arm(w, n_sample, steps, threads):
    """Time the CPU oracle's factorize + k-RHS solve (the reference's
    algorithm, numpy/LAPACK) on a bounded N=n_sample instance of workload w.
    BLAS is pinned to one thread and the per-level node loops use `threads`
    workers, the reference's best configuration."""
    from threadpoolctl import threadpool_limits
    from oracle import hks_oracle as O
    from paper_1701_02324_b200 import workloads as W
    ws = w.scaled(n_sample)
    x = W.points(ws, 0)
    b = W.rhs(ws, 0)
    kern = {"family": "gaussian", "h": w.h}
    with threadpool_limits(limits=1, user_api="blas"):
        t0 = time.perf_counter()
        inst = O.pipeline(x, kern, w.leaf_size, w.tau, w.max_rank, w.samples, "knn_augmented", 0,
                          kappa=w.kappa, threads=threads)
        t_setup = time.perf_counter() - t0
        tree, sk, coup = inst["tree"], inst["skel"], inst["coup"]
        bt = b[tree.perm]
        times, tf, ts = [], [], []
        for _ in range(steps):
            t0 = time.perf_counter()
            fac = O.factorize(tree, sk, inst["leaf"], coup, w.lam, threads=threads)
            t1 = time.perf_counter()
            for j in range(b.shape[1]):  # solve_multi is a column loop (solver.py:262-270)
                O.solve(tree, sk, coup, fac, bt[:, j])
            t2 = time.perf_counter()
            times.append(t2 - t0)
            tf.append(t1 - t0)
            ts.append(t2 - t1)
    t = statistics.median(times)
    return {
        "value": n_sample / t, "t_step": t, "t_factorize": statistics.median(tf),
        "t_solve": statistics.median(ts), "setup_s": t_setup, "cores": threads,
        "sample": (f"{w.name} generator/kernel/ranks at N={n_sample} (depth {tree.depth}), factorize + "
                   f"{b.shape[1]}-RHS solve, {steps} steps, median; setup (tree+kNN+skeletons) untimed"),
    }


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=10.0):
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        self.skip = len(self.lines)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        region = self.lines[getattr(self, "skip", 0):] or self.lines[-1:]  # samples inside the timed region
        for ln in region:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- GPU arm

class SingleRunner:
    """One GPU: the whole workload through the public API (N=1 line, and
    the replicas fallback)."""

    def __init__(self, w, seed, knn_trees=0):
        import torch
        import paper_1701_02324_b200 as hk
        from paper_1701_02324_b200 import _native as N
        from paper_1701_02324_b200 import workloads as W
        self.hk, self.N, self.w = hk, N, w
        x = W.points(w, seed)
        self.b = W.rhs(w, seed)
        kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
        cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples,
                                sample_mode="knn_augmented", seed=seed)
        setup = {}
        ps = hk.PointSet(x)
        _, setup["h2d_points"] = timed(ps.device)
        tree, setup["build_tree"] = timed(lambda: hk.build_tree(ps, w.leaf_size, seed=seed))
        if knn_trees:
            knn, setup["knn"] = timed(lambda: hk.knn_approx(tree.points, w.kappa, trees=knn_trees))
        else:
            knn, setup["knn"] = timed(lambda: hk.knn_bruteforce(tree.points, w.kappa))
        skels, setup["skeletonize"] = timed(lambda: hk.build_skeletons(tree, kern, cfg, knn=knn))
        self.op, setup["assemble"] = timed(lambda: hk.build_operator(tree, skels, kern))
        self.setup = {k: round(v, 4) for k, v in setup.items()}
        print(f"bench: {w.name} N={w.n} setup {self.setup}", file=sys.stderr, flush=True)
        self.tree = tree
        # right-hand sides resident in tree order, column-major (k, n)
        self.B = N.to_device(np.ascontiguousarray(self.b[np.asarray(tree.perm)].T))
        self.n_job = w.n
        self.Bh = torch.from_numpy(np.ascontiguousarray(self.b)).pin_memory()

    def factorize(self):
        return self.hk.factorize(self.op, self.w.lam)

    def solve(self, f):
        from paper_1701_02324_b200.solver import solve_device
        if self.w.method != "hybrid":
            return solve_device(f, self.B)
        # C5: GMRES on the treecode matvec, preconditioned by the factorization,
        # one right-hand side at a time (krylov.py:155-188)
        from paper_1701_02324_b200.krylov import hybrid_solve_multi
        X, reps = hybrid_solve_multi(self.op, f, self.B.t(), tol=self.w.gmres_tol, max_iter=500,
                                     restart=self.w.gmres_restart)  # k GMRES solves, batched operators
        self.krylov = [r.iterations for r in reps]
        return X.t()

    def accuracy(self, f):
        """Sampled-row metrics at full N (metrics.sampled_error_report) for
        the first right-hand side, beside the reference's own values on the
        same generator at N = 16384 / 65536 (tests/golden/ladder_*.npz)."""
        from paper_1701_02324_b200 import metrics as M
        t0 = time.perf_counter()
        rep = M.sampled_error_report(self.op, f, b=self.b[np.asarray(self.tree.perm), 0], rows=256, seed=0)
        rep["seconds"] = round(time.perf_counter() - t0, 3)
        ref = {}
        for n in (16384, 65536):
            g = ROOT / "tests" / "golden" / f"ladder_{self.w.name.lower()}_n{n}.npz"
            if g.exists():
                z = np.load(g)
                ref[str(n)] = {"matvec_relerr_vs_K": float(z["sampled_matvec_relerr"]),
                               "true_residual": float(z["sampled_true_residual"]),
                               "residual_vs_Ktilde": float(z["relres_ktilde"][0])}
        if ref:
            rep["reference_at_reduced_n"] = ref
        return rep

    def relres(self, X):
        import torch
        res = self.hk.treecode.hmatvec_device(self.op, X[:1].contiguous(), self.w.lam)[0] - self.B[0]
        return float(torch.linalg.vector_norm(res) / torch.linalg.vector_norm(self.B[0]))

    def e2e(self):
        """pinned host B (input order) -> host x through the public API.  The
        H2D copy of B runs on a copy stream beside the factorization (it
        does not depend on it); the solve waits for it, and x comes back as
        one D2H copy into pinned memory."""
        import torch
        if self.w.method != "hybrid":
            cs = getattr(self, "_copy_stream", None) or torch.cuda.Stream()
            self._copy_stream = cs
            with torch.cuda.stream(cs):
                Bd = self.Bh.to(self.N.device(), non_blocking=True)
            ev = cs.record_event()
            f = self.hk.factorize(self.op, self.w.lam)
            torch.cuda.current_stream().wait_event(ev)
            Bd.record_stream(torch.cuda.current_stream())
            X = self.hk.solve_multi(f, Bd, in_tree_order=False)
            xh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True)
            xh.copy_(X, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return xh
        # hybrid_solve takes tree-ordered host vectors (krylov.py:155-188)
        f = self.hk.factorize(self.op, self.w.lam)
        perm = np.asarray(self.tree.perm)
        bt = self.b[perm]
        from paper_1701_02324_b200.krylov import hybrid_solve_multi
        xt, _ = hybrid_solve_multi(self.op, f, bt, tol=self.w.gmres_tol, max_iter=500, restart=self.w.gmres_restart)
        x = np.empty_like(self.b)
        x[perm] = xt
        return x

    @property
    def io_bytes(self):
        return int(self.b.nbytes), int(self.b.nbytes)

    def factor_bytes(self):
        from paper_1701_02324_b200.solver import _FACTOR_BUFS
        return 8 * int(sum(self.op.layout.sizes[b] for b in _FACTOR_BUFS))


class ShardedRunner:
    """P = 2^p GPUs: one global seeded instance subtree-sharded over the
    ranks (paper_1701_02324_b200/sharded.py; NCCL only for the shard-root
    exchange).  Strong scaling (default): the instance is the config's N,
    each rank owns N / P points.  Weak (--weak): P x N points, every rank's
    shard the single-GPU workload's N."""

    def __init__(self, w, world, rank, weak=False):
        import torch
        import paper_1701_02324_b200 as hk
        from paper_1701_02324_b200 import _native as N
        from paper_1701_02324_b200 import sharded as S
        from paper_1701_02324_b200 import workloads as W
        self.hk, self.N, self.S, self.w = hk, N, S, w
        wg = w.scaled(w.n * world) if weak else w
        self.weak = weak
        x = W.points(wg, 0)
        b = W.rhs(wg, 0)
        kern = hk.KernelSpec("gaussian", h=w.h, regularization=w.lam)
        cfg = hk.SkeletonConfig(tau=w.tau, max_rank=w.max_rank, samples=w.samples,
                                sample_mode="knn_augmented", seed=0)
        self.comm = S.ShardComm()
        setup = {}
        ps = hk.PointSet(x)
        _, setup["h2d_points"] = timed(ps.device)
        tree, setup["build_tree"] = timed(lambda: hk.build_tree(ps, w.leaf_size, seed=0))
        self.spec = spec = S.ShardSpec(wg.n, tree.depth, world, rank)
        knn, setup["knn"] = timed(lambda: S.knn_shard(tree, w.kappa, spec))
        sk, setup["skeletonize"] = timed(lambda: S.build_skeletons_sharded(tree, kern, cfg, knn, spec, self.comm))
        self.op, setup["assemble"] = timed(lambda: S.build_operator_sharded(tree, sk, kern, self.comm))
        self.setup = {k: round(v, 4) for k, v in setup.items()}
        bl = np.ascontiguousarray(b[np.asarray(tree.perm)][spec.begin: spec.end].T)  # (k, n_shard)
        self.b_local = bl
        self.B = N.to_device(bl)
        self.Bh = torch.from_numpy(bl).pin_memory()
        self.n_job = wg.n

    def factorize(self):
        return self.S.factorize_sharded(self.op, self.w.lam)

    def solve(self, f):
        return self.S.solve_sharded(f, self.B)

    def accuracy(self, f):
        return None  # the sampled-row metrics run on the single-GPU line; relres_vs_ktilde is global here

    def relres(self, X):
        import torch
        U = self.S.hmatvec_sharded(self.op, X[:1].contiguous(), self.w.lam)
        num = torch.stack([torch.sum((U[0] - self.B[0]) ** 2), torch.sum(self.B[0] ** 2)])
        self.comm.all_reduce_sum_(num)
        return float(torch.sqrt(num[0] / num[1]))

    def e2e(self):
        """pinned host block of the shard's right-hand sides -> host x rows
        (the H2D copy beside the factorization, as SingleRunner.e2e)."""
        import torch
        cs = getattr(self, "_copy_stream", None) or torch.cuda.Stream()
        self._copy_stream = cs
        with torch.cuda.stream(cs):
            B = self.Bh.to(self.N.device(), non_blocking=True)
        ev = cs.record_event()
        f = self.S.factorize_sharded(self.op, self.w.lam)
        torch.cuda.current_stream().wait_event(ev)
        B.record_stream(torch.cuda.current_stream())
        X = self.S.solve_sharded(f, B)
        xh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True)
        xh.copy_(X, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return xh

    @property
    def io_bytes(self):
        return int(self.b_local.nbytes), int(self.b_local.nbytes)

    def factor_bytes(self):
        from paper_1701_02324_b200.solver import _FACTOR_BUFS
        sk = self.op.skeletons
        return 8 * int(sum(sk.local_layout.sizes[b] + sk.top_layout.sizes[b] for b in _FACTOR_BUFS))


def timed(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def gpu_arm(args, w, rank, world):
    import torch
    from paper_1701_02324_b200 import _native as N

    dev = torch.device("cuda", torch.cuda.current_device())
    run = ShardedRunner(w, world, rank, weak=args.weak) if world > 1 else SingleRunner(w, 0, args.knn_trees)
    stream = torch.cuda.current_stream()

    def step():
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        f = run.factorize()
        e1.record(stream)
        X = run.solve(f)
        e2.record(stream)
        return f, X, (e0, e1, e2)

    # configs whose factor storage is a large share of HBM (C4: 67 GB) keep
    # one factorization alive at a time; the others keep the previous one
    # alive across the next step, like an application that compares them
    lean = run.factor_bytes() * 4 > 0.8 * torch.cuda.mem_get_info()[0]  # 4 sets: new, previous, 2 pending

    clocks = ClockSampler(torch.cuda.current_device())
    if not args.no_clocks:
        clocks.start()  # NVML start-up (it stalls the context) overlaps the warm-up, not the timed steps
    keep = None
    for _ in range(max(args.warmup, 0)):  # same object lifetimes as the timed loop: the allocator
        keep = None if lean else keep     # holds two factorizations' storage before timing starts
        keep = step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if not args.no_clocks:
        clocks.wait_first()
        keep = None if lean else keep
        keep = step()  # the warm-up's last step right before the region (no idle gap)
        torch.cuda.synchronize()
        clocks.skip = len(clocks.lines)
    # factor storage for the timed loop allocated up front (new, previous,
    # and up to two sets whose dgecon estimates may still be running): no
    # GB-sized cudaMalloc inside a timed factorize
    pools = [p for p in ([getattr(run.op, "_factor_pool", None)] + list(getattr(run.op, "_factor_pools", ())))
             if p is not None]
    for p in pools:
        p.reserve(2 if lean else 4)
    sets_before = sum(p.created for p in pools)
    # host hygiene as in timeit: no cyclic-GC pause (tens of ms with a large
    # heap) lands between the timed launches
    gc.collect()
    gc.disable()
    launches0 = N.launch_count()
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    f = keep[0] if keep else None
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only the timed region
    r0.record(stream)
    evs, host_t = [], []
    for _ in range(args.steps):
        h0 = time.perf_counter()
        if lean:
            keep = f = None
        f, X, ev = step()
        host_t.append((time.perf_counter() - h0) * 1e3)
        evs.append(ev)
    f.join_cond()  # the last step's dgecon estimates (condition stream) finish inside the region
    r1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    gc.enable()
    sets_in_region = sum(p.created for p in pools) - sets_before
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    clk = clocks.stop()
    # per-kernel CUDA-event breakdown: the same steps replayed once more with
    # an event pair around every launch (graphs off while profiling)
    N.profile(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    kinds = N.profile(False)
    region_ms = r0.elapsed_time(r1)
    t_fact = [a.elapsed_time(bq) for a, bq, _ in evs]
    t_solve = [bq.elapsed_time(c) for _, bq, c in evs]
    region_ms = max_over_ranks(region_ms, world, dev)
    fact_ms = max_over_ranks(statistics.mean(t_fact), world, dev)   # slowest rank, like the region
    solve_ms = max_over_ranks(statistics.mean(t_solve), world, dev)
    ms_step = region_ms / args.steps

    # parity spot check of the timed solution: residual against Ktilde
    relres = run.relres(X)
    if args.dump_x:
        begin = run.spec.begin if world > 1 else 0
        np.savez(Path(args.dump_x) / f"x_rank{rank}.npz", x=X.cpu().numpy(), begin=begin, n=run.n_job)
    # full-N accuracy (BASELINE.md 4.2 / oracle.py:68-140 at GPU scale):
    # 256 sampled rows of the exact K + lam I against all N columns
    accuracy = None if args.no_accuracy else run.accuracy(f)

    # e2e through the public API: pinned host B -> host x, H2D + D2H inside
    e2e_ms = []
    gc.collect()
    gc.disable()
    for i in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        run.e2e()
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    gc.enable()
    e2e_step = max_over_ranks(statistics.median(e2e_ms), world, dev)
    w_name = w.name
    setup = run.setup

    # roofline of the dominant kernel kind (algorithmic flops / event time)
    tensor_kinds = {"gemm", "getrf", "getrs", "gecon"}
    fp64_pipe_kinds = {"ksum", "eval", "eval_rm"}  # distance + exp on the FP64 pipe (DFMA peak)
    # dominant kind on the critical path: the dgecon estimates run on the
    # low-priority condition stream, overlapped (their time is in `kernels`)
    dom = max((k for k in kinds if k != "gecon" and kinds[k]["launches"]), key=lambda k: kinds[k]["ms"])
    kd = kinds[dom]
    if dom in tensor_kinds or dom in fp64_pipe_kinds:
        pipe = dom in fp64_pipe_kinds
        peak = FP64_DFMA_PEAK_TFLOPS if pipe else FP64_DMMA_PEAK_TFLOPS
        achieved = kd["flops"] / (kd["ms"] * 1e-3) / 1e12
        roof = {"bound": "fp64 pipe" if pipe else "tensor", "kernel": dom, "achieved": round(achieved, 3),
                "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                "peak_source": ("measured FP64 DFMA peak" if pipe else "measured FP64 DMMA peak") +
                               " (profiles/fp64_peaks_r01.jsonl); MEASURED_PEAKS.json has no FP64 entry"}
    else:
        from_peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = from_peaks.get("hbm_gbs", 6544.7)
        achieved = kd["bytes"] / (kd["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    traffic_file = ROOT / "profiles" / "ncu_traffic_r02.json"
    roof["traffic"] = None
    if traffic_file.exists():
        tr = json.loads(traffic_file.read_text())
        roof["traffic"] = tr.get(dom)  # ncu DRAM bytes per launch of this kind (one bench step)
    roof["algorithmic_bytes_per_launch"] = round(kd["bytes"] / max(kd["launches"], 1))
    roof["launch_share"] = round(kd["ms"] / max(sum(v["ms"] for v in kinds.values()), 1e-9), 4)
    total_flops = sum(v["flops"] for v in kinds.values()) / args.steps
    kernels = {k: {"launches": int(v["launches"]), "ms_per_step": round(v["ms"] / args.steps, 4),
                   "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3) if v["flops"] else None,
                   "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
               for k, v in kinds.items() if v["launches"]}
    n_total = run.n_job
    h2d, d2h = run.io_bytes
    result = {
        "metric": "factorize+solve points/s",
        "value": round(n_total / (ms_step * 1e-3), 1),
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak" if world == 1 or args.weak else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": ("synthetic: seeded BASELINE generator (BASELINE.md 4.4), seed 0" if world == 1 else
                 f"synthetic: one seeded instance of {n_total} points (BASELINE.md 4.4), subtree-sharded "
                 f"over {world} ranks ({n_total // world} points each)"),
        "config": {"workload": w.name, "n": w.n, "d": w.d, "leaf": w.leaf_size, "max_rank": w.max_rank,
                   "tau": w.tau, "kappa": w.kappa, "samples": w.samples, "sample_mode": "knn_augmented",
                   "knn": f"approx ({args.knn_trees} random-projection trees)" if args.knn_trees else "exact",
                   "h": w.h, "lambda": w.lam, "nrhs": w.nrhs,
                   "parallelism": f"subtree-sharded x{world} (NCCL shard-root exchange)" if world > 1 else "single",
                   "n_global": n_total,
                   "l2": "no flush: per-step working set (factor storage) exceeds the 126 MB L2"},
        "factorize_points_per_s": round(n_total / (fact_ms * 1e-3), 1),
        "solve_rhs_per_s": round(w.nrhs / (solve_ms * 1e-3), 1),
        "factorize_ms": round(fact_ms, 4),
        "step_ms_each": [round(a + b2, 3) for a, b2 in zip(t_fact, t_solve)],
        "host_ms_each": [round(v, 3) for v in host_t],
        "factorize_ms_each": [round(v, 3) for v in t_fact],
        "solve_ms": round(solve_ms, 4),
        "step_tflops": round(total_flops / (ms_step * 1e-3) / 1e12, 3),
        "setup_s": setup,
        "setup_points_per_s": round(n_total / max_over_ranks(sum(v for k, v in setup.items() if k != "h2d_points"),
                                                             world, dev), 1),
        "relres_vs_ktilde": relres,
        **({"accuracy": accuracy} if accuracy else {}),
        "method": w.method,
        **({"gmres_iterations": getattr(run, "krylov", None), "gmres_tol": w.gmres_tol} if w.method == "hybrid" else {}),
        "roofline": roof,
        "kernels": kernels,
        "e2e": {"value": round(n_total / (e2e_step * 1e-3), 1), "unit": "points/s",
                "ms_per_step": round(e2e_step, 4), "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world},
        "clocks": clk,
        "gpu_launches": int(launches),
        "factor_sets_allocated_in_region": sets_in_region,
    }
    return result


def main():
    args = parse()
    from paper_1701_02324_b200 import workloads as W
    w = W.CONFIGS[args.config]
    if args.points:
        w = w.scaled(args.points)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()

    if args.impl == "reference":
        if rank != 0:
            return
        r = oracle_arm(w, min(args.cpu_sample_n, w.n), max(args.steps, 1), cores)
        out = {"metric": "factorize+solve points/s", "value": round(r["value"], 1), "unit": "points/s",
               "n_gpus": args.gpus, "steps": max(args.steps, 1), "warmup": args.warmup,
               "ms_per_step": round(r["t_step"] * 1e3, 3), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic: seeded BASELINE generator",
               "config": {"workload": w.name, "n": w.n, "sample_n": min(args.cpu_sample_n, w.n)},
               "impl": "reference",
               "cpu_baseline": {"value": round(r["value"], 1), "unit": "points/s", "cores": r["cores"],
                                "kind": "port", "sample": r["sample"]},
               "e2e": {"value": round(r["value"], 1), "unit": "points/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0},
               "factorize_points_per_s": round(min(args.cpu_sample_n, w.n) / r["t_factorize"], 1),
               "solve_rhs_per_s": round(w.nrhs / r["t_solve"], 1)}
        print(json.dumps(out))
        return

    import torch
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
        torch.cuda.set_device(local)
        backend = os.environ.get("HKS_BENCH_BACKEND", "nccl")  # gloo: functional runs of P ranks on one GPU
        if backend == "nccl":
            # NCCL's init lines (ranks, NVLink / NVLS transport) on stderr so a
            # run's log shows every rank joined the communicator
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group(backend)
    result = gpu_arm(args, w, rank, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_arm(w, min(args.cpu_sample_n, w.n), args.cpu_steps, cores)
        result["cpu_baseline"] = {"value": round(r["value"], 1), "unit": "points/s", "cores": r["cores"],
                                  "kind": "port", "sample": r["sample"],
                                  "factorize_points_per_s": round(min(args.cpu_sample_n, w.n) / r["t_factorize"], 1),
                                  "solve_rhs_per_s": round(w.nrhs / r["t_solve"], 1)}
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
