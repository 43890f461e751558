"""``hikersolve``-compatible command line on the GPU path (cli.py of the
reference).

Subcommands gen / build / matvec / factor / solve / krr / bench / verify take the
reference's flags and config file (``key = value`` lines, ``#`` comments,
``lambda`` alias; precedence flags > file > defaults, config.py:17-120) and
print one JSON report of schema ``hikersolve-report-1`` ({version,
config_echo, timings, ranks, errors, krylov}; absent sections omitted,
cli.py:24,215-232).  Failures print one ``ERROR: ...`` line on stderr and
exit 1.  Every numerical stage runs in libhks; ``verify`` reports the
GPU-scale sampled-row metrics (metrics.sampled_error_report) instead of the
reference's dense oracle (limited to n <= 8192 there).

    python -m paper_1701_02324_b200 solve --points x.pts --rhs b.pts --lambda 1e-2
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

REPORT_VERSION = "hikersolve-report-1"
SHAPE_ALIASES = {"cube": "uniform_cube", "sphere": "sphere_surface", "mixture": "gaussian_mixture"}


from .config import Config, apply_overrides, parse_config_file  # noqa: E402

RunConfig = Config  # the name round-1 callers used
read_config = parse_config_file


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.exit(1, f"ERROR: {message}\n")


def _flags(p, *groups):
    if "points" in groups:
        p.add_argument("--points", required=True)
        p.add_argument("--normalize", choices=("unit-box",))
    if "build" in groups:
        p.add_argument("--leaf", type=int)
        p.add_argument("--tau", type=float)
        p.add_argument("--max-rank", dest="max_rank", type=int)
        p.add_argument("--samples", type=int)
        p.add_argument("--sample-mode", dest="sample_mode", choices=("uniform", "knn_augmented", "exact"))
        p.add_argument("--knn", type=int)
        p.add_argument("--kernel", choices=("gaussian", "laplace3d", "polynomial"))
        p.add_argument("--h", type=float)
        p.add_argument("--degree", type=int)
        p.add_argument("--shift", type=float)
        p.add_argument("--lambda", dest="lam", type=float)
    if "krylov" in groups:
        p.add_argument("--tol", type=float)
        p.add_argument("--maxiter", type=int)
        p.add_argument("--restart", type=int)
    p.add_argument("--config")
    p.add_argument("--threads", type=int)
    p.add_argument("--seed", type=int)
    if "gen" not in groups:
        p.add_argument("--out-stats")


def build_parser():
    from .data import SHAPES
    parser = _Parser(prog="hikersolve")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("gen", help="generate a synthetic point set")
    p.add_argument("--shape", required=True, choices=sorted(set(SHAPE_ALIASES) | set(SHAPES)))
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--d", type=int, default=3)
    p.add_argument("--clusters", type=int, default=4)
    p.add_argument("--out", required=True)
    p.add_argument("--format", choices=("binary", "csv"), default="binary")
    _flags(p, "gen")
    p = sub.add_parser("build", help="tree + skeletons, emit statistics")
    _flags(p, "points", "build")
    p = sub.add_parser("matvec", help="fast kernel summation")
    p.add_argument("--weights", required=True)
    p.add_argument("--out")
    p.add_argument("--verify", action="store_true", help="sampled-row error against the true kernel")
    _flags(p, "points", "build")
    p = sub.add_parser("factor", help="factorize and emit statistics")
    _flags(p, "points", "build")
    for name in ("solve", "krr"):
        p = sub.add_parser(name, help="solve (Ktilde + lambda I) x = b" if name == "solve" else
                           "kernel ridge regression")
        if name == "solve":
            _flags(p, "points", "build", "krylov")
            p.add_argument("--rhs", required=True)
            p.add_argument("--out")
        else:
            _flags(p, "build", "krylov")
            p.add_argument("--train", required=True)
            p.add_argument("--labels", required=True)
            p.add_argument("--test")
            p.add_argument("--test-labels", dest="test_labels")
            p.add_argument("--normalize", choices=("unit-box",))
            p.add_argument("--out-weights", dest="out_weights")
            p.add_argument("--out-pred", dest="out_pred")
        p.add_argument("--method", choices=("direct", "hybrid"), default="direct")
        p.add_argument("--operator", choices=("compressed", "dense"), default="compressed")
    p = sub.add_parser("bench", help="scaling benchmark")
    p.add_argument("--sizes", default="")
    p.add_argument("--dense-sizes", dest="dense_sizes", default="")
    p.add_argument("--shape", default="cube", choices=sorted(set(SHAPE_ALIASES) | set(SHAPES)))
    p.add_argument("--d", type=int, default=3)
    p.add_argument("--repeats", type=int, default=5)
    _flags(p, "build")
    p = sub.add_parser("verify", help="sampled-row error metrics on a standard instance")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--d", type=int, default=3)
    p.add_argument("--rows", type=int, default=256)
    _flags(p, "build")
    return parser


def _config(args, base=None):
    cfg = parse_config_file(args.config, base) if getattr(args, "config", None) else (base or Config())
    return apply_overrides(cfg, {k: v for k, v in vars(args).items() if v is not None})


def _sync():
    from . import _native as N
    N.torch().cuda.synchronize()


class _Clock:
    def __init__(self):
        self.t = {}

    def __call__(self, name, fn):
        _sync()
        t0 = time.perf_counter()
        out = fn()
        _sync()
        self.t[name] = time.perf_counter() - t0
        return out


def _points(path, normalize):
    from .pointio import load_points, normalize_unit_box
    ps = load_points(path)
    return normalize_unit_box(ps) if normalize == "unit-box" else ps


def _build(cfg, ps, clock):
    from . import build_operator, build_skeletons, build_tree, knn_bruteforce
    tr = clock("build", lambda: build_tree(ps, cfg.leaf, seed=cfg.seed))
    knn = None
    if cfg.sample_mode == "knn_augmented":
        knn = clock("knn", lambda: knn_bruteforce(tr.points, min(cfg.knn, tr.n - 1)))
    sk = clock("skeletonize", lambda: build_skeletons(tr, cfg.kernel_spec(), cfg.skeleton_config(), knn=knn))
    op = clock("assemble", lambda: build_operator(tr, sk, cfg.kernel_spec()))
    return tr, sk, op


def _report(cfg, command, extra=None, timings=None, ranks=None, errors=None, kr=None):
    echo = {"command": command, **cfg.echo(), **(extra or {})}
    rep = {"version": REPORT_VERSION, "config_echo": echo}
    if timings:
        rep["timings"] = {k: float(v) for k, v in timings.items()}
    if ranks:
        rep["ranks"] = {str(k): int(v) for k, v in ranks.items()}
    if errors:
        rep["errors"] = {k: float(v) for k, v in errors.items()}
    if kr is not None:
        rep["krylov"] = {"iterations": int(kr.iterations), "residuals": [float(r) for r in kr.residuals]}
    return rep


def _make_report(cfg, command, extra_echo=None, timings=None, ranks=None, errors=None, krylov_report=None):
    """The reference's report builder signature (cli.py:215-232)."""
    return _report(cfg, command, extra=extra_echo, timings=timings, ranks=ranks, errors=errors, kr=krylov_report)


def _solve_tree(cfg, op, f, b_tree, method, operator):
    from . import hybrid_solve, solve
    if method == "direct":
        return solve(f, b_tree, in_tree_order=True), None
    mode = "dense_oracle" if operator == "dense" else "compressed"
    return hybrid_solve(op, f, b_tree, tol=cfg.tol, max_iter=cfg.maxiter, restart=cfg.restart, operator_mode=mode)


def cmd_gen(args):
    from .data import generate
    from .pointio import save_points
    cfg = _config(args)
    shape = SHAPE_ALIASES.get(args.shape, args.shape)
    t0 = time.perf_counter()
    save_points(generate(shape, args.n, cfg.seed, d=args.d, k_clusters=args.clusters), args.out, format=args.format)
    return _report(cfg, "gen", {"shape": shape, "n": args.n, "d": args.d, "out": args.out},
                   {"generate": time.perf_counter() - t0})


def cmd_build(args):
    cfg = _config(args)
    ps = _points(args.points, args.normalize)
    clock = _Clock()
    tr, sk, _ = _build(cfg, ps, clock)
    return _report(cfg, "build", {"points": args.points, "n": ps.n, "d": ps.d}, clock.t, sk.max_rank_per_level(tr))


def cmd_matvec(args):
    from . import hmatvec, sampled_error_report
    from .pointio import load_vector, save_vector
    cfg = _config(args)
    ps = _points(args.points, args.normalize)
    w = load_vector(args.weights)
    if w.shape[0] != ps.n:
        raise ValueError(f"weights length {w.shape[0]} does not match n={ps.n}")
    clock = _Clock()
    tr, sk, op = _build(cfg, ps, clock)
    perm = np.asarray(tr.perm)
    u_tree = clock("matvec", lambda: hmatvec(op, w[perm], cfg.lam))
    u = np.empty_like(u_tree)
    u[perm] = u_tree
    if args.out:
        save_vector(u, args.out)
    errors = None
    if args.verify:
        from .metrics import cross_sum, sample_rows
        from . import _native as N
        R = sample_rows(tr.n, 256, cfg.seed)
        x = tr.device_points()
        ref = cross_sum(op.kernel, x, x, N.to_device(w[perm]).reshape(1, -1), rows=N.to_device(R))[0].cpu().numpy()
        ref += cfg.lam * w[perm][R]
        errors = {"matvec_relerr": np.linalg.norm(u_tree[R] - ref) / np.linalg.norm(ref)}
    return _report(cfg, "matvec", {"points": args.points, "n": ps.n, "d": ps.d}, clock.t,
                   sk.max_rank_per_level(tr), errors)


def cmd_factor(args):
    from . import factorize
    cfg = _config(args)
    ps = _points(args.points, args.normalize)
    clock = _Clock()
    tr, sk, op = _build(cfg, ps, clock)
    f = clock("factorize", lambda: factorize(op, cfg.lam))
    for level, secs in f.level_seconds.items():
        clock.t[f"factorize_level{level}"] = secs
    errors = {f"z_cond_L{lev}": c for lev, c in f.z_cond_per_level().items()}
    return _report(cfg, "factor", {"points": args.points, "n": ps.n, "d": ps.d}, clock.t,
                   sk.max_rank_per_level(tr), errors or None)


def cmd_solve(args):
    from . import factorize, hmatvec
    from .pointio import load_vector, save_vector
    cfg = _config(args)
    ps = _points(args.points, args.normalize)
    b = load_vector(args.rhs)
    if b.shape[0] != ps.n:
        raise ValueError(f"rhs length {b.shape[0]} does not match n={ps.n}")
    clock = _Clock()
    tr, sk, op = _build(cfg, ps, clock)
    f = clock("factorize", lambda: factorize(op, cfg.lam))
    perm = np.asarray(tr.perm)
    x_tree, kr = clock("solve", lambda: _solve_tree(cfg, op, f, b[perm], args.method, args.operator))
    x = np.empty_like(x_tree)
    x[perm] = x_tree
    if args.out:
        save_vector(x, args.out)
    resid = hmatvec(op, x_tree, cfg.lam) - b[perm]
    errors = {"residual_vs_Ktilde": np.linalg.norm(resid) / np.linalg.norm(b)}
    if kr is not None:
        errors["final_residual"] = kr.final_residual
    return _report(cfg, "solve", {"points": args.points, "n": ps.n, "d": ps.d, "method": args.method}, clock.t,
                   sk.max_rank_per_level(tr), errors, kr)


def cmd_krr(args):
    from . import cross_predict, factorize, hmatvec
    from .pointio import load_vector, save_vector
    cfg = _config(args)
    train = _points(args.train, args.normalize)
    y = load_vector(args.labels)
    if y.shape[0] != train.n:
        raise ValueError(f"labels length {y.shape[0]} does not match n={train.n}")
    clock = _Clock()
    tr, sk, op = _build(cfg, train, clock)
    f = clock("factorize", lambda: factorize(op, cfg.lam))
    perm = np.asarray(tr.perm)
    w_tree, kr = clock("fit", lambda: _solve_tree(cfg, op, f, y[perm], args.method, args.operator))
    if args.out_weights:
        w = np.empty_like(w_tree)
        w[perm] = w_tree
        save_vector(w, args.out_weights)
    pred_train = hmatvec(op, w_tree, 0.0)
    errors = {"rmse_train": float(np.sqrt(np.mean((pred_train - y[perm]) ** 2)))}
    if args.test:
        test = _points(args.test, args.normalize)
        pred = clock("predict", lambda: cross_predict(cfg.kernel_spec(), test, tr.points, w_tree))
        if args.out_pred:
            save_vector(pred, args.out_pred)
        if args.test_labels:
            yt = load_vector(args.test_labels)
            if yt.shape[0] != test.n:
                raise ValueError(f"test labels length {yt.shape[0]} does not match n={test.n}")
            errors["rmse_test"] = float(np.sqrt(np.mean((pred - yt) ** 2)))
    return _report(cfg, "krr", {"train": args.train, "n": train.n, "d": train.d, "method": args.method}, clock.t,
                   sk.max_rank_per_level(tr), errors, kr)


def standard_pipeline(cfg):
    """The GPU stages packaged for metrics.scaling_benchmark (cli.py:465-490
    of the reference): tree, kNN (knn_augmented only) + skeletons,
    operator, factorize, solve in tree order."""
    from . import build_operator, build_skeletons, build_tree, factorize, knn_bruteforce, solve
    from .metrics import BenchmarkPipeline
    kernel = cfg.kernel_spec()

    def skeletonize(tr):
        knn = None
        if cfg.sample_mode == "knn_augmented":
            knn = knn_bruteforce(tr.points, min(cfg.knn, tr.n - 1))
        return build_skeletons(tr, kernel, cfg.skeleton_config(), knn=knn)

    return BenchmarkPipeline(
        build=lambda ps: build_tree(ps, cfg.leaf, seed=cfg.seed),
        skeletonize=skeletonize,
        assemble=lambda tr, sk: build_operator(tr, sk, kernel),
        factorize=lambda op: factorize(op, cfg.lam),
        solve=lambda f, b: solve(f, b, in_tree_order=True),
    )


def _sizes(text):
    return [int(v) for v in text.split(",") if v.strip()]


class _BenchConfig:
    def __init__(self, shape, d, kernel):
        self.shape, self.d, self.kernel = shape, d, kernel


def cmd_bench(args):
    """Scaling benchmark (cli.py:429-454): phase times per size as
    `<phase>_n<n>` timings and the fitted exponents as `exponent_<phase>`."""
    from .metrics import scaling_benchmark
    cfg = _config(args)
    sizes, dense_sizes = _sizes(args.sizes), _sizes(args.dense_sizes)
    if not sizes and not dense_sizes:
        raise ValueError("bench needs --sizes and/or --dense-sizes")
    shape = SHAPE_ALIASES.get(args.shape, args.shape)
    res = scaling_benchmark(sizes, _BenchConfig(shape, args.d, cfg.kernel_spec()), cfg.seed,
                            pipeline=standard_pipeline(cfg) if sizes else None,
                            dense_sizes=dense_sizes or None, solve_repeats=args.repeats)
    timings = {}
    for phase, values in res["timings"].items():
        ns = res["dense_sizes"] if phase.startswith("dense") else res["sizes"]
        timings.update({f"{phase}_n{n}": v for n, v in zip(ns, values)})
    errors = {f"exponent_{phase}": p for phase, p in res["exponents"].items()}
    extra = {"sizes": res["sizes"], "shape": shape, "d": args.d}
    if dense_sizes:
        extra["dense_sizes"] = dense_sizes
    return _report(cfg, "bench", extra, timings, errors=errors)


VERIFY_DEFAULTS = dict(kernel="gaussian", h=0.3, lam=1e-2, tau=1e-7, sample_mode="exact", max_rank=384)


def cmd_verify(args):
    from . import factorize, sampled_error_report
    from .data import generate
    cfg = _config(args, Config(**VERIFY_DEFAULTS))
    ps = generate("uniform_cube", args.n, cfg.seed, d=args.d)
    clock = _Clock()
    tr, sk, op = _build(cfg, ps, clock)
    f = clock("factorize", lambda: factorize(op, cfg.lam))
    rep = clock("verify", lambda: sampled_error_report(op, f, rows=args.rows, seed=cfg.seed))
    errors = {f"sampled_{k}": v for k, v in rep.items() if k != "rows"}
    return _report(cfg, "verify", {"n": args.n, "d": args.d, "rows": rep["rows"]}, clock.t,
                   sk.max_rank_per_level(tr), errors)


COMMANDS = {"gen": cmd_gen, "build": cmd_build, "matvec": cmd_matvec, "factor": cmd_factor, "solve": cmd_solve,
            "krr": cmd_krr, "bench": cmd_bench, "verify": cmd_verify}


def run(argv=None):
    args = build_parser().parse_args(argv)
    try:
        report = COMMANDS[args.command](args)
    except Exception as exc:  # noqa: BLE001 -- the reference's ERROR: convention (cli.py:524-530)
        print(f"ERROR: {exc}", file=sys.stderr)
        return 1
    text = json.dumps(report, indent=2)
    print(text)
    if getattr(args, "out_stats", None):
        with open(args.out_stats, "w") as fh:
            fh.write(text + "\n")
    return 0


def main():
    sys.exit(run())
