"""CLI host logic without a GPU (paper_1701_02324_b200/cli.py, pointio.py):
config precedence and file errors, PTS1 / CSV round trips and their error
messages, the ERROR: convention (cli.py / config.py / data.py of the
reference; tests/test_cli.py, tests/test_data.py there)."""

import json
import struct

import numpy as np
import pytest

from paper_1701_02324_b200 import cli
from paper_1701_02324_b200.data import PointSet
from paper_1701_02324_b200.pointio import (PointFormatError, load_points, load_vector, normalize_unit_box,
                                           save_points, save_vector)


def test_pts1_roundtrip_and_layout(tmp_path):
    x = np.random.default_rng(0).standard_normal((7, 3))
    p = tmp_path / "a.pts"
    save_points(PointSet(x), p)
    raw = p.read_bytes()
    assert raw[:4] == b"PTS1" and struct.unpack("<QQ", raw[4:20]) == (7, 3) and len(raw) == 20 + 8 * 21
    assert np.array_equal(load_points(p).coords, x)
    save_points(PointSet(x), tmp_path / "a.csv", format="csv")
    assert np.array_equal(load_points(tmp_path / "a.csv", format="csv").coords, x)  # 17 digits: exact
    save_vector(np.arange(5.0), tmp_path / "v.pts")
    assert np.array_equal(load_vector(tmp_path / "v.pts"), np.arange(5.0))


def test_pts1_errors(tmp_path):
    p = tmp_path / "bad.pts"
    p.write_bytes(b"XXXX" + struct.pack("<QQ", 1, 1) + b"\0" * 8)
    with pytest.raises(PointFormatError, match="bad magic"):
        load_points(p)
    p.write_bytes(b"PTS1" + struct.pack("<QQ", 4, 2) + b"\0" * 16)
    with pytest.raises(PointFormatError, match="truncated payload"):
        load_points(p)
    p.write_bytes(b"PTS1")
    with pytest.raises(PointFormatError, match="truncated header"):
        load_points(p)
    c = tmp_path / "bad.csv"
    c.write_text("1,2\n3,x\n")
    with pytest.raises(PointFormatError, match="line 2: non-numeric"):
        load_points(c, format="csv")
    c.write_text("1,2\n3\n")
    with pytest.raises(PointFormatError, match="line 2: expected 2 columns"):
        load_points(c, format="csv")
    save_points(PointSet(np.ones((3, 2))), p)
    with pytest.raises(PointFormatError, match="d=1"):
        load_vector(p)


def test_unit_box():
    ps = normalize_unit_box(PointSet(np.array([[1.0, 5.0], [3.0, 5.0]])))
    assert np.array_equal(ps.coords, [[0.0, 0.0], [1.0, 0.0]])


def test_config_precedence_and_errors(tmp_path):
    f = tmp_path / "c.cfg"
    f.write_text("# comment\nlambda = 0.25\nleaf = 32  # trailing\nh=2\n")
    args = cli.build_parser().parse_args(["build", "--points", "p", "--config", str(f), "--h", "3"])
    cfg = cli._config(args)
    assert (cfg.lam, cfg.leaf, cfg.h) == (0.25, 32, 3.0)  # flag beats file beats default
    assert cli.RunConfig().max_rank == 64 and cfg.echo()["lambda"] == 0.25
    f.write_text("bogus = 1\n")
    with pytest.raises(ValueError, match="line 1: unknown key"):
        cli.read_config(f)
    f.write_text("leaf = many\n")
    with pytest.raises(ValueError, match="bad value"):
        cli.read_config(f)
    f.write_text("leaf\n")
    with pytest.raises(ValueError, match="expected key = value"):
        cli.read_config(f)


def test_gen_report_and_error_convention(tmp_path, capsys):
    out = tmp_path / "g.pts"
    assert cli.run(["gen", "--shape", "cube", "--n", "50", "--d", "4", "--out", str(out), "--seed", "3"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["version"] == "hikersolve-report-1" and rep["config_echo"]["command"] == "gen"
    assert set(rep) == {"version", "config_echo", "timings"}  # absent sections omitted
    assert load_points(out).coords.shape == (50, 4)
    assert cli.run(["build", "--points", str(tmp_path / "missing.pts")]) == 1
    assert capsys.readouterr().err.startswith("ERROR: ")
    with pytest.raises(SystemExit) as e:
        cli.run(["solve", "--points", "x"])  # --rhs missing: parser error, same convention
    assert e.value.code == 1


def test_bench_host_checks(capsys):
    """bench's argument errors (cli.py:429-434) and the scaling benchmark's
    host logic (oracle.py:170-187), no GPU work."""
    from paper_1701_02324_b200 import metrics
    assert cli.run(["bench"]) == 1
    assert "bench needs --sizes and/or --dense-sizes" in capsys.readouterr().err
    with pytest.raises(ValueError, match="injected pipeline"):
        metrics.scaling_benchmark([128], None, 0, pipeline=None)
    assert metrics.scaling_benchmark([], None, 0) == {"sizes": [], "timings": {}, "exponents": {}}
    n = np.array([128, 256, 512, 1024])
    assert metrics.fit_exponent(n, 3e-6 * n ** 1.5) == pytest.approx(1.5)
    with pytest.raises(ValueError, match="limited to n <= 8192"):
        metrics.dense_kernel_matrix(None, PointSet(np.zeros((8193, 1))), 1.0)


SCHEMA = json.loads((__import__("pathlib").Path(__file__).parent / "golden" / "report_schema.json").read_text())


def test_report_schema_property_suite():
    """200 randomized reports through the reference's report builder
    signature (cli.py:215-232) all satisfy the reference's REPORT_SCHEMA
    (tests/helpers.py:145-177, frozen by tests/golden/make_golden.py), with
    absent sections omitted, never null (test_cli.py:281-309)."""
    import jsonschema
    from paper_1701_02324_b200 import Config, KrylovReport
    rng = np.random.default_rng(12)
    cfg = Config()
    for _ in range(200):
        timings = ranks = errors = krep = None
        if rng.random() < 0.7:
            timings = {f"phase{i}": float(rng.random()) for i in range(rng.integers(1, 4))}
        if rng.random() < 0.5:
            ranks = {int(i): int(rng.integers(0, 64)) for i in range(rng.integers(1, 5))}
        if rng.random() < 0.5:
            errors = {f"metric{i}": float(rng.random()) for i in range(rng.integers(1, 4))}
        if rng.random() < 0.4:
            krep = KrylovReport(iterations=int(rng.integers(0, 50)),
                                residuals=[float(v) for v in rng.random(rng.integers(0, 9))])
        rep = cli._make_report(cfg, "test", timings=timings, ranks=ranks, errors=errors, krylov_report=krep)
        jsonschema.validate(rep, SCHEMA)
        assert None not in rep.values()
        json.dumps(rep)
    bad = cli._make_report(cfg, "test")
    bad["extra"] = 1
    with pytest.raises(jsonschema.ValidationError):
        jsonschema.validate(bad, SCHEMA)


def test_config_module_matches_reference_surface(tmp_path):
    """Config / parse_config_file / apply_overrides (config.py:17-120):
    defaults, alias, precedence, thread resolution, error messages."""
    from paper_1701_02324_b200 import Config
    from paper_1701_02324_b200.config import apply_overrides, parse_config_file
    f = tmp_path / "c.cfg"
    f.write_text("# comment\nlambda = 0.5\nleaf = 128  # trailing\nsample_mode = knn_augmented\n")
    cfg = parse_config_file(f)
    assert (cfg.lam, cfg.leaf, cfg.sample_mode, cfg.max_rank) == (0.5, 128, "knn_augmented", 64)
    cfg = apply_overrides(cfg, {"leaf": 64, "bogus": 3})
    assert cfg.leaf == 64 and cfg.lam == 0.5
    assert Config(threads=4).effective_threads() == 4 and Config(threads=0).effective_threads() >= 1
    assert list(Config().echo())[:6] == ["kernel", "h", "degree", "shift", "lambda", "leaf"]
    for text, msg in (("warp_factor = 9\n", "unknown key"), ("tau: 1e-5\n", "line 1"), ("leaf = many\n", "bad value")):
        f.write_text(text)
        with pytest.raises(ValueError, match=msg):
            parse_config_file(f)
