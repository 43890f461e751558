"""The hikersolve-compatible CLI end to end on the GPU (gen -> build /
factor / solve / matvec / krr / verify), reports checked against the
schema sections and the oracle where one applies."""

import json
from pathlib import Path

import jsonschema
import numpy as np
import pytest

from oracle import hks_oracle as O

pytestmark = pytest.mark.gpu


def _run(capsys, *argv):
    from paper_1701_02324_b200 import cli
    rc = cli.run(list(argv))
    cap = capsys.readouterr()
    assert rc == 0, cap.err
    rep = json.loads(cap.out)
    # every GPU report against the reference's own REPORT_SCHEMA (tests/helpers.py:145-177)
    jsonschema.validate(rep, json.loads((Path(__file__).parent / "golden" / "report_schema.json").read_text()))
    return rep


def test_cli_pipeline(tmp_path, capsys):
    from paper_1701_02324_b200.pointio import load_vector, save_vector
    pts = tmp_path / "x.pts"
    _run(capsys, "gen", "--shape", "cube", "--n", "1500", "--d", "3", "--out", str(pts), "--seed", "2")
    common = ["--points", str(pts), "--leaf", "128", "--max-rank", "48", "--tau", "1e-7", "--h", "0.4",
              "--lambda", "1e-2", "--sample-mode", "knn_augmented", "--knn", "8", "--samples", "192"]
    rep = _run(capsys, "build", *common)
    assert set(rep["timings"]) >= {"build", "knn", "skeletonize", "assemble"} and 1 <= rep["ranks"]["1"] <= 48
    rep = _run(capsys, "factor", *common)
    assert "factorize" in rep["timings"] and any(k.startswith("z_cond_L") for k in rep["errors"])
    b = np.random.default_rng(1).standard_normal(1500)
    save_vector(b, tmp_path / "b.pts")
    rep = _run(capsys, "solve", *common, "--rhs", str(tmp_path / "b.pts"), "--out", str(tmp_path / "xs.pts"))
    # the algorithm's own stability on this instance: the CPU oracle gives ~1e-7 here too
    assert rep["errors"]["residual_vs_Ktilde"] < 1e-6
    rep = _run(capsys, "solve", *common, "--rhs", str(tmp_path / "b.pts"), "--method", "hybrid", "--tol", "1e-10")
    assert rep["krylov"]["iterations"] >= 1 and rep["errors"]["final_residual"] < 1e-9  # GMRES refines it
    rep = _run(capsys, "matvec", *common, "--weights", str(tmp_path / "b.pts"), "--out", str(tmp_path / "u.pts"),
               "--verify")
    assert 0 < rep["errors"]["matvec_relerr"] < 1.0
    u = load_vector(tmp_path / "u.pts")
    x = load_vector(tmp_path / "xs.pts")
    assert u.shape == (1500,) and x.shape == (1500,)


def test_cli_krr(tmp_path, capsys):
    from paper_1701_02324_b200.pointio import load_vector, save_points, save_vector
    from paper_1701_02324_b200.data import PointSet
    rng = np.random.default_rng(4)
    xtr, xte = rng.random((1200, 2)), rng.random((200, 2))
    f = lambda z: np.sin(3 * z[:, 0]) + z[:, 1] ** 2
    save_points(PointSet(xtr), tmp_path / "tr.pts")
    save_points(PointSet(xte), tmp_path / "te.pts")
    save_vector(f(xtr), tmp_path / "ytr.pts")
    save_vector(f(xte), tmp_path / "yte.pts")
    rep = _run(capsys, "krr", "--train", str(tmp_path / "tr.pts"), "--labels", str(tmp_path / "ytr.pts"),
               "--test", str(tmp_path / "te.pts"), "--test-labels", str(tmp_path / "yte.pts"),
               "--out-weights", str(tmp_path / "w.pts"), "--out-pred", str(tmp_path / "p.pts"),
               "--leaf", "128", "--h", "0.3", "--lambda", "1e-3", "--max-rank", "64", "--tau", "1e-10")
    assert rep["errors"]["rmse_test"] < 0.1 and rep["errors"]["rmse_train"] < 0.1
    # the prediction is K(test, train) w exactly (cli.py:415-422), checked against dense oracle rows
    w = load_vector(tmp_path / "w.pts")
    pred = load_vector(tmp_path / "p.pts")
    ref = O.kernel_block("gaussian", xte, xtr, h=0.3) @ w
    np.testing.assert_allclose(pred, ref, rtol=0, atol=1e-11 * np.abs(ref).max())


def test_cli_verify(capsys):
    rep = _run(capsys, "verify", "--n", "2000", "--rows", "128")
    e = rep["errors"]
    assert e["sampled_residual_vs_Ktilde"] < 1e-6  # oracle/hks_oracle.py on this instance: 1.36e-7
    assert e["sampled_matvec_relerr_vs_K"] < 1e-3  # exact sampling, tau 1e-7: Ktilde is close to K
    assert rep["config_echo"]["sample_mode"] == "exact"


def test_cli_bench(capsys):
    """The scaling benchmark through the GPU pipeline (test_cli.py:168-178 of
    the reference): per-size phase timings and fitted exponents, dense
    contrast included."""
    rep = _run(capsys, "bench", "--sizes", "128,256", "--dense-sizes", "64,128", "--leaf", "32", "--max-rank", "16",
               "--samples", "32", "--repeats", "2", "--threads", "1")
    assert "exponent_factorize" in rep["errors"] and "exponent_dense_factor" in rep["errors"]
    assert "factorize_n256" in rep["timings"] and "dense_solve_n128" in rep["timings"]
    assert rep["config_echo"]["sizes"] == [128, 256] and rep["config_echo"]["dense_sizes"] == [64, 128]
    assert all(v > 0 for v in rep["timings"].values())


def test_scaling_benchmark_dense_matches_oracle():
    """dense_kernel_matrix on the GPU equals the oracle's dense K + lam I."""
    from paper_1701_02324_b200 import metrics
    from paper_1701_02324_b200.data import generate
    from paper_1701_02324_b200.kernels import KernelSpec
    ps = generate("uniform_cube", 300, 5, d=3)
    k = KernelSpec("gaussian", h=0.4, regularization=0.1)
    A = metrics.dense_kernel_matrix(k, ps, 0.1)
    ref = O.kernel_block("gaussian", ps.coords, ps.coords, h=0.4) + 0.1 * np.eye(300)
    np.testing.assert_allclose(A, ref, rtol=1e-13, atol=1e-15)
