"""CPU-only checks of the drop-in boundary: libhks.so loads, exports every
entry point include/hks.h declares, and the host-side layout / plan logic
agrees with the reference's tree arithmetic (no GPU compute calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hks.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(hks_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1701_02324_b200 import _native as N
    lib = N.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/hks.h but not exported"
    assert lib.hks_abi_version() == 1


def test_python_signatures_cover_the_header():
    from paper_1701_02324_b200 import _native as N
    import paper_1701_02324_b200.skeleton  # noqa: F401  (registers its entry points)
    missing = [n for n in declared_symbols() if n not in N.SIGNATURES and n != "hks_last_error"]
    assert not missing, missing


@pytest.mark.parametrize("n,leaf", [(10, 5), (1000, 64), (4097, 256), (262144, 512)])
def test_layout_matches_reference_ranges(n, leaf):
    from paper_1701_02324_b200 import _native as N
    from paper_1701_02324_b200.tree import node_ranges, tree_depth
    from oracle import hks_oracle as O
    depth = tree_depth(n, leaf)
    assert depth == O.tree_depth(n, leaf)
    b, e = node_ranges(n, depth)
    ob, oe = O.node_ranges(n, depth)
    assert np.array_equal(b, ob) and np.array_equal(e, oe)
    lay = N.Layout(n, depth, 64)
    nn = (1 << (depth + 1)) - 1
    first_leaf = (1 << depth) - 1
    sizes = e - b
    # leaf LU slots are size^2, contiguous in heap order
    lu = lay.off[N.BUF_LEAF_LU]
    assert np.all(lu[:first_leaf] == -1)
    assert np.array_equal(np.diff(lu[first_leaf:]), (sizes[first_leaf:-1] ** 2))
    assert lay.sizes[N.BUF_LEAF_LU] == int((sizes[first_leaf:] ** 2).sum())
    # rank caps: leaves min(s, m); internal min(s, r_l + r_r); root no skeleton
    assert lay.off[N.BUF_INTERP, 0] == -1 and lay.off[N.BUF_SKEL, 0] == -1
    assert lay.sizes[N.BUF_STATS] == 3 * nn


def test_layout_rejects_bad_arguments():
    from paper_1701_02324_b200 import _native as N
    with pytest.raises(N.HksError):
        N.Layout(0, 0, 1)
    assert "bad arguments" in N.last_error()


def test_workload_generators_match_baseline_shapes():
    from paper_1701_02324_b200 import workloads as W
    for key, w in W.CONFIGS.items():
        small = w.scaled(1000)
        x = W.points(small, 0)
        assert x.shape == (1000, w.d) and np.all(np.isfinite(x))
        if w.generator == "sparse784":
            assert np.allclose(np.linalg.norm(x, axis=1), 1.0)
            assert 0.7 < np.mean(x == 0.0) < 0.9
        if w.generator == "mixture8":
            assert np.allclose(x.mean(0), 0.0, atol=1e-12) and np.allclose(x.std(0), 1.0)
    c1 = W.points(W.CONFIGS["C1"].scaled(64), 0)
    assert np.array_equal(c1, np.random.default_rng([0, 0, 0]).random((64, 8)))


def test_public_api_matches_reference_names():
    import paper_1701_02324_b200 as hk
    reference_all = {
        "Config", "DenseFactor", "Factorization", "FactorizationError", "HierarchicalOperator",
        "KernelSpec", "KrylovReport", "PartitionTree", "PivotedQRResult", "PointSet", "Skeleton",
        "SkeletonConfig", "SkeletonSet", "SingularMatrixError", "build_operator", "build_skeletons",
        "build_tree", "eval_block", "eval_system_diag_shift", "factor_dense", "factorize", "generate",
        "gmres", "hmatvec", "hybrid_solve", "interpolative_decomposition", "knn_bruteforce", "levels",
        "load_points", "materialize_ktilde", "pivoted_qr", "save_points", "solve", "solve_dense",
        "solve_multi", "upward_pass"}
    # Config / load_points / save_points are the reference's host CLI and
    # file-format layer, outside the accelerated path
    out_of_scope = {"Config", "load_points", "save_points"}
    missing = sorted(reference_all - out_of_scope - set(hk.__all__))
    assert not missing, missing


def test_kernel_spec_validation_matches_reference():
    import paper_1701_02324_b200 as hk
    for spec in [dict(family="gaussian", h=0.0), dict(family="gaussian", h=-1.0),
                 dict(family="polynomial", degree=0), dict(family="polynomial", shift=-0.5),
                 dict(family="nope"), dict(regularization=-1.0)]:
        with pytest.raises(ValueError):
            hk.KernelSpec(**spec)
    with pytest.raises(ValueError):
        hk.SkeletonConfig(tau=0.0)
    with pytest.raises(ValueError):
        hk.SkeletonConfig(sample_mode="bogus")


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_1701_02324_b200 as hk
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hk.eval_block(hk.KernelSpec(), np.zeros((2, 2)), np.zeros((2, 2)))


def test_profile_kind_names_match_step_kinds():
    """KIND_NAMES (hks_profile's per-kind layout) follows plan.h's StepKind
    enum up to kNumKinds; the stream-control kinds after it are not timed."""
    import re
    from pathlib import Path
    from paper_1701_02324_b200 import _native as N
    src = (Path(__file__).resolve().parents[1] / "paper_1701_02324_b200" / "csrc" / "plan.h").read_text()
    body = re.search(r"enum StepKind \{(.*?)\};", src, re.S).group(1)
    body = re.sub(r"//[^\n]*", "", body)
    kinds = [k.strip() for k in body.split(",") if k.strip()]
    nk = int(re.search(r"constexpr int kNumKinds = (\d+);", src).group(1))
    assert kinds[nk:] == ["ST_FORK", "ST_JOIN"]
    assert len(N.KIND_NAMES) == nk
    assert [k[3:].lower() for k in kinds[:nk]] == [{"eval": "eval_cm"}.get(n, n) for n in N.KIND_NAMES]
