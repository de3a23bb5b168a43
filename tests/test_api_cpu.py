"""CPU: the drop-in API surface and its validation (reference
tests/test_operators.py:245-264 and operators.py:120-129, 315-318, 334-349)."""

import pathlib
import numpy as np
import pytest

import paper_1711_00903_b200 as hx
from paper_1711_00903_b200.operators import OperatorInstance


def test_public_names_mirror_reference():
    for name in ("BENCHMARKS", "BP1", "BP35", "BP3", "AccessCounters", "FieldVector",
                 "OperatorInstance", "UnsupportedVariantError", "apply_bp1", "apply_bp3",
                 "apply_bp35", "apply_operator", "make_operator", "build_cube_mesh",
                 "perturb_mesh", "geometric_factors", "trilinear_jacobian",
                 "DegenerateGeometryError", "HexMesh", "GeometricFactors", "gl_rule",
                 "gll_rule", "lagrange_eval", "lagrange_deriv", "interp_matrix",
                 "diff_matrix_gll", "diff_matrix_gl", "traffic", "flop_model",
                 "roofline_global", "roofline_shared", "shared_bandwidth_ansatz",
                 "contract_dim", "measure_stream_bandwidth", "BandwidthCalibration",
                 "roofline_series", "RooflineSeries", "TrafficModel", "QuadratureRule",
                 "legendre_and_derivative", "OperatorMatrix", "interpolate_to_gl",
                 "project_to_gll"):
        assert hasattr(hx, name), name
    assert hx.BENCHMARKS == ("BP1.0", "BP3.5", "BP3.0")
    assert hx.VARIANTS == ("baseline", "fused", "symfused")


def test_make_operator_validation(perturbed_single):
    with pytest.raises(ValueError):
        hx.make_operator("BP9", 2, perturbed_single)
    with pytest.raises(ValueError):
        hx.make_operator(hx.BP1, 2, perturbed_single, variant="turbo")
    with pytest.raises(hx.UnsupportedVariantError):
        hx.make_operator(hx.BP35, 2, perturbed_single, variant="symfused")
    with pytest.raises(ValueError):
        hx.make_operator(hx.BP3, 2, perturbed_single, lam=-1.0)
    with pytest.raises(ValueError):
        hx.make_operator(hx.BP3, 16, perturbed_single)
    assert issubclass(hx.UnsupportedVariantError, ValueError)


def _fake_op(bp, deg=1, n_el=1):
    return OperatorInstance(bp, deg, 0.0, None, None, None, "fused", n_el)


def test_apply_shape_mismatch_and_bp_mismatch():
    op = _fake_op(hx.BP1, 2)
    with pytest.raises(ValueError):
        hx.apply_operator(op, hx.FieldVector.constant(1, 8))
    with pytest.raises(ValueError):
        hx.apply_bp35(_fake_op(hx.BP1), hx.FieldVector.constant(1, 8))
    with pytest.raises(ValueError):
        hx.apply_bp1(_fake_op(hx.BP3), hx.FieldVector.constant(1, 8))
    with pytest.raises(ValueError):
        hx.apply_bp3(_fake_op(hx.BP35), hx.FieldVector.constant(1, 8))


def test_field_vector():
    v = hx.FieldVector.random(3, 8, seed=5)
    np.testing.assert_array_equal(v.data.ravel(),
                                  np.random.default_rng(5).standard_normal(24))
    assert v.data.shape == (3, 8)
    with pytest.raises(ValueError):
        hx.FieldVector(2, 8, np.zeros(15))
    c = hx.FieldVector.constant(2, 8, 3.0)
    assert c.flat().sum() == 48.0
    import torch
    t = hx.FieldVector(2, 4, torch.arange(8, dtype=torch.float32))
    assert t.data.dtype == torch.float64 and tuple(t.data.shape) == (2, 4)
    assert not t.on_device


def test_counters_merge_and_linearity():
    a = hx.AccessCounters(1, 2, 3, 4, 5, 6, 7)
    a.merge(hx.AccessCounters(1, 1, 1, 1, 1, 1, 1))
    assert a == hx.AccessCounters(2, 3, 4, 5, 6, 7, 8)
    per = hx.element_counters(hx.BP3, "fused", 7)
    # fused global bytes equal Table 1 exactly (reference test_perf.py:80-95)
    t = hx.traffic(hx.BP3, 7)
    assert per["global_reads"] + per["global_writes"] == t.bytes_per_element
    assert per["flops"] == hx.flop_model(hx.BP3, "fused", 7)


def test_mesh_helpers():
    m = hx.build_cube_mesh(8, 2.0)
    assert m.n_el == 512
    a, det = hx.trilinear_jacobian(hx.build_cube_mesh(1, 2.0).vertices[0], 0.1, -0.2, 0.7)
    np.testing.assert_allclose(a, np.eye(3), atol=1e-14)
    flat = hx.build_cube_mesh(1, 2.0).vertices[0].copy()
    flat[:, 2] = 0.0
    with pytest.raises(hx.DegenerateGeometryError):
        hx.trilinear_jacobian(flat, 0.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        hx.build_cube_mesh(0, 2.0)


def test_every_module_imports():
    """Every product module, tool and entry point at least compiles and the
    package modules import without a GPU (GPU-only tests must not be the first
    place a syntax error shows up)."""
    import importlib
    import pathlib

    root = pathlib.Path(__file__).resolve().parents[1]
    for path in [root / "bench.py", root / "__graft_entry__.py",
                 *sorted((root / "paper_1711_00903_b200").glob("*.py")),
                 *sorted((root / "tools").glob("*.py")),
                 *sorted((root / "oracle").glob("*.py"))]:
        compile(path.read_text(), str(path), "exec")
    for path in sorted((root / "paper_1711_00903_b200").glob("*.py")):
        if path.stem != "__init__":
            importlib.import_module(f"paper_1711_00903_b200.{path.stem}")


def test_element_helper_validation_before_device():
    """interpolate_to_gl / project_to_gll reject bad shapes / matrices on the
    host (ValueError, like the reference's contract_dim) before any launch."""
    mat = hx.interp_matrix(3)
    with pytest.raises(ValueError):
        hx.interpolate_to_gl(np.zeros((5, 5, 5)), mat)
    with pytest.raises(ValueError):
        hx.project_to_gll(np.zeros((4, 4, 4)), mat)
    with pytest.raises(ValueError):
        hx.interpolate_to_gl(np.zeros((4, 4, 4)), np.zeros((4, 4)))


def _brute_contract(mat, t, axis):
    """Triple loop (reference test_reference_ops.py brute_force_contract)."""
    shape = list(t.shape)
    shape[axis] = mat.shape[0]
    out = np.zeros(shape)
    for idx in np.ndindex(*shape):
        src = list(idx)
        acc = 0.0
        for b in range(t.shape[axis]):
            src[axis] = b
            acc += mat[idx[axis], b] * t[tuple(src)]
        out[idx] = acc
    return out


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_contract_dim_known_answers(axis):
    """reference test_reference_ops.py:80-122: identity, constants through I,
    triple loop, adjointness, Kronecker form; torch tensors give the same."""
    import torch
    rng = np.random.default_rng(axis)
    t = rng.standard_normal((3, 3, 3))
    np.testing.assert_array_equal(hx.contract_dim(np.eye(3), t, axis), t)
    np.testing.assert_allclose(hx.contract_dim(hx.interp_matrix(2), np.full((3, 3, 3), 4.2), axis),
                               4.2, atol=1e-13)
    t2 = rng.standard_normal((2, 2, 2))
    mat = rng.standard_normal((3, 2))
    got = hx.contract_dim(mat, t2, axis)
    np.testing.assert_allclose(got, _brute_contract(mat, t2, axis), atol=1e-14)
    np.testing.assert_allclose(hx.contract_dim(mat, torch.from_numpy(t2), axis).numpy(), got,
                               atol=1e-15)
    m = rng.standard_normal((5, 4))
    u = rng.standard_normal((4, 4, 4))
    shape = [4, 4, 4]
    shape[axis] = 5
    v = rng.standard_normal(shape)
    lhs = np.vdot(hx.contract_dim(m, u, axis), v)
    rhs = np.vdot(u, hx.contract_dim(m.T, v, axis))
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_contract_dim_triple_is_kronecker(degree):
    m = hx.interp_matrix(degree).entries
    n = degree + 1
    u = np.random.default_rng(degree).standard_normal((n, n, n))
    t = hx.contract_dim(m, hx.contract_dim(m, hx.contract_dim(m, u, 1), 2), 0)
    np.testing.assert_allclose(t.ravel(), np.kron(m, np.kron(m, m)) @ u.ravel(), atol=1e-12)


def test_contract_dim_errors():
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError):
        hx.contract_dim(np.ones((3, 4)), rng.standard_normal((3, 3, 3)), 0)
    with pytest.raises(ValueError):
        hx.contract_dim(np.ones((3, 3)), rng.standard_normal((3, 3)), 0)
    with pytest.raises(ValueError):
        hx.contract_dim(np.ones((3, 3)), rng.standard_normal((3, 3, 3)), 3)


def test_measure_stream_bandwidth_validation():
    """reference test_perf.py:163-167 (checked before any allocation)."""
    with pytest.raises(ValueError):
        hx.measure_stream_bandwidth(1024)
    with pytest.raises(ValueError):
        hx.measure_stream_bandwidth(1 << 22, trials=2)


def test_report_calibrate_usage_errors():
    """The calibrate command's usage exits (reference cli.py:350-355) need no GPU."""
    from paper_1711_00903_b200.report import main
    assert main(["calibrate", "--bytes", "100"]) == 2
    assert main(["calibrate", "--bytes", str(1 << 22), "--repeats", "2"]) == 2


def _bench(*args, env=None):
    import json
    import subprocess
    import sys
    root = pathlib.Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, str(root / "bench.py"), *args], capture_output=True,
                         text=True, timeout=600, cwd=root, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [line for line in res.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_runs_the_reference_on_cpu():
    """bench.py --impl reference needs no GPU: it times the unmodified
    reference (baseline/_ref, tools/install_reference.sh) on the host."""
    d = _bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_gpus_2_relaunch_prints_one_line():
    """--gpus 2 outside torchrun re-launches under torch.distributed.run;
    only rank 0 runs the reference arm and prints."""
    d = _bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["n_gpus"] == 2
