"""GPU: device element helpers interpolate_to_gl / project_to_gll
(reference operators.py:352-364) through hx_interp_elements, against the
reference's golden outputs and its own known-answer tests
(test_operators.py:30-64, TestInterpolationProjection)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402
from oracle import hexbench_oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("deg", [1, 2, 3, 5, 7, 8, 15])
def test_golden_reference_vectors(deg, golden):
    """Batched device helpers == the reference's per-element functions."""
    mat = hx.interp_matrix(deg)
    gl = hx.interpolate_to_gl(golden[f"helper_N{deg}_q"], mat)
    np.testing.assert_allclose(gl, golden[f"helper_N{deg}_gl"], rtol=0, atol=1e-13)
    gll = hx.project_to_gll(golden[f"helper_N{deg}_t"], mat)
    np.testing.assert_allclose(gll, golden[f"helper_N{deg}_gll"], rtol=0, atol=1e-13)
    # one element at a time, exactly the reference call shape
    one = hx.interpolate_to_gl(golden[f"helper_N{deg}_q"][1], mat)
    assert one.shape == (deg + 2,) * 3
    np.testing.assert_array_equal(one, gl[1])


@pytest.mark.parametrize("deg", range(1, 16))
def test_every_degree_against_oracle_ragged_batch(deg):
    rng = np.random.default_rng(deg)
    n, m = deg + 1, deg + 2
    mat = hx.interp_matrix(deg).entries
    for n_el in (1, 7, 40):
        q = rng.standard_normal((n_el, n, n, n))
        t = rng.standard_normal((n_el, m, m, m))
        got = hx.interpolate_to_gl(q, mat)
        assert orc.rel_l2(got, orc.interp_passes(mat, q)) <= 1e-13
        got = hx.project_to_gll(t, mat)
        assert orc.rel_l2(got, orc.project_passes(mat, t)) <= 1e-13


def test_constant_preserved():
    """test_operators.py:31-34."""
    q = np.full((3, 3, 3), 2.5)
    out = hx.interpolate_to_gl(q, hx.interp_matrix(2))
    np.testing.assert_allclose(out, 2.5, atol=1e-13)


def test_linear_field_exact():
    """test_operators.py:36-41."""
    gll = hx.gll_rule(2).nodes
    gl = hx.gl_rule(3).nodes
    q = np.broadcast_to(gll, (2, 2, 2)).copy()
    out = hx.interpolate_to_gl(q, hx.interp_matrix(1))
    np.testing.assert_allclose(out, np.broadcast_to(gl, (3, 3, 3)), atol=1e-14)


def test_matches_dense_kronecker(rng):
    """test_operators.py:43-53."""
    m = hx.interp_matrix(2).entries
    q = rng.standard_normal((3, 3, 3))
    big = np.kron(m, np.kron(m, m))
    np.testing.assert_allclose(hx.interpolate_to_gl(q, hx.interp_matrix(2)).ravel(),
                               big @ q.ravel(), atol=1e-13)
    v = rng.standard_normal((4, 4, 4))
    np.testing.assert_allclose(hx.project_to_gll(v, hx.interp_matrix(2)).ravel(),
                               big.T @ v.ravel(), atol=1e-13)


def test_adjointness(rng):
    """test_operators.py:55-61."""
    op = hx.interp_matrix(3)
    u = rng.standard_normal((4, 4, 4))
    v = rng.standard_normal((5, 5, 5))
    lhs = np.vdot(hx.interpolate_to_gl(u, op), v)
    rhs = np.vdot(u, hx.project_to_gll(v, op))
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


def test_zero():
    """test_operators.py:63-64."""
    assert not hx.project_to_gll(np.zeros((3, 3, 3)), hx.interp_matrix(1)).any()


def test_device_tensors_stay_on_device():
    mat = hx.interp_matrix(7)
    q = torch.randn(5, 8, 8, 8, dtype=torch.float64, device="cuda")
    t = hx.interpolate_to_gl(q, mat)
    assert t.is_cuda and t.shape == (5, 9, 9, 9)
    back = hx.project_to_gll(t, mat)
    assert back.is_cuda and back.shape == (5, 8, 8, 8)
    # BP1.0 is project(GwJ * interpolate(q)): with unit weights it is I^T I
    ref = orc.project_passes(mat.entries, orc.interp_passes(mat.entries, q.cpu().numpy()))
    assert orc.rel_l2(back.cpu().numpy(), ref) <= 1e-13


def test_errors():
    mat = hx.interp_matrix(3)
    with pytest.raises(ValueError):
        hx.interpolate_to_gl(np.zeros((5, 5, 5)), mat)       # wrong extent
    with pytest.raises(ValueError):
        hx.interpolate_to_gl(np.full((4, 4, 4), np.nan), mat)  # non-finite
    with pytest.raises(ValueError):
        hx.interpolate_to_gl(np.zeros((4, 4, 4)), np.full((5, 4), np.inf))  # non-finite matrix
    # any other finite matrix is accepted (dense passes), like contract_dim
    m = np.ones((5, 4)) + np.eye(5, 4)
    q = np.random.default_rng(0).standard_normal((4, 4, 4))
    np.testing.assert_allclose(hx.interpolate_to_gl(q, m), orc.interp_passes(m, q[None])[0],
                               rtol=0, atol=1e-12)


def test_measure_stream_bandwidth():
    """reference test_perf.py:149-161 on the device copy calibration."""
    cal = hx.measure_stream_bandwidth(1 << 22, trials=5)
    assert cal.mean_bandwidth > 0 and np.isfinite(cal.mean_bandwidth)
    assert len(cal.trial_times) == 5 and all(t > 0 for t in cal.trial_times)
    rates = [cal.bytes_transferred / t for t in cal.trial_times]
    assert min(rates) <= cal.mean_bandwidth <= max(rates)
    a = hx.measure_stream_bandwidth(1 << 22, trials=5).mean_bandwidth
    b = hx.measure_stream_bandwidth(1 << 23, trials=5).mean_bandwidth
    assert 0.3 < b / a < 3.0
    big = hx.measure_stream_bandwidth(1 << 30, trials=5)
    # one-way bytes / time: half the HBM traffic of the copy, below the peak
    assert 1e12 < big.mean_bandwidth < big.theoretical_peak


def test_contract_dim_on_device():
    mat = hx.interp_matrix(7)
    u = np.random.default_rng(0).standard_normal((8, 8, 8))
    for axis in range(3):
        got = hx.contract_dim(mat, torch.from_numpy(u).cuda(), axis)
        assert got.is_cuda
        np.testing.assert_allclose(got.cpu().numpy(), hx.contract_dim(mat, u, axis),
                                   rtol=0, atol=1e-13)
