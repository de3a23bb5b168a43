"""GPU: the fused <q, A q> matvec, the CG vector kernels and the CG driver
(paper_1711_00903_b200/cg.py), checked against the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402
from oracle import hexbench_oracle as orc  # noqa: E402
from paper_1711_00903_b200 import _native  # noqa: E402
from paper_1711_00903_b200.cg import CGWorkspace, cg_iterations, cg_solve  # noqa: E402

pytestmark = pytest.mark.gpu

BPS = (hx.BP1, hx.BP35, hx.BP3)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def mesh3():
    return hx.perturb_mesh(hx.build_cube_mesh(3, 2.0), amplitude=0.15, seed=7)


def oracle_apply(op, q):
    return orc.apply(op.bp, op.degree, op.lam, None if op.interp is None else op.interp.entries,
                     None if op.diff is None else op.diff.entries, op.factors.data, q)


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 3, 7, 12])
def test_fused_energy_matches_dot(bp, deg, mesh3):
    op = hx.make_operator(bp, deg, mesh3, lam=0.8)
    q = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    out = torch.empty_like(q)
    ref = torch.empty_like(q)
    hx.apply_device(op, q, ref)
    L = _native.lib()
    npart = L.hx_energy_partials()
    part = torch.empty(npart, dtype=torch.float64, device="cuda")
    en = torch.zeros(1, dtype=torch.float64, device="cuda")
    _native.check(L.hx_apply_energy(op.plan.handle, q.data_ptr(), op.device_factors.data_ptr(),
                                    out.data_ptr(), op.n_el, part.data_ptr(), npart,
                                    en.data_ptr(), None, None))
    torch.cuda.synchronize()
    # the matvec output of the energy instantiation is the plain matvec
    assert float((out - ref).abs().max()) <= 1e-15 * float(ref.abs().max())
    dot = float(torch.dot(q.reshape(-1), ref.reshape(-1)))
    assert abs(float(en.item()) - dot) <= 1e-12 * abs(dot)
    np.testing.assert_allclose(out.cpu().numpy(), oracle_apply(op, q.cpu().numpy()),
                               rtol=0, atol=1e-12 * float(ref.abs().max()))


def test_dot_kernel():
    L = _native.lib()
    npart = L.hx_energy_partials()
    part = torch.empty(npart, dtype=torch.float64, device="cuda")
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    for n in (0, 1, 1000, 3_000_001):
        u = torch.randn(n, dtype=torch.float64, device="cuda")
        v = torch.randn(n, dtype=torch.float64, device="cuda")
        _native.check(L.hx_dot(u.data_ptr(), v.data_ptr(), n, part.data_ptr(), npart,
                               res.data_ptr(), None))
        ref = float(torch.dot(u, v)) if n else 0.0
        assert abs(float(res.item()) - ref) <= 1e-12 * max(1.0, abs(ref))


@pytest.mark.parametrize("bp", BPS)
def test_cg_solves_block_diagonal_system(bp, mesh3):
    """A x = b for the SPD (lam > 0) operator; residual checked with the oracle."""
    op = hx.make_operator(bp, 3, mesh3, lam=1.0)
    b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda",
                    generator=torch.Generator("cuda").manual_seed(0))
    res = cg_solve(op, b, tol=1e-11, maxiter=2000, check_every=5)
    assert res.converged, res.residual_norms[-3:]
    x = res.x.cpu().numpy()
    bn = b.cpu().numpy()
    r = bn - oracle_apply(op, x)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(bn)


def test_cg_bitwise_reproducible(mesh3):
    op = hx.make_operator(hx.BP35, 5, mesh3, lam=0.5)
    b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    w = CGWorkspace(b)
    x1 = cg_iterations(op, b, 25, w)
    x2 = cg_iterations(op, b, 25, w)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)


def test_report_bench_schema():
    """Reporting integration: the reference's `hexbench bench` run keys
    (cli.py:262-284) filled from device timings."""
    from paper_1711_00903_b200.report import bench_runs

    runs = bench_runs([hx.BP1, hx.BP35], [2], 3, repeats=3)
    ref_keys = {"bp", "degree", "variant", "elements", "wall_time_mean_s", "wall_time_median_s",
                "achieved_flops_per_s", "flops", "counted_global_bytes",
                "counted_scratch_bytes", "model_bytes", "syncs", "bandwidth_bytes_per_s",
                "r_global_flops_per_s"}
    for r in runs:
        assert ref_keys <= set(r)
        assert r["counted_global_bytes"] == r["model_bytes"]
        assert r["wall_time_median_s"] > 0 and r["gdof_per_s"] > 0
    assert "r_shared_flops_per_s" in runs[0] and "r_shared_flops_per_s" not in runs[1]


def test_report_cli_json_and_csv(tmp_path):
    """`python -m paper_1711_00903_b200.report {bench,roofline}` (the reference
    cli.py:235-347 commands) write the JSON / CSV schemas."""
    import csv
    import json

    from paper_1711_00903_b200.report import main

    out = tmp_path / "bench.json"
    assert main(["bench", "--bp", "3.5", "--degrees", "2", "--elements", "2", "--repeats", "2",
                 "--out", str(out)]) == 0
    payload = json.loads(out.read_text())
    assert payload["command"] == "bench" and len(payload["runs"]) == 1
    assert payload["runs"][0]["bp"] == hx.BP35
    out = tmp_path / "roof.csv"
    assert main(["roofline", "--bp", "1.0", "--degrees", "1..3", "--elements", "2",
                 "--bandwidth", "6000", "--format", "csv", "--out", str(out)]) == 0
    rows = list(csv.reader(out.open()))
    assert rows[0] == ["bp", "N", "F", "bytes", "R_global", "R_shared"]
    assert [int(r[1]) for r in rows[1:]] == [1, 2, 3]
    assert all(float(r[4]) > 0 and float(r[5]) > 0 for r in rows[1:])
    out = tmp_path / "cal.json"
    assert main(["calibrate", "--bytes", str(1 << 24), "--repeats", "4", "--out", str(out)]) == 0
    payload = json.loads(out.read_text())  # cli.py:356-363
    assert payload["command"] == "calibrate" and payload["bytes"] == 1 << 24
    assert len(payload["trial_times_s"]) == 4 and payload["mean_bytes_per_s"] > 0
    assert main(["calibrate", "--bytes", "100"]) == 2


def test_graphed_element_local_cg_bitwise(mesh3):
    from paper_1711_00903_b200.cg import cg_solve

    op = hx.make_operator(hx.BP3, 4, mesh3, lam=0.8)
    b = torch.from_numpy(np.random.default_rng(6).standard_normal((27, op.n_p))).cuda()
    eager = cg_solve(op, b, tol=1e-11, check_every=10)
    graphed = cg_solve(op, b, tol=1e-11, check_every=10, graph=True)
    assert eager.converged and graphed.converged and graphed.iterations == eager.iterations
    np.testing.assert_array_equal(graphed.x.cpu().numpy(), eager.x.cpu().numpy())


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 2, 7, 10, 13])
def test_apply_energy_dir_matches_unfused(bp, deg, mesh3):
    """hx_apply_energy_dir == hx_cg_direction then hx_apply_energy, bit for bit
    (p, A p and <p, A p>), on a mesh of more tiles than one CTA covers."""
    mesh = hx.perturb_mesh(hx.build_cube_mesh(5 if deg < 10 else 3, 2.0), 0.1, seed=deg)
    op = hx.make_operator(bp, deg, mesh, lam=0.7)
    g = torch.Generator("cuda").manual_seed(deg)
    shape = (op.n_el, op.n_p)
    p0 = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    r = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    rr = torch.tensor([1.7, 0.3], dtype=torch.float64, device="cuda")
    L = _native.lib()
    npart = L.hx_energy_partials()
    part = torch.empty(npart, dtype=torch.float64, device="cuda")
    outs = []
    for fused in (False, True):
        p = p0.clone()
        ap = torch.full_like(p, float("nan"))
        en = torch.zeros(1, dtype=torch.float64, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        if fused:
            _native.check(L.hx_apply_energy_dir(
                op.plan.handle, p.data_ptr(), r.data_ptr(), rr[0:1].data_ptr(),
                rr[1:2].data_ptr(), op.device_factors.data_ptr(), ap.data_ptr(), op.n_el,
                part.data_ptr(), npart, en.data_ptr(), flag.data_ptr(), None))
        else:
            _native.check(L.hx_cg_direction(p.data_ptr(), r.data_ptr(), p.numel(),
                                            rr[0:1].data_ptr(), rr[1:2].data_ptr(), None))
            _native.check(L.hx_apply_energy(op.plan.handle, p.data_ptr(),
                                            op.device_factors.data_ptr(), ap.data_ptr(),
                                            op.n_el, part.data_ptr(), npart, en.data_ptr(),
                                            flag.data_ptr(), None))
        torch.cuda.synchronize()
        assert int(flag.item()) == 0
        outs.append((p, ap, en))
    (pu, apu, enu), (pf, apf, enf) = outs
    assert torch.equal(pf, pu) and torch.equal(apf, apu) and torch.equal(enf, enu)
    beta = 1.7 / 0.3
    torch.testing.assert_close(pf, r + beta * p0, rtol=1e-15, atol=1e-15)


def test_apply_energy_dir_rejects_aliasing(mesh3):
    op = hx.make_operator(hx.BP35, 3, mesh3)
    L = _native.lib()
    npart = L.hx_energy_partials()
    part = torch.empty(npart, dtype=torch.float64, device="cuda")
    v = torch.zeros(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    u = torch.zeros_like(v)
    s = torch.ones(2, dtype=torch.float64, device="cuda")
    f = op.device_factors.data_ptr()

    def call(p, r, out, n=op.n_el, rr=s.data_ptr()):
        return L.hx_apply_energy_dir(op.plan.handle, p, r, rr, rr, f, out, n, part.data_ptr(),
                                     npart, s.data_ptr(), None, None)

    e = _native.HX_EINVAL
    assert call(v.data_ptr(), v.data_ptr(), u.data_ptr()) == e  # p == r
    assert call(v.data_ptr(), u.data_ptr(), v.data_ptr()) == e  # out == p
    assert call(v.data_ptr(), u.data_ptr(), u.data_ptr()) == e  # out == r
    assert call(v.data_ptr(), u.data_ptr(), part.data_ptr(), rr=None) == e
    assert call(None, None, None, n=0) == _native.HX_OK


@pytest.mark.parametrize("bp", BPS)
def test_cg_fused_direction_bitwise(bp, mesh3):
    """The fused iteration produces the unfused iterates bit for bit."""
    op = hx.make_operator(bp, 4, mesh3, lam=0.9)
    b = torch.from_numpy(np.random.default_rng(11).standard_normal((27, op.n_p))).cuda()
    w = CGWorkspace(b)
    xf = cg_iterations(op, b, 17, w).clone()
    xu = cg_iterations(op, b, 17, w, fuse_direction=False)
    torch.cuda.synchronize()
    assert torch.equal(xf, xu)
    a = cg_solve(op, b, tol=1e-11, check_every=5)
    u = cg_solve(op, b, tol=1e-11, check_every=5, fuse_direction=False)
    assert a.converged and a.iterations == u.iterations
    np.testing.assert_array_equal(a.x.cpu().numpy(), u.x.cpu().numpy())
