"""GPU parity: the sm_100a kernels through the C ABI against the oracle, the
reference's golden vectors and the reference's known-answer properties.

Bar (north star): relative L2 <= 1e-12 in FP64 against the CPU reference on
identical inputs; the reference's own per-test tolerances where it states
one (test_operators.py, test_acceptance.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402
from oracle import hexbench_oracle as orc  # noqa: E402
from paper_1711_00903_b200 import _native  # noqa: E402

pytestmark = pytest.mark.gpu

BPS = (hx.BP1, hx.BP35, hx.BP3)
TAG = {hx.BP1: "bp1", hx.BP35: "bp35", hx.BP3: "bp3"}
PARITY = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert _native.lib().hx_device_ok() == 1, "not an sm_100 device"


def oracle_apply(op, q):
    interp = None if op.interp is None else op.interp.entries
    diff = None if op.diff is None else op.diff.entries
    return orc.apply(op.bp, op.degree, op.lam, interp, diff, op.factors.data, q)


def sub_mesh(mesh, n):
    return hx.HexMesh(n, mesh.vertices[:n], mesh.extent)


def dev_apply(op, q):
    qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    out = hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, qd))
    return out.data.cpu().numpy()


@pytest.fixture(scope="module")
def mesh3():
    return hx.perturb_mesh(hx.build_cube_mesh(3, 2.0), amplitude=0.15, seed=7)


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", range(1, 16))
def test_degree_sweep_matches_oracle(bp, deg, mesh3):
    """Every degree 1..15, ragged element counts (not multiples of the tile)."""
    rng = np.random.default_rng(deg)
    for n_el in (1, 13, 27):
        op = hx.make_operator(bp, deg, sub_mesh(mesh3, n_el), lam=0.7)
        q = rng.standard_normal((n_el, op.n_p))
        got = dev_apply(op, q)
        ref = oracle_apply(op, q)
        assert orc.rel_l2(got, ref) <= PARITY, (bp, deg, n_el, orc.rel_l2(got, ref))
        assert orc.rel_inf(got, ref) <= PARITY


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 2, 3, 4, 5, 6, 7, 8, 11, 15])
def test_golden_reference_vectors(bp, deg, golden):
    """Against outputs of the reference itself; for N<=4 with the reference's
    exact geometric factors uploaded, otherwise with device-generated ones."""
    key = f"{TAG[bp]}_N{deg}_"
    verts = golden[key + "vertices"]
    mesh = hx.HexMesh(verts.shape[0], verts, 2.0)
    q = golden[key + "q"]
    for lam in (0.0, 0.7):
        fac = golden[key + "factors"] if deg <= 4 else None
        op = hx.make_operator(bp, deg, mesh, lam=lam, factors=fac)
        got = dev_apply(op, q)
        ref = golden[key + f"out_lam{lam}"]
        assert orc.rel_l2(got, ref) <= PARITY, (bp, deg, lam, orc.rel_l2(got, ref))


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 2, 3, 4, 7, 15])
def test_device_geometric_factors(bp, deg, golden):
    key = f"{TAG[bp]}_N{deg}_"
    ref = golden[key + "factors"]
    verts = golden[key + "vertices"][: ref.shape[0]]
    op = hx.make_operator(bp, deg, hx.HexMesh(ref.shape[0], verts, 2.0))
    assert orc.rel_l2(op.factors.data, ref) <= 1e-14


@pytest.mark.parametrize("bp", BPS)
def test_host_path_bitwise_equals_device_path(bp, mesh3):
    """hx_apply_host (numpy in/out, chunked PCIe pipeline) == hx_apply."""
    op = hx.make_operator(bp, 7, mesh3, lam=1.0)
    q = np.random.default_rng(3).standard_normal((op.n_el, op.n_p))
    host = hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, q))
    assert isinstance(host.data, np.ndarray)
    np.testing.assert_array_equal(host.data, dev_apply(op, q))
    # force several chunks through the three-stream pipeline
    out = np.empty_like(q)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    hx.apply_host(op, q, out, flag, chunk_el=5)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out, host.data)


def test_host_pipeline_layout_and_stream_changes(mesh3):
    """hx_apply_host back to back on one workspace with changing chunk sizes
    (the slot layout changes under in-flight work) and changing streams:
    every result is bitwise the device apply."""
    op = hx.make_operator(hx.BP35, 7, mesh3, lam=1.0)
    rng = np.random.default_rng(11)
    qs = [torch.from_numpy(rng.standard_normal((op.n_el, op.n_p))).pin_memory()
          for _ in range(6)]
    outs = [torch.empty_like(q).pin_memory() for q in qs]
    nbytes = _native.lib().hx_apply_host_workspace(op.plan.handle, 9)
    work = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for i, (q, out) in enumerate(zip(qs, outs)):
        st = streams[i % 2]
        hx.apply_host(op, q.numpy(), out.numpy(), stream=st.cuda_stream,
                      chunk_el=(9, 4, 4, 2, 9, 5)[i], work=work)
    torch.cuda.synchronize()
    for q, out in zip(qs, outs):
        np.testing.assert_array_equal(out.numpy(), dev_apply(op, q.numpy()))


def test_mass_volume_known_answers():
    """test_operators.py:68-78, test_acceptance.py:227-240 (conservation)."""
    cube = hx.build_cube_mesh(1, 2.0)
    op = hx.make_operator(hx.BP1, 2, cube)
    assert abs(hx.apply_bp1(op, hx.FieldVector.constant(1, 27)).flat().sum() - 8.0) < 1e-12
    tiled = hx.build_cube_mesh(8, 2.0)
    op = hx.make_operator(hx.BP1, 1, tiled)
    assert abs(hx.apply_bp1(op, hx.FieldVector.constant(512, 8)).flat().sum() - 8.0) < 1e-10
    for side in (8, 16):
        m = hx.build_cube_mesh(side, 2.0)
        for bp in BPS:
            op = hx.make_operator(bp, 2, m, lam=1.0)
            total = hx.apply_operator(op, hx.FieldVector.constant(m.n_el, op.n_p),
                                      threads=4).flat().sum()
            assert abs(total - 8.0) <= 1e-10, (side, bp, total)


@pytest.mark.parametrize("bp", [hx.BP35, hx.BP3])
def test_constant_null_space(bp, perturbed_mesh2):
    for deg in range(1, 9):
        op = hx.make_operator(bp, deg, perturbed_mesh2, lam=0.0)
        out = hx.apply_operator(op, hx.FieldVector.constant(8, op.n_p))
        assert np.max(np.abs(out.flat())) < 1e-10, (bp, deg)


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 3, 6, 7])
def test_adjoint_symmetry_and_psd(bp, deg, perturbed_single, rng):
    """test_acceptance.py:80-111 (<Au,v> = <u,Av>), test_operators.py:201-206."""
    op = hx.make_operator(bp, deg, perturbed_single, lam=0.4)
    us = rng.standard_normal((100, op.n_p))
    vs = rng.standard_normal((100, op.n_p))
    au = np.stack([dev_apply(op, u[None]) [0] for u in us])
    av = np.stack([dev_apply(op, v[None])[0] for v in vs])
    lhs = np.einsum("pi,pi->p", au, vs)
    rhs = np.einsum("pi,pi->p", us, av)
    assert np.max(np.abs(lhs - rhs) / np.maximum(1.0, np.abs(lhs))) <= 1e-11
    assert np.min(np.einsum("pi,pi->p", au, us)) >= -1e-10


def test_back_to_back_applies_on_one_stream_bitwise(mesh3):
    """Device applies launch as programmatic dependent launches: a chain
    x_{k+1} = A_k x_k queued on one stream with no sync -- across operators,
    with a torch kernel rewriting the input in between -- must equal the
    same chain run one synchronised apply at a time, bit for bit (each
    kernel waits for its predecessor before touching q / out)."""
    ops = [hx.make_operator(bp, 7, mesh3, lam=1.0) for bp in BPS]
    x0 = torch.from_numpy(np.random.default_rng(9).standard_normal(
        (mesh3.n_el, ops[0].n_p))).cuda()

    def chain(sync):
        xs, x = [], x0
        for k in range(9):
            op = ops[k % 3]
            y = torch.empty_like(x)
            hx.apply_device(op, x, y)
            if k % 4 == 1:
                y.mul_(0.5)  # a foreign kernel between two applies
            if sync:
                torch.cuda.synchronize()
            xs.append(y)
            x = y
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in xs]

    for got, want in zip(chain(False), chain(True)):
        np.testing.assert_array_equal(got, want)


def test_element_permutation_bitwise(perturbed_mesh2, rng):
    """test_operators.py:208-220."""
    perm = rng.permutation(8)
    shuffled = hx.HexMesh(8, perturbed_mesh2.vertices[perm], perturbed_mesh2.extent)
    op = hx.make_operator(hx.BP3, 2, perturbed_mesh2, lam=0.5)
    op_p = hx.make_operator(hx.BP3, 2, shuffled, lam=0.5)
    q = rng.standard_normal((8, 27))
    np.testing.assert_array_equal(dev_apply(op, q)[perm], dev_apply(op_p, q[perm]))


@pytest.mark.parametrize("bp", BPS)
def test_partition_invariance_bitwise(bp, mesh3):
    """Sharded applies over the reference's linspace ranges reproduce the
    one-shot apply bit for bit (test_acceptance.py:210-224 analogue)."""
    from paper_1711_00903_b200.shard import ShardedOperator

    op = hx.make_operator(bp, 5, mesh3, lam=0.5)
    q = np.random.default_rng(9).standard_normal((27, op.n_p))
    full = dev_apply(op, q)
    for world in (2, 4, 8):
        parts = []
        for r in range(world):
            sh = ShardedOperator(bp, 5, mesh3, lam=0.5, rank=r, world_size=world)
            lo, hi = sh.range
            qd = torch.from_numpy(q[lo:hi].copy()).cuda()
            out = torch.empty_like(qd)
            sh.apply_device(qd, out)
            parts.append(out.cpu().numpy())
        np.testing.assert_array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("bp", BPS)
def test_unaligned_device_views(bp, mesh3):
    """q / out views that are only 8-byte aligned (the bulk-copy staging
    needs 16) still give the aligned result bit for bit."""
    op = hx.make_operator(bp, 7, mesh3, lam=0.7)
    q = np.random.default_rng(5).standard_normal((27, op.n_p))
    ref = dev_apply(op, q)
    buf = torch.empty(27 * op.n_p + 1, dtype=torch.float64, device="cuda")
    qd = buf[1:].view(27, op.n_p)
    qd.copy_(torch.from_numpy(q))
    obuf = torch.empty_like(buf)
    out = obuf[1:].view(27, op.n_p)
    hx.apply_device(op, qd, out)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)


def test_non_finite_input_raises(perturbed_single):
    op = hx.make_operator(hx.BP1, 1, perturbed_single)
    with pytest.raises(ValueError):
        hx.apply_operator(op, hx.FieldVector(1, 8, np.array([np.nan] + [0.0] * 7)))
    op = hx.make_operator(hx.BP3, 7, perturbed_single)
    bad = np.zeros((1, 512))
    bad[0, 511] = np.inf
    with pytest.raises(ValueError):
        hx.apply_operator(op, hx.FieldVector(1, 512, bad))
    op = hx.make_operator(hx.BP35, 4, perturbed_single)
    bad = torch.zeros((1, 125), dtype=torch.float64, device="cuda")
    bad[0, 60] = float("nan")
    with pytest.raises(ValueError):
        hx.apply_operator(op, hx.FieldVector(1, 125, bad))


@pytest.mark.parametrize("bp", BPS)
def test_non_finite_detected_in_every_position(bp, mesh3):
    """A single inf / nan anywhere -- any element of a ragged batch, any node,
    any chunk of the host pipeline -- sets the flag (operators.py:317-318);
    a clean batch never does."""
    op = hx.make_operator(bp, 3, mesh3, lam=0.5)
    rng = np.random.default_rng(21)
    q = rng.standard_normal((op.n_el, op.n_p))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    hx.apply_device(op, qd, out, flag)
    out_h = np.empty_like(q)
    hx.apply_host(op, q, out_h, flag, chunk_el=4)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    for e, node, val in ((0, 0, np.inf), (13, op.n_p // 2, np.nan), (op.n_el - 1, op.n_p - 1,
                                                                       -np.inf)):
        bad = q.copy()
        bad[e, node] = val
        for path in ("device", "host"):
            flag.zero_()
            if path == "device":
                hx.apply_device(op, torch.from_numpy(bad).cuda(), out, flag)
            else:
                hx.apply_host(op, bad, out_h, flag, chunk_el=4)
            torch.cuda.synchronize()
            assert int(flag.item()) & 1, (e, node, path)


def test_degenerate_geometry_raises():
    flat = hx.build_cube_mesh(1, 2.0).vertices.copy()
    flat[0, :, 2] = 0.0
    with pytest.raises(hx.DegenerateGeometryError):
        hx.make_operator(hx.BP3, 2, hx.HexMesh(1, flat, 2.0))


@pytest.mark.parametrize("bp", BPS)
def test_empty_mesh(bp):
    op = hx.make_operator(bp, 3, hx.HexMesh(0, np.zeros((0, 8, 3)), 2.0))
    out = hx.apply_operator(op, hx.FieldVector(0, 64, np.zeros(0)))
    assert out.data.shape == (0, 64)


def test_counters_charged(perturbed_mesh2):
    for bp in BPS:
        c = hx.AccessCounters()
        op = hx.make_operator(bp, 3, perturbed_mesh2, lam=0.1)
        hx.apply_operator(op, hx.FieldVector.constant(8, op.n_p), c)
        assert c.flops == 8 * hx.flop_model(bp, "fused", 3)
        assert c.global_reads + c.global_writes == 8 * hx.traffic(bp, 3).bytes_per_element


@pytest.mark.parametrize("bp", BPS)
def test_full_size_config_sampled_parity_and_symmetry(bp):
    """BASELINE configs at full size (N=7; E=4096 for BP1.0, 32768 otherwise):
    element-locality makes parity on a sampled element subset exact, and the
    global symmetry <Au, v> = <u, Av> covers every element."""
    side = 16 if bp == hx.BP1 else 32
    mesh = hx.perturb_mesh(hx.build_cube_mesh(side, 2.0), amplitude=0.15, seed=7)
    op = hx.make_operator(bp, 7, mesh, lam=1.0)
    u = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device()
    v = hx.FieldVector.random(mesh.n_el, op.n_p, seed=1).to_device()
    au = hx.apply_operator(op, u).data
    av = hx.apply_operator(op, v).data
    lhs = float(torch.dot(au.reshape(-1), v.data.reshape(-1)))
    rhs = float(torch.dot(u.data.reshape(-1), av.reshape(-1)))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs))
    idx = np.unique(np.linspace(0, mesh.n_el - 1, 300).astype(int))
    sub = hx.HexMesh(len(idx), mesh.vertices[idx], mesh.extent)
    op_s = hx.make_operator(bp, 7, sub, lam=1.0)
    ref = oracle_apply(op_s, u.data.cpu().numpy()[idx])
    got = au.cpu().numpy()[idx]
    assert orc.rel_l2(got, ref) <= PARITY
    # linearity at full size: A(2u - v) = 2Au - Av
    w = hx.FieldVector(mesh.n_el, op.n_p, 2 * u.data - v.data)
    aw = hx.apply_operator(op, w).data
    assert float((aw - (2 * au - av)).norm() / aw.norm()) <= 1e-14


def test_full_size_device_factors_match_reference_sample():
    """Device geometric factors of the whole E=32768 BASELINE mesh against
    the reference's geometric_factors (mesh.py:101-139) on 24 sampled
    elements (tests/golden/factors_e32768.npz, make_factor_sample.py), for
    the GLL(8) rule of BP3.5 and the GL(9) rule of BP1.0 / BP3.0."""
    import os
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "factors_e32768.npz"))
    idx = fx["elements"]
    mesh = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
    np.testing.assert_array_equal(mesh.vertices[idx], fx["vertices"])
    for bp, key in ((hx.BP35, "gll8"), (hx.BP3, "gl9"), (hx.BP1, "gl9")):
        op = hx.make_operator(bp, 7, mesh)
        q = 8 if bp == hx.BP35 else 9
        ref = fx[key].reshape(len(idx), 7, q ** 3)
        packed = op.device_factors.view(mesh.n_el, op.plan.elem_stride)[torch.from_numpy(idx)]
        got = packed.view(len(idx), op.plan.n_slots, op.plan.slot_stride)[:, :, :q ** 3]
        got = got.cpu().numpy()
        want = ref if op.plan.n_slots == 7 else ref[:, 6:7]
        if op.plan.n_slots == 1:  # BP1.0's GwJ slot is i-major: (k, j, i) at i*q^2 + k*q + j
            want = want.reshape(len(idx), 1, q, q, q).transpose(0, 1, 4, 2, 3).reshape(
                len(idx), 1, q ** 3)
        assert orc.rel_l2(got, want) <= 1e-14, (bp, orc.rel_l2(got, want))


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("deg", [1, 2, 4, 7, 8, 15])
def test_unfused_baseline_path_matches_oracle(bp, deg, mesh3):
    """apply_baseline (paper Kernel-1 structure, intermediates in HBM) gives
    the same operator as the fused kernels and the oracle."""
    rng = np.random.default_rng(100 + deg)
    for n_el in (1, 27):
        op = hx.make_operator(bp, deg, sub_mesh(mesh3, n_el), lam=0.7)
        q = rng.standard_normal((n_el, op.n_p))
        got = hx.apply_baseline(op, torch.from_numpy(q).cuda()).cpu().numpy()
        ref = oracle_apply(op, q)
        assert orc.rel_l2(got, ref) <= PARITY, (bp, deg, n_el, orc.rel_l2(got, ref))
        np.testing.assert_allclose(got, dev_apply(op, q), rtol=0,
                                   atol=1e-12 * max(1.0, np.abs(ref).max()))
    bad = torch.zeros((1, op.n_p), dtype=torch.float64, device="cuda")
    bad[0, 0] = float("inf")
    op1 = hx.make_operator(bp, deg, sub_mesh(mesh3, 1), lam=0.7)
    with pytest.raises(ValueError):
        hx.apply_baseline(op1, bad)


@pytest.mark.parametrize("bp", BPS)
def test_apply_range_over_partition_bitwise(bp, mesh3):
    """hx_apply_range over the reference chunking's ranges (operators.py:324)
    fills the full output bit for bit like one hx_apply."""
    from paper_1711_00903_b200.shard import partition

    op = hx.make_operator(bp, 7, mesh3, lam=0.3)
    q = torch.from_numpy(np.random.default_rng(4).standard_normal((27, op.n_p))).cuda()
    full = torch.empty_like(q)
    hx.apply_device(op, q, full)
    out = torch.full_like(q, float("nan"))
    L = _native.lib()
    for lo, hi in partition(27, 4):
        _native.check(L.hx_apply_range(op.plan.handle, _native.ptr(q),
                                       _native.ptr(op.device_factors), _native.ptr(out), lo, hi,
                                       None, None))
    np.testing.assert_array_equal(out.cpu().numpy(), full.cpu().numpy())
    assert L.hx_apply_range(op.plan.handle, _native.ptr(q), _native.ptr(op.device_factors),
                            _native.ptr(out), 5, 4, None, None) == _native.HX_EINVAL


def test_host_path_concurrent_threads_on_one_plan(mesh3):
    """Two host threads driving hx_apply_host on the same plan at once
    (ctypes drops the GIL): the shared pipeline is serialised per plan and
    both results are exact."""
    import threading

    op = hx.make_operator(hx.BP35, 5, mesh3, lam=0.5)
    qs = [np.random.default_rng(s).standard_normal((27, op.n_p)) for s in (1, 2)]
    want = [dev_apply(op, q) for q in qs]
    outs = [np.empty_like(q) for q in qs]
    errors = []

    def work(i):
        try:
            for _ in range(20):
                hx.apply_host(op, qs[i], outs[i], chunk_el=4)
                torch.cuda.synchronize()
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for got, ref in zip(outs, want):
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("bp,deg,n_el", [
    # q / out offsets e*n^3 and factor offsets e*elem_stride pass 2^31
    (hx.BP1, 15, 7 * 75_715),
    # factor offsets e*elem_stride pass 2^31 (elem_stride 3584 / 5110)
    (hx.BP35, 7, 7 * 87_000),
    (hx.BP3, 7, 7 * 61_000),
])
def test_64bit_offsets_periodic_mesh(bp, deg, n_el, mesh3):
    """Maximum-size edge case: element counts whose double offsets exceed
    2^31 (17-56 GB on the device).  The mesh and q repeat with period 7, so
    A q must repeat bitwise (element-locality, reference operators.py:300-302)
    and its first period must match the oracle; a non-finite value in the
    last element is still detected (operators.py:317-318)."""
    period = 7
    small = sub_mesh(mesh3, period)
    reps = n_el // period
    mesh = hx.HexMesh(n_el, np.tile(small.vertices, (reps, 1, 1)), small.extent)
    op = hx.make_operator(bp, deg, mesh, lam=0.7)
    assert max(n_el * op.n_p, n_el * op.plan.elem_stride) > 2 ** 31
    q7 = np.random.default_rng(deg).standard_normal((period, op.n_p))
    q = torch.from_numpy(q7).cuda().repeat(reps, 1)
    out = torch.empty_like(q)
    hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(reps, period, -1), out[:period].expand(reps, period, -1))
    ref = oracle_apply(hx.make_operator(bp, deg, small, lam=0.7), q7)
    assert orc.rel_l2(out[:period].cpu().numpy(), ref) <= PARITY
    del out
    q[-1, -1] = float("inf")
    with pytest.raises(ValueError):
        hx.apply_operator(op, hx.FieldVector(n_el, op.n_p, q))
    del q, op
    torch.cuda.empty_cache()
