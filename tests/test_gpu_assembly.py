"""GPU: gather-scatter (hx_dss) and the assembled CG solve
(cg_solve_assembled) against the oracle's Q Q^T, dense linear algebra and a
manufactured Poisson solution."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402
from oracle import hexbench_oracle as orc  # noqa: E402
from paper_1711_00903_b200 import _native  # noqa: E402
from paper_1711_00903_b200.cg import CGWorkspace, cg_solve_assembled, gather_scatter  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("side,deg", [(1, 3), (2, 1), (3, 2), (3, 4), (2, 7), (4, 3)])
@pytest.mark.parametrize("mask", [False, True])
def test_dss_matches_oracle_and_is_continuous(side, deg, mask):
    n3 = (deg + 1) ** 3
    u = np.random.default_rng(side * 10 + deg).standard_normal((side ** 3, n3))
    got = gather_scatter(torch.from_numpy(u).cuda(), side, deg, mask).cpu().numpy()
    ref = orc.dss(u, side, deg, mask)
    assert orc.rel_l2(got, ref) <= 1e-15
    # every copy of a global node holds the bit-identical sum
    gidx = orc.cube_global_index(side, deg).ravel()
    first = np.full(gidx.max() + 1, np.nan)
    first[gidx[::-1]] = got.ravel()[::-1]
    np.testing.assert_array_equal(first[gidx], got.ravel())


def test_dot_dss_is_global_inner_product():
    side, deg = 3, 3
    n3 = (deg + 1) ** 3
    rng = np.random.default_rng(1)
    # continuous representatives of two global vectors
    gidx = orc.cube_global_index(side, deg)
    ug, vg = rng.standard_normal((2, gidx.max() + 1))
    u, v = ug[gidx], vg[gidx]
    dev = [torch.from_numpy(a).cuda() for a in (u, v)]
    part = torch.empty(_native.lib().hx_energy_partials(), dtype=torch.float64, device="cuda")
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().hx_dot_dss(_native.ptr(dev[0]), _native.ptr(dev[1]), side, deg,
                                           0, side ** 3, _native.ptr(part), part.numel(),
                                           _native.ptr(res), None))
    assert abs(float(res) - float(ug @ vg)) <= 1e-12 * abs(float(ug @ vg))
    assert u.shape == (side ** 3, n3)


def _assembled_case(bp, side, deg, lam):
    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(bp, deg, mesh, lam=lam)
    b = np.random.default_rng(3).standard_normal((mesh.n_el, op.n_p))
    return mesh, op, b


@pytest.mark.parametrize("bp,lam,mask", [(hx.BP35, 0.0, True), (hx.BP3, 0.3, True),
                                         (hx.BP1, 0.0, False), (hx.BP35, 1.0, False)])
def test_assembled_cg_matches_oracle_cg(bp, lam, mask):
    side, deg = 3, 3
    mesh, op, b = _assembled_case(bp, side, deg, lam)
    res = cg_solve_assembled(op, side, torch.from_numpy(b).cuda(), tol=1e-12,
                             mask_boundary=mask)
    assert res.converged
    interp = None if op.interp is None else op.interp.entries
    diff = None if op.diff is None else op.diff.entries
    ref, _ = orc.assembled_cg(lambda p: orc.apply(bp, deg, lam, interp, diff, op.factors.data, p),
                       b, side, deg, mask, tol=1e-12)
    assert orc.rel_l2(res.x.cpu().numpy(), ref) <= 1e-9


def test_assembled_cg_matches_dense_solve():
    """BP3.5 Poisson, Dirichlet: x_G = A_G^{-1} b_G with A_G assembled densely
    from the oracle element operator (column g = Q^T A_L Q e_g)."""
    side, deg = 2, 3
    mesh, op, b = _assembled_case(hx.BP35, side, deg, 0.0)
    gidx = orc.cube_global_index(side, deg)
    ng = gidx.max() + 1
    diff = op.diff.entries
    fac = op.factors.data
    cols = np.zeros((ng, ng))
    for g in range(ng):
        ul = (gidx == g).astype(float)
        cols[:, g] = orc.scatter_add(orc.apply(hx.BP35, deg, 0.0, None, diff, fac, ul), gidx, ng)
    inner = ~orc.cube_boundary(side, deg)
    bg = orc.scatter_add(b, gidx, ng)
    xg = np.zeros(ng)
    xg[inner] = np.linalg.solve(cols[np.ix_(inner, inner)], bg[inner])
    res = cg_solve_assembled(op, side, torch.from_numpy(b).cuda(), tol=1e-13)
    assert orc.rel_l2(res.x.cpu().numpy(), xg[gidx]) <= 1e-10


def test_poisson_manufactured_solution_spectral_accuracy():
    """-lap u = f on [0,2]^3, u = prod sin(pi x / 2): BP3.5 stiffness, BP1.0
    load vector, assembled CG on the device -> max nodal error ~2e-10 at
    side 3, N = 7 (the oracle solve gives the same)."""
    side, deg = 3, 7
    mesh = hx.build_cube_mesh(side, 2.0)
    x = orc.node_coords(mesh.vertices, hx.gll_rule(deg + 1).nodes)
    u_ex = np.prod(np.sin(np.pi * x / 2), axis=-1)
    f = 3 * (np.pi / 2) ** 2 * u_ex
    mass = hx.make_operator(hx.BP1, deg, mesh)
    b = hx.apply_operator(mass, hx.FieldVector(mesh.n_el, mass.n_p, torch.from_numpy(f).cuda()))
    stiff = hx.make_operator(hx.BP35, deg, mesh, lam=0.0)
    res = cg_solve_assembled(stiff, side, b.data, tol=1e-13, work=CGWorkspace(b.data))
    assert res.converged and res.iterations < 300
    assert np.abs(res.x.cpu().numpy() - u_ex).max() < 1e-8


@pytest.mark.parametrize("world", [2, 3])
def test_dss_range_semantics_match_global(world):
    """Each rank's range [lo, hi) gathered from its padded halo buffer
    [base, top) reproduces the global gather-scatter bit for bit, and the
    ranks' weighted dots sum to the global one (multi-GPU kernels, driven
    here rank by rank on one device)."""
    from paper_1711_00903_b200.cg import AssembledShard

    side, deg = 5, 3
    n3 = (deg + 1) ** 3
    u = np.random.default_rng(11).standard_normal((side ** 3, n3))
    ud = torch.from_numpy(u).cuda()
    full = gather_scatter(ud, side, deg, True).cpu().numpy()
    L = _native.lib()
    part = torch.empty(L.hx_energy_partials(), dtype=torch.float64, device="cuda")
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    total = 0.0
    for r in range(world):
        sh = AssembledShard(side, deg, r, world)
        pad = ud[sh.base:sh.top].contiguous()
        got = gather_scatter(pad, side, deg, True, shard=sh).cpu().numpy()
        np.testing.assert_array_equal(got, full[sh.lo:sh.hi])
        own = ud[sh.lo:sh.hi].contiguous()
        _native.check(L.hx_dot_dss(_native.ptr(own), _native.ptr(own), side, deg, sh.lo, sh.hi,
                                   _native.ptr(part), part.numel(), _native.ptr(res), None))
        total += float(res)
    gidx = orc.cube_global_index(side, deg)
    ref = float(np.sum(u * u / orc.multiplicity(side, deg)))
    assert abs(total - ref) <= 1e-12 * ref


@pytest.mark.parametrize("side,deg", [(1, 2), (3, 3), (4, 7)])
def test_inplace_separable_dss_matches_oracle(side, deg):
    """hx_dss_inplace (three face passes) == the oracle's pass form bit for
    bit, == Q Q^T to rounding; a rank's halo-padded buffer reproduces the
    full result on its own elements exactly."""
    from paper_1711_00903_b200.cg import AssembledShard

    n3 = (deg + 1) ** 3
    u = np.random.default_rng(side * 7 + deg).standard_normal((side ** 3, n3))
    L = _native.lib()
    ud = torch.from_numpy(u).cuda()
    _native.check(L.hx_dss_inplace(_native.ptr(ud), side, deg, 0, side ** 3, None))
    got = ud.cpu().numpy()
    np.testing.assert_array_equal(got, orc.dss_passes(u, side, deg))
    assert orc.rel_l2(got, orc.dss(u, side, deg)) <= 1e-15
    if side ** 3 >= 2 * (side * side + side + 1):
        for r in range(2):
            sh = AssembledShard(side, deg, r, 2)
            pad = torch.from_numpy(u[sh.base:sh.top].copy()).cuda()
            _native.check(L.hx_dss_inplace(_native.ptr(pad), side, deg, sh.base, sh.top, None))
            np.testing.assert_array_equal(sh.own(pad).cpu().numpy(), got[sh.lo:sh.hi])


@pytest.mark.parametrize("world", [1, 2])
def test_cg_update_assembled_kernel(world):
    """hx_cg_update_assembled on each rank's range (y/z passes in place on the
    halo buffer, x pass fused): x += a p, r -= a mask QQ^T ap, <r,r>_w."""
    from paper_1711_00903_b200.cg import AssembledShard

    side, deg = 4, 3
    n3 = (deg + 1) ** 3
    rng = np.random.default_rng(21)
    E = side ** 3
    x, p, r, ap = rng.standard_normal((4, E, n3))
    rr, pap = 2.5, 1.25
    alpha = rr / pap
    w_ref = orc.dss(ap, side, deg, mask=True)
    x_ref = x + alpha * p
    r_ref = r - alpha * w_ref
    L = _native.lib()
    part = torch.empty(L.hx_energy_partials(), dtype=torch.float64, device="cuda")
    total = 0.0
    for rank in range(world):
        sh = AssembledShard(side, deg, rank, world)
        dev = {k: torch.from_numpy(v[sh.lo:sh.hi].copy()).cuda()
               for k, v in (("x", x), ("p", p), ("r", r))}
        ap_pad = torch.from_numpy(ap[sh.base:sh.top].copy()).cuda()
        rrd = torch.tensor([rr], dtype=torch.float64, device="cuda")
        papd = torch.tensor([pap], dtype=torch.float64, device="cuda")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        _native.check(L.hx_cg_update_assembled(
            _native.ptr(dev["x"]), _native.ptr(dev["p"]), _native.ptr(dev["r"]),
            _native.ptr(ap_pad), side, deg, 1, sh.lo, sh.hi, sh.base, sh.top, _native.ptr(rrd),
            _native.ptr(papd), _native.ptr(part), part.numel(), _native.ptr(out), None))
        np.testing.assert_allclose(dev["x"].cpu().numpy(), x_ref[sh.lo:sh.hi], rtol=0,
                                   atol=1e-14)
        np.testing.assert_allclose(dev["r"].cpu().numpy(), r_ref[sh.lo:sh.hi], rtol=1e-13,
                                   atol=1e-13)
        total += float(out)
    want = float(np.sum(r_ref ** 2 / orc.multiplicity(side, deg)))
    assert abs(total - want) <= 1e-12 * want


def test_dss_argument_errors():
    u = torch.zeros(8 * 27, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        gather_scatter(u, 3, 2)            # wrong size for the mesh
    with pytest.raises(ValueError):
        gather_scatter(u, 2, 2, out=u)     # in-place is rejected


def _sharded_cg_worker(rank, world, port, result_path):
    import os
    import torch.distributed as dist

    from paper_1711_00903_b200.cg import AssembledShard
    from paper_1711_00903_b200.shard import ShardedOperator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)  # both ranks share the one GPU (gloo moves the scalars/halos)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        side, deg = 4, 3
        mesh = hx.build_cube_mesh(side, 2.0)
        sh = AssembledShard(side, deg, rank, world)
        op = ShardedOperator(hx.BP35, deg, mesh, lam=0.0, rank=rank, world_size=world).op
        b = np.random.default_rng(3).standard_normal((side ** 3, (deg + 1) ** 3))
        res = cg_solve_assembled(op, side, torch.from_numpy(b[sh.lo:sh.hi].copy()).cuda(),
                                 tol=1e-12, shard=sh)
        np.save(f"{result_path}.{rank}.npy", res.x.cpu().numpy())
        np.save(f"{result_path}.{rank}.it.npy", np.array([res.iterations, res.converged]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_assembled_cg_two_ranks_on_one_gpu(tmp_path):
    """The multi-GPU assembled CG end to end -- kernels over element ranges,
    halo exchange, all-reduced scalars -- as two ranks sharing the GPU (gloo
    carries the exchange here, NCCL on a multi-GPU node): the gathered
    solution equals the one-rank solve."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    base = str(tmp_path / "x")
    mp.spawn(_sharded_cg_worker, args=(2, port, base), nprocs=2, join=True)
    x2 = np.concatenate([np.load(f"{base}.{r}.npy") for r in range(2)])
    its = [np.load(f"{base}.{r}.it.npy") for r in range(2)]
    side, deg = 4, 3
    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(hx.BP35, deg, mesh, lam=0.0)
    b = np.random.default_rng(3).standard_normal((side ** 3, (deg + 1) ** 3))
    ref = cg_solve_assembled(op, side, torch.from_numpy(b).cuda(), tol=1e-12)
    assert all(bool(i[1]) for i in its) and its[0][0] == its[1][0]
    assert orc.rel_l2(x2, ref.x.cpu().numpy()) <= 1e-10


def test_graphed_assembled_cg_is_bitwise_the_eager_one():
    """graph=True replays the captured iteration blocks: same iterates bit for
    bit as the eager loop (same kernels, same order, deterministic sums)."""
    side, deg = 3, 4
    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(hx.BP35, deg, mesh, lam=0.0)
    b = torch.from_numpy(np.random.default_rng(8).standard_normal((mesh.n_el, op.n_p))).cuda()
    eager = cg_solve_assembled(op, side, b, tol=1e-11, check_every=10)
    graphed = cg_solve_assembled(op, side, b, tol=1e-11, check_every=10, graph=True)
    assert eager.converged and graphed.converged
    assert graphed.iterations == -(-eager.iterations // 10) * 10
    # the eager solve stopped at its check; the graphed one at the same check
    np.testing.assert_array_equal(graphed.x.cpu().numpy(), eager.x.cpu().numpy())


@pytest.mark.parametrize("bp", [hx.BP1, hx.BP35, hx.BP3])
def test_assembled_cg_fused_direction_bitwise(bp):
    """The direction update fused into the matvec (hx_apply_energy_dir) gives
    the unfused assembled iterates bit for bit, eager and graphed."""
    side, deg = 3, 5
    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(bp, deg, mesh, lam=0.0 if bp != hx.BP1 else 1.0)
    b = torch.from_numpy(np.random.default_rng(5).standard_normal((mesh.n_el, op.n_p))).cuda()
    fused = cg_solve_assembled(op, side, b, tol=1e-11, check_every=10)
    plain = cg_solve_assembled(op, side, b, tol=1e-11, check_every=10, fuse_direction=False)
    assert fused.converged and fused.iterations == plain.iterations
    np.testing.assert_array_equal(fused.x.cpu().numpy(), plain.x.cpu().numpy())
    graphed = cg_solve_assembled(op, side, b, tol=1e-11, check_every=10, graph=True)
    np.testing.assert_array_equal(graphed.x.cpu().numpy(), fused.x.cpu().numpy())
