"""CPU, world_size 2 over gloo: the element partition, the gathered result and
the CG-style all-reduced dot of the multi-GPU path (paper_1711_00903_b200/shard.py).
The per-rank apply is stood in for by the oracle (test-only), so the test
covers the host-side sharding logic without a GPU."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1711_00903_b200 import shard  # noqa: E402


def test_partition_matches_reference_chunking():
    for n_el in (0, 1, 7, 27, 32768):
        for world in (1, 2, 3, 4, 8):
            parts = shard.partition(n_el, world)
            b = np.linspace(0, n_el, world + 1).astype(int)  # operators.py:324
            assert parts == list(zip(b[:-1].tolist(), b[1:].tolist()))
            assert parts[0][0] == 0 and parts[-1][1] == n_el
    with pytest.raises(ValueError):
        shard.partition(8, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import hexbench_oracle as orc
        from paper_1711_00903_b200 import basis, mesh as pm, quadrature

        mesh = pm.perturb_mesh(pm.build_cube_mesh(3, 2.0), seed=7)
        local, (lo, hi) = shard.shard_mesh(mesh, rank, world)
        deg = 3
        fac = pm.geometric_factors(local, quadrature.gll_rule(deg + 1)).data
        q_all = np.random.default_rng(0).standard_normal((mesh.n_el, (deg + 1) ** 3))
        out = orc.apply("BP3.5", deg, 0.5, None, basis.diff_matrix_gll(deg).entries, fac,
                        q_all[lo:hi])
        out_t = torch.from_numpy(out)
        full = shard.gather_field(out_t, mesh.n_el, world)
        dot = shard.global_dot(torch.from_numpy(q_all[lo:hi].copy()), out_t)
        if rank == 0:
            np.savez(result_path, full=full.numpy(), dot=dot.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_dot(tmp_path):
    from oracle import hexbench_oracle as orc
    from paper_1711_00903_b200 import basis, mesh as pm, quadrature

    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    res = np.load(path)
    mesh = pm.perturb_mesh(pm.build_cube_mesh(3, 2.0), seed=7)
    fac = pm.geometric_factors(mesh, quadrature.gll_rule(4)).data
    q = np.random.default_rng(0).standard_normal((27, 64))
    ref = orc.apply("BP3.5", 3, 0.5, None, basis.diff_matrix_gll(3).entries, fac, q)
    # element-local operator: sharded and gathered == one shot, bit for bit
    np.testing.assert_array_equal(res["full"], ref)
    assert abs(float(res["dot"][0]) - float(np.sum(q * ref))) <= 1e-12 * abs(float(np.sum(q * ref)))


def _halo_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import hexbench_oracle as orc
        from paper_1711_00903_b200.cg import AssembledShard

        side, deg = 4, 2
        n3 = (deg + 1) ** 3
        u = np.random.default_rng(5).standard_normal((side ** 3, n3))
        sh = AssembledShard(side, deg, rank, world)
        pad = sh.padded(torch.zeros(1, n3, dtype=torch.float64))
        sh.own(pad).copy_(torch.from_numpy(u[sh.lo:sh.hi]))
        sh.exchange(pad)
        # halo rows now hold the neighbours' data exactly
        np.testing.assert_array_equal(pad.numpy(), u[sh.base:sh.top])
        got = orc.dss_range(pad.numpy(), side, deg, sh.lo, sh.hi, sh.base, mask=True)
        want = orc.dss(u, side, deg, mask=True)[sh.lo:sh.hi]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-14)
        dist.barrier()
        if rank == 0:
            np.save(result_path, np.array([1.0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_assembled_halo_exchange_gloo(world, tmp_path):
    """Multi-GPU assembled CG host logic: each rank's halo (side^2 + side + 1
    elements either side, from its direct neighbours) holds every copy of
    every node of its own elements, so the rank-local gather-scatter equals
    the global one on the rank's range."""
    res = str(tmp_path / "ok.npy")
    mp.spawn(_halo_worker, args=(world, _free_port(), res), nprocs=world, join=True)
    assert np.load(res)[0] == 1.0


def test_assembled_shard_ranges():
    from paper_1711_00903_b200.cg import AssembledShard

    side = 8
    for world in (1, 2, 4):
        shards = [AssembledShard(side, 3, r, world) for r in range(world)]
        assert shards[0].lo == 0 and shards[-1].hi == side ** 3
        for a, b in zip(shards, shards[1:]):
            assert a.hi == b.lo
            assert a.top - a.hi == min(a.halo, side ** 3 - a.hi)
    with pytest.raises(ValueError):
        AssembledShard(4, 3, 0, 8)   # 8 elements per rank < 4^2 + 4 + 1
