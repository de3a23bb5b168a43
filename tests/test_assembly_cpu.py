"""CPU: the assembly checker (oracle cube_global_index / dss) that the GPU
gather-scatter is tested against.  The reference has no assembly, so the
numbering is pinned to the reference's mesh geometry instead: element-local
GLL nodes with the same global id must map to the same physical point under
the reference trilinear map (mesh.py:93-98) of build_cube_mesh (mesh.py:44-56),
and a CG solve on the oracle operators must converge to a manufactured
Poisson solution at the spectral rate."""

import numpy as np
import pytest

import paper_1711_00903_b200 as hx
from oracle import hexbench_oracle as orc
from paper_1711_00903_b200 import basis
from paper_1711_00903_b200 import mesh as pm


def node_coords(mesh, degree):
    return orc.node_coords(mesh.vertices, hx.gll_rule(degree + 1).nodes)


@pytest.mark.parametrize("side,deg", [(1, 2), (2, 1), (2, 3), (3, 2)])
def test_global_numbering_matches_mesh_geometry(side, deg):
    mesh = hx.build_cube_mesh(side, 2.0)
    x = node_coords(mesh, deg)
    # the batched map agrees with the product's per-point trilinear_map
    r = hx.gll_rule(deg + 1).nodes
    e = mesh.n_el - 1
    np.testing.assert_allclose(x[e, -1], pm.trilinear_map(mesh.vertices[e], r[-1], r[-1], r[-1]),
                               rtol=0, atol=1e-14)
    np.testing.assert_allclose(x[e, 1], pm.trilinear_map(mesh.vertices[e], r[1], r[0], r[0]),
                               rtol=0, atol=1e-14)
    gidx = orc.cube_global_index(side, deg)
    ng = (side * deg + 1) ** 3
    assert np.array_equal(np.unique(gidx), np.arange(ng))
    first = np.zeros((ng, 3))
    first[gidx.ravel()] = x.reshape(-1, 3)
    np.testing.assert_allclose(first[gidx], x, rtol=0, atol=1e-14)
    # distinct ids are distinct points
    pts = np.round(first, 12)
    assert len(np.unique(pts, axis=0)) == ng


def test_dss_identities():
    rng = np.random.default_rng(0)
    side, deg = 2, 3
    u = rng.standard_normal((8, 64))
    v = rng.standard_normal((8, 64))
    mult = orc.multiplicity(side, deg)
    np.testing.assert_array_equal(orc.dss(np.ones((8, 64)), side, deg), mult)
    # Q Q^T is symmetric; the masked version too
    for mask in (False, True):
        lhs = np.sum(orc.dss(u, side, deg, mask) * v)
        rhs = np.sum(u * orc.dss(v, side, deg, mask))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert set(np.unique(mult)) == {1, 2, 4, 8}


def test_oracle_assembled_poisson_manufactured_solution():
    """-lap u = f on [0,2]^3, u = prod sin(pi x / 2), u = 0 on the boundary:
    BP3.5 stiffness + BP1.0 load vector, assembled CG -> spectral accuracy."""
    side, deg = 2, 5
    n = deg + 1
    mesh = hx.build_cube_mesh(side, 2.0)
    x = node_coords(mesh, deg)
    u_ex = np.prod(np.sin(np.pi * x / 2), axis=-1)
    f = 3 * (np.pi / 2) ** 2 * u_ex
    f35 = pm.geometric_factors(mesh, hx.gll_rule(n)).data
    f1 = pm.geometric_factors(mesh, hx.gl_rule(n + 1)).data
    interp = basis.interp_matrix(deg).entries
    diff = basis.diff_matrix_gll(deg).entries
    b = orc.apply(orc.BP1, deg, 0.0, interp, None, f1, f)
    sol, its = orc.assembled_cg(lambda p: orc.apply(orc.BP35, deg, 0.0, None, diff, f35, p),
                         b, side, deg, True)
    assert its < 200
    assert np.abs(sol - u_ex).max() < 1e-5


@pytest.mark.parametrize("side,deg", [(1, 2), (2, 1), (3, 2), (2, 4)])
def test_separable_passes_equal_gather_scatter(side, deg):
    """Q Q^T = (x pass)(y pass)(z pass): the separable form the device uses
    per CG iteration equals the gather form, and leaves every copy of a node
    bit-identical."""
    u = np.random.default_rng(side + deg).standard_normal((side ** 3, (deg + 1) ** 3))
    got = orc.dss_passes(u, side, deg)
    np.testing.assert_allclose(got, orc.dss(u, side, deg), rtol=1e-14, atol=1e-14)
    gidx = orc.cube_global_index(side, deg).ravel()
    first = np.full(gidx.max() + 1, np.nan)
    first[gidx[::-1]] = got.ravel()[::-1]
    np.testing.assert_array_equal(first[gidx], got.ravel())
