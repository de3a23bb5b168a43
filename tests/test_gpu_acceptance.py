"""GPU: the reference's output-side acceptance criteria (SPEC.md:523-534,
tests/test_acceptance.py) re-run against the sm_100a kernels with the
reference's own meshes, loops and tolerances.  C1 (dense-oracle equivalence)
is covered transitively by tests/test_gpu_parity.py::test_golden_reference_vectors
(the reference outputs it compares against met C1 when generated)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def mesh1():
    """test_acceptance.py:35-37: one perturbed element."""
    return hx.perturb_mesh(hx.build_cube_mesh(1, 2.0), seed=11)


def variants_for(bp):
    return ("baseline", "fused") if bp == hx.BP35 else ("baseline", "fused", "symfused")


def _replicate(mesh1, count):
    return hx.HexMesh(count, np.repeat(mesh1.vertices, count, axis=0), mesh1.extent)


def test_criterion_03_null_space_and_symmetry(mesh1):
    """test_acceptance.py:80-111: constants annihilated at lam=0 (<=1e-10);
    <Au, v> = <u, Av> over 100 random pairs, lam=0.4, N=1..8 (<=1e-11).  The
    100 pairs run as one 100-element apply of the same element."""
    rng = np.random.default_rng(9)
    worst_null = worst_sym = 0.0
    for bp in (hx.BP35, hx.BP3):
        for variant in variants_for(bp):
            for deg in range(1, 9):
                op0 = hx.make_operator(bp, deg, mesh1, lam=0.0, variant=variant)
                ones = hx.FieldVector.constant(1, op0.n_p)
                worst_null = max(worst_null,
                                 float(np.max(np.abs(hx.apply_operator(op0, ones).flat()))))
    many = _replicate(mesh1, 100)
    for bp in hx.BENCHMARKS:
        for variant in variants_for(bp):
            for deg in range(1, 9):
                op = hx.make_operator(bp, deg, many, lam=0.4, variant=variant)
                us = rng.standard_normal((100, op.n_p))
                vs = rng.standard_normal((100, op.n_p))
                au = hx.apply_operator(op, hx.FieldVector(100, op.n_p, us)).data
                av = hx.apply_operator(op, hx.FieldVector(100, op.n_p, vs)).data
                lhs = np.einsum("pi,pi->p", au, vs)
                rhs = np.einsum("pi,pi->p", us, av)
                rel = np.max(np.abs(lhs - rhs) / np.maximum(1.0, np.abs(lhs)))
                worst_sym = max(worst_sym, float(rel))
    assert worst_null <= 1e-10, worst_null
    assert worst_sym <= 1e-11, worst_sym


def test_criterion_09_thread_invariance():
    """test_acceptance.py:210-224: outputs and counters independent of
    `threads`, bit for bit."""
    mesh = hx.build_cube_mesh(3, 2.0)
    rng = np.random.default_rng(5)
    for bp in hx.BENCHMARKS:
        op = hx.make_operator(bp, 3, mesh, lam=0.5)
        q = hx.FieldVector(27, op.n_p, rng.standard_normal(27 * op.n_p))
        c1, c8 = hx.AccessCounters(), hx.AccessCounters()
        out1 = hx.apply_operator(op, q, c1, threads=1)
        out8 = hx.apply_operator(op, q, c8, threads=8)
        assert c1 == c8, bp
        np.testing.assert_array_equal(out1.data, out8.data)


def test_criterion_10_conservation():
    """test_acceptance.py:227-240: the constant field's action integrates to
    the mesh volume (8) within 1e-10 on 8^3 and 16^3 meshes, N=2, lam=1."""
    worst = 0.0
    for side in (8, 16):
        mesh = hx.build_cube_mesh(side, 2.0)
        volume = mesh.extent ** 3
        for bp in hx.BENCHMARKS:
            op = hx.make_operator(bp, 2, mesh, lam=1.0)
            ones = hx.FieldVector.constant(mesh.n_el, op.n_p)
            total = hx.apply_operator(op, ones, threads=4).flat().sum()
            worst = max(worst, abs(total - volume))
    assert worst <= 1e-10, worst
