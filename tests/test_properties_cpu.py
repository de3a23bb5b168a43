"""CPU property tests (hypothesis) of the host-side logic the kernels rely
on: the element partition, the assembled-shard halos, the lane orders of the
layout generator and the gather-scatter algebra of the assembly checker."""

import os
import sys

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import hexbench_oracle as orc
from paper_1711_00903_b200 import shard
from paper_1711_00903_b200.cg import AssembledShard

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tools"))
import gen_layouts  # noqa: E402


@given(st.integers(0, 10 ** 6), st.integers(1, 64))
def test_partition_covers_contiguously(n_el, world):
    parts = shard.partition(n_el, world)
    assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == n_el
    assert all(lo <= hi for lo, hi in parts)
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    sizes = [hi - lo for lo, hi in parts]
    assert max(sizes) - min(sizes) <= 1


@given(st.integers(2, 40), st.integers(1, 8), st.integers(1, 15))
def test_assembled_shard_halo_holds_every_neighbour(side, world, deg):
    e = side ** 3
    if min(hi - lo for lo, hi in shard.partition(e, world)) < side * side + side + 1:
        return  # rejected configuration (covered by test_assembled_shard_ranges)
    for r in range(world):
        sh = AssembledShard(side, deg, r, world)
        for el in (sh.lo, sh.hi - 1):
            cx, cy, cz = el // (side * side), (el // side) % side, el % side
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dz in (-1, 0, 1):
                        x, y, z = cx + dx, cy + dy, cz + dz
                        if 0 <= x < side and 0 <= y < side and 0 <= z < side:
                            nb = (x * side + y) * side + z
                            assert sh.base <= nb < sh.top


@given(st.integers(1, 17), st.integers(1, 17))
def test_pair_coords_is_a_bijection(d0, d1):
    seen = {gen_layouts.pair_coords(ln, d0, d1) for ln in range(d0 * d1)}
    assert seen == {(k, a) for k in range(d0) for a in range(d1)}


@settings(max_examples=25, deadline=None)
@given(st.integers(1, 3), st.integers(1, 3), st.integers(0, 2 ** 31))
def test_gather_scatter_algebra(side, deg, seed):
    n3 = (deg + 1) ** 3
    rng = np.random.default_rng(seed)
    u, v = rng.standard_normal((2, side ** 3, n3))
    mult = orc.multiplicity(side, deg)
    du = orc.dss(u, side, deg)
    # Q Q^T is symmetric, and applying it to a continuous vector scales by the multiplicity
    assert abs(np.sum(du * v) - np.sum(u * orc.dss(v, side, deg))) <= 1e-10 * (1 + abs(np.sum(du * v)))
    np.testing.assert_allclose(orc.dss(du, side, deg), mult * du, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(orc.dss_passes(u, side, deg), du, rtol=1e-13, atol=1e-13)
