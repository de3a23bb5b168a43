#!/usr/bin/env python3
"""Reference geometric factors for a sample of the BASELINE-size mesh.

The full-size parity tests feed the oracle device-generated factors; this
fixture pins the device generator itself at E=32768 (BASELINE configs[1],
perturb_mesh(build_cube_mesh(32, 2.0), 0.15, seed=7)): the reference's
geometric_factors (mesh.py:101-139) on 24 elements spread over the mesh, for
the GLL(8) rule of BP3.5 and the GL(9) rule of BP1.0 / BP3.0 at N=7.

Runs ONLY in the build container (imports /root/reference/pkg/src):

    python tests/golden/make_factor_sample.py

Output: tests/golden/factors_e32768.npz (committed): `elements` (indices),
`vertices` (their reference corners), `gll8`, `gl9` ((24, 7, q, q, q)).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from hexbench.mesh import HexMesh, build_cube_mesh, geometric_factors, perturb_mesh  # noqa: E402
from hexbench.quadrature import gl_rule, gll_rule  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "factors_e32768.npz")


def main():
    mesh = perturb_mesh(build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
    elements = np.unique(np.concatenate([[0, 1, 31, 1023, 1024, 16383, 32767],
                                         np.random.default_rng(0).integers(0, 32768, 17)]))
    sub = HexMesh(len(elements), mesh.vertices[elements], mesh.extent)
    np.savez_compressed(OUT, elements=elements, vertices=sub.vertices,
                        gll8=geometric_factors(sub, gll_rule(8)).data,
                        gl9=geometric_factors(sub, gl_rule(9)).data)
    print(f"wrote {OUT}: {len(elements)} elements")


if __name__ == "__main__":
    main()
