#!/usr/bin/env python3
"""Generate the golden fixtures from the reference implementation itself.

Runs ONLY in the build container, where the reference is importable from
/root/reference/pkg/src (it does not exist on the GPU box).  Output:
tests/golden/golden.npz (committed).  Re-run with

    python tests/golden/make_golden.py

Contents (keys are prefixed ``{bp}_N{deg}_``):
  vertices : mesh corners used (perturb_mesh(build_cube_mesh(side, 2.0), 0.15, seed))
  interp / diff / nodes / weights : the reference 1-D matrices and rule
  factors  : reference geometric_factors (full for N<=4, element 0 otherwise)
  q, out_lam{L} : FieldVector.random input and reference apply_operator output
plus ``helper_N{deg}_{q,gl,t,gll}`` (reference interpolate_to_gl / project_to_gll
on three random element tensors),
plus ``counters_{bp}_{variant}_N{deg}`` (one-element counter values, lam=1),
``traffic`` / ``flops`` tables and quadrature rules.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hexbench import dense, perf  # noqa: E402
from hexbench.mesh import build_cube_mesh, perturb_mesh  # noqa: E402
from hexbench.operators import (BENCHMARKS, BP1, BP3, BP35, AccessCounters,  # noqa: E402
                                FieldVector, apply_operator, interpolate_to_gl,
                                make_operator, project_to_gll)
from hexbench.reference_ops import interp_matrix  # noqa: E402
from hexbench.quadrature import gl_rule, gll_rule  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# (degree, elements per side): 2x2x2 meshes for N<=4 and the headline N=7,
# a single element elsewhere (keeps the committed fixture small)
CASES = [(1, 2), (2, 2), (3, 2), (4, 2), (5, 1), (6, 1), (7, 2), (8, 1), (11, 1), (15, 1)]
LAMS = (0.0, 0.7)


def tag(bp):
    return {BP1: "bp1", BP35: "bp35", BP3: "bp3"}[bp]


def main():
    g = {}
    for deg, side in CASES:
        mesh = perturb_mesh(build_cube_mesh(side, 2.0), amplitude=0.15, seed=7)
        for bp in BENCHMARKS:
            key = f"{tag(bp)}_N{deg}_"
            op = make_operator(bp, deg, mesh, lam=LAMS[1])
            q = FieldVector.random(mesh.n_el, op.n_p, seed=deg)
            g[key + "vertices"] = mesh.vertices
            g[key + "q"] = q.data
            if op.interp is not None:
                g[key + "interp"] = op.interp.entries
            if op.diff is not None:
                g[key + "diff"] = op.diff.entries
            rule = gll_rule(deg + 1) if bp == BP35 else gl_rule(deg + 2)
            g[key + "nodes"] = rule.nodes
            g[key + "weights"] = rule.weights
            fac = op.factors.data
            if deg <= 4:
                g[key + "factors"] = fac
            elif deg in (7, 15):
                g[key + "factors"] = fac[:1]
            for lam in LAMS:
                opl = make_operator(bp, deg, mesh, lam=lam)
                out = apply_operator(opl, q)
                g[key + f"out_lam{lam}"] = out.data
                if deg <= dense.MAX_ORACLE_DEGREE and lam > 0:
                    # record the dense-oracle error the reference itself achieves
                    worst = 0.0
                    for e in range(mesh.n_el):
                        v = mesh.vertices[e]
                        if bp == BP1:
                            mat = dense.assemble_mass(v, deg)
                        elif bp == BP35:
                            mat = dense.assemble_stiffness_collocation(v, deg, lam)
                        else:
                            mat = dense.assemble_stiffness_full_quadrature(
                                v, deg, lam, cross_check=False)
                        ref = dense.dense_apply(mat, q.data[e])
                        worst = max(worst, np.max(np.abs(out.data[e] - ref))
                                    / max(1.0, np.max(np.abs(ref))))
                    g[key + "dense_err"] = np.array(worst)
    one = build_cube_mesh(1, 2.0)
    for bp in BENCHMARKS:
        for variant in ("baseline", "fused", "symfused"):
            if variant == "symfused" and bp == BP35:
                continue
            rows = []
            for deg in range(1, 16):
                c = AccessCounters()
                apply_operator(make_operator(bp, deg, one, lam=1.0, variant=variant),
                               FieldVector.constant(1, (deg + 1) ** 3), c)
                rows.append([c.global_reads, c.global_writes, c.scratch_reads,
                             c.scratch_writes, c.interp_matrix_reads, c.flops, c.syncs])
            g[f"counters_{tag(bp)}_{variant}"] = np.array(rows, dtype=np.int64)
        g[f"traffic_{tag(bp)}"] = np.array(
            [[perf.traffic(bp, d).reads_doubles, perf.traffic(bp, d).writes_doubles]
             for d in range(1, 16)], dtype=np.int64)
        g[f"flops_{tag(bp)}"] = np.array([perf.flop_model(bp, "fused", d)
                                          for d in range(1, 16)], dtype=np.int64)
        for variant in ("fused", "symfused", "baseline"):
            if variant == "symfused" and bp == BP35:
                continue
            ser = perf.roofline_series(bp, range(1, 16), 512, 549e9, variant=variant,
                                       b_sh=perf.shared_bandwidth_ansatz())
            g[f"roofline_{tag(bp)}_{variant}"] = np.array(
                [[p.r_global, np.nan if p.r_shared is None else p.r_shared]
                 for p in ser.points])
    # element helpers (operators.py:352-364): 3 random element tensors per degree
    rng = np.random.default_rng(2024)
    for deg in (1, 2, 3, 5, 7, 8, 15):
        n, m = deg + 1, deg + 2
        mat = interp_matrix(deg)
        q = rng.standard_normal((3, n, n, n))
        t = rng.standard_normal((3, m, m, m))
        g[f"helper_N{deg}_q"] = q
        g[f"helper_N{deg}_gl"] = np.stack([interpolate_to_gl(x, mat) for x in q])
        g[f"helper_N{deg}_t"] = t
        g[f"helper_N{deg}_gll"] = np.stack([project_to_gll(x, mat) for x in t])
    for n in range(1, 21):
        r = gl_rule(n)
        g[f"gl{n}"] = np.stack([r.nodes, r.weights])
        if n >= 2:
            r = gll_rule(n)
            g[f"gll{n}"] = np.stack([r.nodes, r.weights])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB, {len(g)} arrays)")


if __name__ == "__main__":
    main()
