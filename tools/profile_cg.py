#!/usr/bin/env python3
"""A few assembled-CG iterations (BP3.5 N=7, side 32) for an ncu launch list:
    ncu --metrics gpu__time_duration.sum ... python tools/profile_cg.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402
from paper_1711_00903_b200.cg import CGWorkspace, cg_iterations, cg_iterations_assembled  # noqa: E402

mesh = hx.build_cube_mesh(32, 2.0)
op = hx.make_operator(hx.BP35, 7, mesh, lam=0.0)
b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
w = CGWorkspace(b)
cg_iterations_assembled(op, 32, b, 3, w)
cg_iterations(op, b, 3, w)
torch.cuda.synchronize()
print("ok")
