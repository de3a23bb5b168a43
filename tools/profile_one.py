#!/usr/bin/env python3
"""Launch one operator a few times at its BASELINE size for an ncu capture:
    ncu ... python tools/profile_one.py bp35|bp1|bp3 [side] [degree]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402

BP = {"bp1": hx.BP1, "bp35": hx.BP35, "bp3": hx.BP3}[sys.argv[1]]
SIDE = int(sys.argv[2]) if len(sys.argv) > 2 else 32
DEG = int(sys.argv[3]) if len(sys.argv) > 3 else 7

mesh = hx.perturb_mesh(hx.build_cube_mesh(SIDE, 2.0), amplitude=0.15, seed=7)
op = hx.make_operator(BP, DEG, mesh, lam=1.0)
q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
out = torch.empty_like(q)
for _ in range(3):
    hx.apply_device(op, q, out)
torch.cuda.synchronize()
print("ok", BP, DEG, mesh.n_el)
