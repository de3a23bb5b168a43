#!/usr/bin/env python3
"""apply_operator on host numpy data: pageable arrays vs page-locked ones
(BP3.5 N=7 E=32768), and the cost of page-locking 134 MB on the fly."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402

mesh = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
op = hx.make_operator(hx.BP35, 7, mesh, lam=1.0)
q = np.random.default_rng(0).standard_normal((mesh.n_el, op.n_p))
fv = hx.FieldVector(mesh.n_el, op.n_p, q)
for _ in range(2):
    hx.apply_operator(op, fv)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    hx.apply_operator(op, fv)
print("pageable numpy apply_operator ms", (time.perf_counter() - t) / 5 * 1e3)
qp = torch.from_numpy(q).pin_memory()
op_ = torch.empty_like(qp).pin_memory()
for _ in range(2):
    hx.apply_host(op, qp.numpy(), op_.numpy())
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    hx.apply_host(op, qp.numpy(), op_.numpy())
    torch.cuda.synchronize()
print("pinned apply_host ms", (time.perf_counter() - t) / 5 * 1e3)
cudart = torch.cuda.cudart()
a = np.empty_like(q)
t = time.perf_counter()
for _ in range(5):
    cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    cudart.cudaHostUnregister(a.ctypes.data)
print("register+unregister 134 MB ms", (time.perf_counter() - t) / 5 * 1e3)
