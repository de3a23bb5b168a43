#!/usr/bin/env python3
"""e2e (hx_apply_host) step time vs pipeline chunk size, BP3.5 N=7 E=32768,
20 back-to-back steps (the bench protocol)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1711_00903_b200 as hx
from paper_1711_00903_b200 import _native
mesh = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
op = hx.make_operator(hx.BP35, 7, mesh, lam=1.0)
n = mesh.n_el * op.n_p
qh = torch.empty(n, dtype=torch.float64).pin_memory().numpy(); qh[:] = np.random.default_rng(0).standard_normal(n)
oh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
for chunk in (256, 512, 1024, 2048, 4096, 8192, 12288, 16384):
    nb = _native.lib().hx_apply_host_workspace(op.plan.handle, chunk)
    work = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
    for _ in range(3): hx.apply_host(op, qh, oh, chunk_el=chunk, work=work)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): hx.apply_host(op, qh, oh, chunk_el=chunk, work=work)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"chunk {chunk:5d} el ({chunk*op.n_p*8/2**20:.0f} MiB): {ms:.3f} ms  {n/ms/1e6:.2f} GDOF/s", flush=True)
