#!/usr/bin/env python3
"""BP1.0 stored vs on-the-fly geometry at N=7 (E=4096 flushed, E=32768), one
JSON line per (lib, geometry, E); HX_LIB_PATH selects the library."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
for side in (16, 32, 46):
    mesh = hx.perturb_mesh(hx.build_cube_mesh(side, 2.0), amplitude=0.15, seed=7)
    for geometry in ("stored", "on_the_fly"):
        op = hx.make_operator(hx.BP1, 7, mesh, lam=1.0, geometry=geometry)
        q = torch.randn(mesh.n_el, op.n_p, dtype=torch.float64, device="cuda")
        out = torch.empty_like(q)
        for _ in range(3):
            hx.apply_device(op, q, out)
        times = []
        for _ in range(15):
            flush.add_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            hx.apply_device(op, q, out)
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e))
        ms = statistics.median(times)
        print(json.dumps({"lib": os.path.basename(os.environ.get("HX_LIB_PATH", "default")),
                          "geometry": geometry, "n_el": mesh.n_el, "us": ms * 1e3,
                          "gdof_per_s": mesh.n_el * op.n_p / ms / 1e6}), flush=True)
        del op, q, out
        torch.cuda.empty_cache()
