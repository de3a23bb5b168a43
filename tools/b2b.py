#!/usr/bin/env python3
"""Back-to-back applies with only a start / stop event around K launches
(no per-launch events between them): the stream of applies programmatic
dependent launch can overlap.  Prints one JSON line per operator.

    python tools/b2b.py [steps] [BP:side ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfgs = sys.argv[2:] or ["BP3.5:32", "BP3.0:32", "BP1.0:32"]
res = {"lib": os.path.basename(os.environ.get("HX_LIB_PATH", "default"))}
for c in cfgs:
    bp, side = c.split(":")
    mesh = hx.perturb_mesh(hx.build_cube_mesh(int(side), 2.0), amplitude=0.15, seed=7)
    op = hx.make_operator(bp, 7, mesh, lam=1.0)
    q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
    out = torch.empty_like(q)
    for _ in range(5):
        hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        for _ in range(steps):
            hx.apply_device(op, q, out)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        best = ms if best is None else min(best, ms)
    b = hx.traffic(bp, 7, mesh.n_el).bytes_per_element * mesh.n_el
    res[c] = {"ms": round(best, 4), "gdof": round(mesh.n_el * op.n_p / best / 1e6, 2),
              "frac": round(b / best / 1e6 / 6554.9, 4)}
print(json.dumps(res), flush=True)
