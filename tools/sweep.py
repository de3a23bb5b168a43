#!/usr/bin/env python3
"""Time the three N=7 BASELINE configs with whatever library HX_LIB_PATH
points at (tuning experiments; prints one JSON line).  L2-warm; a GPU spacer
before each timed launch keeps host launch latency out of small-E times
(added after tune24: earlier BP1.0:16 entries include it)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1711_00903_b200 as hx

def run(bp, side, deg=7, steps=30, warmup=5):
    mesh = hx.perturb_mesh(hx.build_cube_mesh(side, 2.0), amplitude=0.15, seed=7)
    op = hx.make_operator(bp, deg, mesh, lam=1.0)
    q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
    out = torch.empty_like(q)
    for _ in range(warmup):
        hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    ev = []
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)  # spacer: the launch is queued before `s` (bench.gpu_spacer)
        s.record(); hx.apply_device(op, q, out); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    ms = statistics.median(s.elapsed_time(e) for s, e in ev)
    b = hx.traffic(bp, deg, mesh.n_el).bytes_per_element * mesh.n_el
    return {"gdof": round(mesh.n_el * op.n_p / ms / 1e6, 2), "frac": round(b / ms / 1e6 / 6554.9, 4),
            "ms": round(ms, 4), "threads": op.plan.threads, "epb": op.plan.elements_per_tile}

cfgs = sys.argv[2:] or ["BP3.5:32", "BP3.0:32", "BP1.0:32"]
res = {"lib": os.path.basename(os.environ.get("HX_LIB_PATH", "default")), "tag": sys.argv[1]}
for c in cfgs:
    bp, side = c.split(":")
    deg = 7
    if ":" in side:
        side, deg = side.split(":")
    res[c] = run(bp, int(side), int(deg))
print(json.dumps(res), flush=True)
