#!/usr/bin/env python3
"""Host-memory paths at the headline size (BP3.5 N=7 E=32768): the drop-in
apply_operator on plain (pageable) numpy arrays -- hx_apply_host_staged --
for several staging chunk sizes, against the pinned hx_apply_host pipeline
and the PCIe bound.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402
from paper_1711_00903_b200 import operators  # noqa: E402

REPS = 10
mesh = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
op = hx.make_operator(hx.BP35, 7, mesh, lam=1.0)
q = np.random.default_rng(0).standard_normal((mesh.n_el, op.n_p))
fv = hx.FieldVector(mesh.n_el, op.n_p, q)
res = {"threads": int(os.environ.get("HX_HOST_THREADS", os.cpu_count() or 1))}


def wall(fn, reps=REPS):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return round(float(np.median(ts)) * 1e3, 3)


res["apply_operator_numpy_ms"] = wall(lambda: hx.apply_operator(op, fv))
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
dst = np.empty_like(q)
dst[:] = 0.0
for mib in (4, 8, 16, 32, 64):
    ch = operators.host_chunk_elements(op, mib << 20)
    res[f"staged_pinned_out_{mib}MiB_ms"] = wall(
        lambda: operators._apply_numpy(op, q, operators._pinned_empty(q.shape), flag, stream, ch))
    res[f"staged_pageable_out_{mib}MiB_ms"] = wall(
        lambda: operators._apply_numpy(op, q, dst, flag, stream, ch))
qp = torch.from_numpy(q).pin_memory()
op_ = torch.empty_like(qp).pin_memory()
for mib in (16, 32, 64):
    ch = operators.host_chunk_elements(op, mib << 20)
    work = operators._device_work(op, ch)
    res[f"pinned_apply_host_{mib}MiB_ms"] = wall(
        lambda: hx.apply_host(op, qp.numpy(), op_.numpy(), chunk_el=ch, work=work))
t = time.perf_counter()
a = np.empty_like(q)
a[:] = q
res["numpy_copy_134MB_fresh_ms"] = round((time.perf_counter() - t) * 1e3, 3)
print(json.dumps(res), flush=True)
