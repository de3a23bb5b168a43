#!/bin/bash
# r2_49: fused CG direction with the loads hoisted above the stores -- CG /
# assembly GPU tests, then the element-local and assembled CG timings x3
mkdir -p gpurun_out/r2_49
timeout 900 python -m pytest tests/test_gpu_cg.py tests/test_gpu_assembly.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2_49/tests.txt 2>&1
echo "exit $?" >> gpurun_out/r2_49/tests.txt
timeout 600 python - > gpurun_out/r2_49/cg.jsonl 2>&1 <<'PY'
import json, bench
import paper_1711_00903_b200 as hx
mesh = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
op = hx.make_operator(hx.BP35, 7, mesh, lam=1.0)
for rep in range(3):
    r = bench.cg_report(op, mesh, iters=50)
    print(json.dumps({"rep": rep, "fused_ms": r["ms_per_iteration"],
                      "unfused_ms": r["unfused_direction"]["ms_per_iteration"]}), flush=True)
PY
