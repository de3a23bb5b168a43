#!/bin/bash
# r2_48: CG direction fused into the matvec -- GPU tests of the CG / assembly
# suites and the parity suite, then the default bench (details carry the CG rows)
mkdir -p gpurun_out/r2_48
timeout 1500 python -m pytest tests/test_gpu_cg.py tests/test_gpu_assembly.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2_48/tests.txt 2>&1
echo "exit $?" >> gpurun_out/r2_48/tests.txt
timeout 900 python bench.py > gpurun_out/r2_48/bench.json 2> gpurun_out/r2_48/bench.err
cp -f gpurun_out/bench_details.json gpurun_out/r2_48/ 2>/dev/null
