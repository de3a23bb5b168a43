#!/bin/bash
# r2_51: compute-sanitizer on the fused CG direction path (memcheck +
# racecheck), then the full GPU suite and smoke on the committed head
OUT=gpurun_out/r2_51
mkdir -p $OUT
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_cg.py tests/test_gpu_assembly.py -q -x -p no:cacheprovider \
  -k "dir or fused or cg_bitwise or graphed" > $OUT/memcheck.log 2>&1
echo "exit $?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_cg.py -q -x -p no:cacheprovider -k "apply_energy_dir_matches" > $OUT/racecheck.log 2>&1
echo "exit $?" >> $OUT/racecheck.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.txt 2>&1
echo "exit $?" >> $OUT/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
echo "exit $?" >> $OUT/smoke.txt
