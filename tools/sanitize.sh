#!/bin/bash
# compute-sanitizer passes over the GPU parity suites (run on the GPU box):
#   memcheck (out-of-bounds / misaligned), racecheck (shared-memory hazards),
#   synccheck (barrier misuse).   bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out/sanit}
mkdir -p "$OUT"
timeout 2000 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_helpers.py tests/test_gpu_assembly.py \
  tests/test_gpu_cg.py tests/test_gpu_acceptance.py tests/test_gpu_hostpath.py -q -x -p no:cacheprovider \
  -k "not full_size and not sharded_assembled and not 64bit and not two_ranks and not report_cli" \
  > "$OUT/memcheck.log" 2>&1
echo "exit $?" >> "$OUT/memcheck.log"
timeout 2000 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 \
  --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_helpers.py \
  tests/test_gpu_assembly.py -q -x -p no:cacheprovider \
  -k "degree_sweep or every_degree or golden or dss or cg_update" > "$OUT/racecheck.log" 2>&1
echo "exit $?" >> "$OUT/racecheck.log"
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 99 python -m pytest \
  tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "degree_sweep" > "$OUT/synccheck.log" 2>&1
echo "exit $?" >> "$OUT/synccheck.log"
