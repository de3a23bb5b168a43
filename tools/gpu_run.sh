#!/bin/bash
# One gpurun session: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (from the repo root, on the GPU box):  bash tools/gpu_run.sh [tag] [stages]
#   stages: any of smoke,tests,bench,launches,ncu (default: all)
TAG=${1:-r01}
STAGES=${2:-smoke,tests,bench,launches,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
if [[ $STAGES == *smoke* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi
if [[ $STAGES == *tests* ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
fi
if [[ $STAGES == *bench* ]]; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/bench.err"
fi
if [[ $STAGES == *launches* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file "$OUT/launches.csv" python bench.py --quick --steps 5 --warmup 3 \
    > "$OUT/launches.log" 2>&1
fi
if [[ $STAGES == *ncu* ]]; then
  for K in bp35 bp1 bp3; do
    timeout 600 ncu --set full --clock-control none --import-source on \
      -k "regex:${K}_kernel" -s 1 -c 1 -o "$OUT/prof_${K}" \
      python tools/profile_one.py "$K" > "$OUT/ncu_${K}.log" 2>&1
  done
fi
if [[ $STAGES == *sweep* ]]; then
  timeout 1500 python tools/degree_sweep.py --out "$OUT/degree_sweep.jsonl" > "$OUT/degree_sweep.log" 2>&1
fi
if [[ $STAGES == *probe* ]]; then
  timeout 120 ./tools/fp64_probe > "$OUT/fp64_probe.txt" 2>&1
fi
echo done > "$OUT/DONE"
