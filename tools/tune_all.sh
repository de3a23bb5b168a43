#!/bin/bash
# Degree sweep for every tuning-variant library (autotuning of the launch shape).
OUT=gpurun_out/${1:-tune}
mkdir -p "$OUT"
for lib in paper_1711_00903_b200/variants/lib_*.so; do
  name=$(basename $lib .so)
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 \
    --bps "${BPS:-BP1.0,BP3.5,BP3.0}" --degrees "${DEGREES:-1..15}" \
    --out "$OUT/tune.jsonl" > "$OUT/$name.log" 2>&1
done
echo done > "$OUT/DONE"
