#!/bin/bash
# Run tools/sweep.py for every variant library (tuning experiments).
OUT=gpurun_out/${1:-sweep}
shift
mkdir -p "$OUT"
for lib in paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py "$(basename $lib .so)" "$@" >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
done
echo done >> "$OUT/sweep.err"
