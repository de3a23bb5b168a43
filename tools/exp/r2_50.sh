#!/bin/bash
# r2_50: BP1.0 N=7 config-1 (E=4096, L2 flushed single launches) across
# launch shapes -- does a different shape fill the 148 SMs better at small E?
OUT=gpurun_out/r2_50
mkdir -p $OUT
for i in 1 2; do
  python tools/small_e.py BP1.0 2368 4096 5328 8192 >> $OUT/small_e.jsonl
  for lib in paper_1711_00903_b200/variants/lib_t*.so; do
    echo "{\"lib\": \"$(basename $lib)\"}" >> $OUT/small_e.jsonl
    HX_LIB_PATH=$PWD/$lib python tools/small_e.py BP1.0 2368 4096 5328 8192 >> $OUT/small_e.jsonl
  done
done
