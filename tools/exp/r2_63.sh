#!/bin/bash
# r2_63: BP1.0 N=8..15 launch shapes re-measured on the round-2 kernel
# (product policy vs uniform 256-thread target with 1-3 CTAs/SM and 128-thread
# CTAs with 2 / 4 CTAs/SM), config 4, back to back
OUT=gpurun_out/r2_63
mkdir -p $OUT
python tools/degree_sweep.py --bps BP1.0 --degrees 8..15 >> $OUT/sweep.jsonl
for v in t256_m1 t256_m2 t256_m3 t128_m2 t128_m4; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so python tools/degree_sweep.py --bps BP1.0 --degrees 8..15 >> $OUT/sweep.jsonl
done
python tools/degree_sweep.py --bps BP1.0 --degrees 8..15 >> $OUT/sweep.jsonl
