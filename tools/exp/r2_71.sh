#!/bin/bash
# r2_71: low-degree (N=1..9) launch shapes re-measured on the final kernels
OUT=gpurun_out/r2_71
mkdir -p $OUT
python tools/degree_sweep.py --degrees 1..9 >> $OUT/sweep.jsonl
for v in t128_m4 t192_m3 t256_m2 t384_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_bp3_$v.so python tools/degree_sweep.py --bps BP3.0 --degrees 1..9 >> $OUT/sweep.jsonl
done
for v in t192_m3 t384_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_bp1_$v.so python tools/degree_sweep.py --bps BP1.0 --degrees 1..9 >> $OUT/sweep.jsonl
done
for v in t128_m4 t256_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_bp35_$v.so python tools/degree_sweep.py --bps BP3.5 --degrees 1..9 >> $OUT/sweep.jsonl
done
python tools/degree_sweep.py --degrees 1..9 >> $OUT/sweep.jsonl
