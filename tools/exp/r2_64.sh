#!/bin/bash
# r2_64: BP3.5 / BP3.0 N=8..15 launch shapes re-measured after the lane-order
# changes (tune57-59), config 4, back to back
OUT=gpurun_out/r2_64
mkdir -p $OUT
python tools/degree_sweep.py --bps BP3.5,BP3.0 --degrees 8..15 >> $OUT/sweep.jsonl
for v in t256_m1 t256_m3 t384_m1 t192_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_bp35_$v.so python tools/degree_sweep.py --bps BP3.5 --degrees 8..15 >> $OUT/sweep.jsonl
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_bp3_$v.so python tools/degree_sweep.py --bps BP3.0 --degrees 8..15 >> $OUT/sweep.jsonl
done
python tools/degree_sweep.py --bps BP3.5,BP3.0 --degrees 8..15 >> $OUT/sweep.jsonl
