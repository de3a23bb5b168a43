#!/bin/bash
# r2_72: BP3.5 S3 factors 1 / 2 points ahead in a register ring, N=7..15
OUT=gpurun_out/r2_72
mkdir -p $OUT
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.5 --degrees 7..15 >> $OUT/sweep.jsonl
  for f in 1 2; do
    HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_b35fpf$f.so python tools/degree_sweep.py --bps BP3.5 --degrees 7..15 >> $OUT/sweep.jsonl
  done
done
