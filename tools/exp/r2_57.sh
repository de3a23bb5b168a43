#!/bin/bash
# r2_57: BP3.0 N=10..15 -- the next tile's factors prefetched into L2 one
# tile ahead (at S6, with the next q) instead of at S2 of their own tile
OUT=gpurun_out/r2_57
mkdir -p $OUT
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.0 --degrees 10..15 >> $OUT/sweep.jsonl
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_pfa10.so python tools/degree_sweep.py --bps BP3.0 --degrees 10..15 >> $OUT/sweep.jsonl
done
