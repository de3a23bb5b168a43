#!/bin/bash
# r2_53: BP3.0 S5 factors loaded 1-3 points ahead into a register ring
# (HX_BP3_FPF) at N = 7..15, config-4 sizes, back to back, x2
OUT=gpurun_out/r2_53
mkdir -p $OUT
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.0 --degrees 7..15 --out /dev/null | sed 's/^/{"lib": "product", "l": /; s/$/}/' >> $OUT/sweep.jsonl
  for f in 1 2 3; do
    HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_fpf$f.so python tools/degree_sweep.py --bps BP3.0 --degrees 7..15 --out /dev/null | sed "s/^/{\"lib\": \"fpf$f\", \"l\": /; s/\$/}/" >> $OUT/sweep.jsonl
  done
done
