#!/bin/bash
# r2_56: BP3.0 -- the next tile's S1 q line loaded into registers during S7 /
# S8 / S9 (HX_BP3_QAHEAD) vs loaded in S1 (product), back to back, x3
OUT=gpurun_out/r2_56
mkdir -p $OUT
for i in 1 2 3; do
  python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  for v in qa7 qa8 qa9; do
    HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  done
done
