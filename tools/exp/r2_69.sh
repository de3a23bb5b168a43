#!/bin/bash
# r2_69: BP3.0 -- the next tile's q L2 prefetch issued at S4 / S5 / S8
# instead of S6 (HX_QPF_BP3), N=7 back to back x3
OUT=gpurun_out/r2_69
mkdir -p $OUT
for i in 1 2 3; do
  python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  for v in qpf4 qpf5 qpf8; do
    HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  done
done
