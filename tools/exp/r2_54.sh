#!/bin/bash
# r2_54: the first tile's factors prefetched in the prologue (before the PDL
# wait, so under the previous apply's drain) -- product (on) vs HX_PRO_FAC=0,
# back to back, interleaved x4
OUT=gpurun_out/r2_54
mkdir -p $OUT
for i in 1 2 3 4; do
  python tools/b2b.py 40 BP3.5:32 BP3.0:32 BP3.0:46 BP3.5:46 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_noprofac.so python tools/b2b.py 40 BP3.5:32 BP3.0:32 BP3.0:46 BP3.5:46 >> $OUT/b2b.jsonl
done
