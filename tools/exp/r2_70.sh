#!/bin/bash
# r2_70: global loads cached in L2 only (-Xptxas -dlcm=cg) vs the default
# (L1 + L2) -- the streamed q / factor loads no longer allocate in L1
OUT=gpurun_out/r2_70
mkdir -p $OUT
V=$PWD/paper_1711_00903_b200/variants/lib_dlcmcg.so
for i in 1 2; do
  python tools/b2b.py 40 BP3.5:32 BP3.0:32 BP1.0:32 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$V python tools/b2b.py 40 BP3.5:32 BP3.0:32 BP1.0:32 >> $OUT/b2b.jsonl
done
python tools/degree_sweep.py --degrees 9..15 >> $OUT/sweep.jsonl
HX_LIB_PATH=$V python tools/degree_sweep.py --degrees 9..15 >> $OUT/sweep.jsonl
