#!/bin/bash
# r2_60: BP3.5 S2 / S4 lane orders (k-fastest / k-paired, HX_GEN_BP35_ORD) --
# parity of the variant, config-4 BP3.5 sweep x2 and the N=7 headline back to
# back x3, product vs variant
OUT=gpurun_out/r2_60
mkdir -p $OUT
V=$PWD/paper_1711_00903_b200/variants/lib_ord35.so
HX_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg.py -q -x -p no:cacheprovider -k "BP3.5" > $OUT/parity.txt 2>&1
echo "exit $?" >> $OUT/parity.txt
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.5 --degrees 3..15 >> $OUT/sweep.jsonl
  HX_LIB_PATH=$V python tools/degree_sweep.py --bps BP3.5 --degrees 3..15 >> $OUT/sweep.jsonl
done
for i in 1 2 3; do
  python tools/b2b.py 40 BP3.5:32 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$V python tools/b2b.py 40 BP3.5:32 >> $OUT/b2b.jsonl
done
