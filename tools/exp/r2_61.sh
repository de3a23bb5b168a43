#!/bin/bash
# r2_61: BP3.0 k-paired S2 / S8 lane order (ORD 4) allowed at every degree
# (the model picks it with ORD 8 at N = 4, 8, 10, 12) -- parity, config-4
# BP3.0 sweep x2, product vs variant
OUT=gpurun_out/r2_61
mkdir -p $OUT
V=$PWD/paper_1711_00903_b200/variants/lib_ord3.so
HX_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.txt 2>&1
echo "exit $?" >> $OUT/parity.txt
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.0 --degrees 2..15 >> $OUT/sweep.jsonl
  HX_LIB_PATH=$V python tools/degree_sweep.py --bps BP3.0 --degrees 2..15 >> $OUT/sweep.jsonl
done
