#!/bin/bash
# r2_59: BP3.0 N=7 with the k-paired S2 / S8 lane order (ORD 4, conflict-free
# X / Y / Z in the bank model) vs the product, back to back x3; parity of it
OUT=gpurun_out/r2_59
mkdir -p $OUT
V=$PWD/paper_1711_00903_b200/variants/lib_ord4.so
HX_LIB_PATH=$V timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.txt 2>&1
echo "exit $?" >> $OUT/parity.txt
for i in 1 2 3; do
  python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$V python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
done
HX_LIB_PATH=$V timeout 600 ncu --set full --clock-control none -k regex:bp3_kernel -s 1 -c 1 -o $OUT/prof_bp3_ord4 python tools/profile_one.py bp3 > $OUT/ncu.log 2>&1
