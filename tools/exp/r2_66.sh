#!/bin/bash
# r2_66: BP3.0 fused r-derivative stage order (ORD bit 16, kFR) at N=7..9 --
# parity, back to back at N=7 x3, config-4 N=7..9, product vs variant
OUT=gpurun_out/r2_66
mkdir -p $OUT
V=$PWD/paper_1711_00903_b200/variants/lib_fr.so
HX_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg.py -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.txt 2>&1
echo "exit $?" >> $OUT/parity.txt
for i in 1 2 3; do
  python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$V python tools/b2b.py 40 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
done
python tools/degree_sweep.py --bps BP3.0 --degrees 7..9 >> $OUT/sweep.jsonl
HX_LIB_PATH=$V python tools/degree_sweep.py --bps BP3.0 --degrees 7..9 >> $OUT/sweep.jsonl
HX_LIB_PATH=$V timeout 600 ncu --set full --clock-control none -k regex:bp3_kernel -s 1 -c 1 -o $OUT/prof_bp3_fr python tools/profile_one.py bp3 > $OUT/ncu.log 2>&1
