#!/bin/bash
# r2_52: ncu --set full of the high-degree kernels (BP1.0 N=15, BP3.0 N=12 and
# N=15) at config-4 size, with source-level stall sampling
OUT=gpurun_out/r2_52
mkdir -p $OUT
for spec in "bp1 23 15" "bp3 23 15" "bp3 25 12"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1_kernel -s 2 -c 1 \
    -o $OUT/prof_$1_n$3 python tools/profile_one.py $1 $2 $3 > $OUT/ncu_$1_n$3.log 2>&1
  ncu -i $OUT/prof_$1_n$3.ncu-rep --page source --csv > $OUT/src_$1_n$3.csv 2>/dev/null
  ncu -i $OUT/prof_$1_n$3.ncu-rep --page raw --csv > $OUT/raw_$1_n$3.csv 2>/dev/null
done
