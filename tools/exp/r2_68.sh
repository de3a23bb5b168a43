#!/bin/bash
# r2_68: the CG iteration's kernels -- launch list of 3 assembled + 3
# element-local iterations, and ncu --set full of the fused direction +
# matvec kernel (bp35_kernel<7, 1, 1>)
OUT=gpurun_out/r2_68
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/cg_launches.csv python tools/profile_cg.py > $OUT/launches.log 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:bp35_kernel<7, 1, 1>|bp35_kernel" -s 5 -c 1 \
  -o $OUT/prof_bp35_dir python tools/profile_cg.py > $OUT/ncu.log 2>&1
