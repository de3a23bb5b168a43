# r2_25: ncu of the N=8 dips (BP3.0, BP1.0) and BP1.0 N=12
OUT=gpurun_out/r2_25
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp3_kernel" -s 1 -c 1 -o $OUT/prof_bp3_n8 python tools/profile_one.py bp3 41 8 > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp1_kernel" -s 1 -c 1 -o $OUT/prof_bp1_n8 python tools/profile_one.py bp1 41 8 > $OUT/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp1_kernel" -s 1 -c 1 -o $OUT/prof_bp1_n12 python tools/profile_one.py bp1 28 12 > $OUT/ncu3.log 2>&1
echo done > $OUT/DONE
