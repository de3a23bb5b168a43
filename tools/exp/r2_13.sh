# r2_13: ncu of the split-warp BP3.0 kernel vs the product at N=12 (side 28)
OUT=gpurun_out/r2_13
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_split_g2.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp3s?_kernel" -s 1 -c 1 -o $OUT/prof_split12 python tools/profile_one.py bp3 28 12 > $OUT/ncu_split.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp3s?_kernel" -s 1 -c 1 -o $OUT/prof_prod12 python tools/profile_one.py bp3 28 12 > $OUT/ncu_prod.log 2>&1
echo done > $OUT/DONE
