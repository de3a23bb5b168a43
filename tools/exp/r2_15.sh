# r2_15: BP3.0 N=7 permuted lane tables, entries kept in two opaque registers
OUT=gpurun_out/r2_15
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "BP3.0" > $OUT/parity_default.log 2>&1; echo "exit $?" >> $OUT/parity_default.log
for rep in 1 2 3; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_noperm.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.0:32 BP3.0:46 BP3.0:16 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp3_kernel" -s 1 -c 1 -o $OUT/prof_bp3 python tools/profile_one.py bp3 > $OUT/ncu_bp3.log 2>&1
echo done > $OUT/DONE
