# r2_08: full GPU tests; BP1.0 diagnostic variants (no q / no GwJ / no store HBM streams)
OUT=gpurun_out/r2_08
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP1.0:16 BP1.0:32 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
