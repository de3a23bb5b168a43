# r2_05/r2_06: BP1.0 variant libraries (prefetch order; launch shapes)
OUT=gpurun_out/${1:-r2_05}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:40 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
