# r2_32: BP3.0 / BP1.0 N=7 launch shapes across E (the degree-sweep tune only saw E=97,336)
OUT=gpurun_out/r2_32
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do
timeout 300 python tools/sweep.py prod BP3.5:16 BP3.5:32 BP3.0:16 BP3.0:24 BP3.0:32 BP3.0:46 BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
for lib in paper_1711_00903_b200/variants/lib_bp3_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.0:16 BP3.0:24 BP3.0:32 BP3.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
for lib in paper_1711_00903_b200/variants/lib_t*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
echo done > $OUT/DONE
