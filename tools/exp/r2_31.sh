# r2_31: BP3.5 N=7 fixed per-launch cost: deeper initial prefetch, launch shapes, at E = 4096 .. 97,336
OUT=gpurun_out/r2_31
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.5:16 BP3.5:24 BP3.5:32 BP3.5:40 BP3.5:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
echo done > $OUT/DONE
