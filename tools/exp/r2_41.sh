# r2_41: BP3.0 factor L2-prefetch point (S1 / S2 product / S3 / next tile at S6), back to back
OUT=gpurun_out/r2_41
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
    HX_LIB_PATH=$PWD/$lib python tools/b2b.py 20 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  done
done
echo done > $OUT/DONE
