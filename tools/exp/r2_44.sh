# r2_44: N=7 launch shapes under back-to-back (PDL) timing
OUT=gpurun_out/r2_44
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do
  python tools/b2b.py 20 BP1.0:32 BP1.0:46 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  for lib in paper_1711_00903_b200/variants/lib_t*.so; do
    HX_LIB_PATH=$PWD/$lib python tools/b2b.py 20 BP1.0:32 BP1.0:46 >> $OUT/b2b.jsonl
  done
  for lib in paper_1711_00903_b200/variants/lib_bp3_*.so; do
    HX_LIB_PATH=$PWD/$lib python tools/b2b.py 20 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  done
done
echo done > $OUT/DONE
