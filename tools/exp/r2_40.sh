# r2_40: fuller pre-wait prologue (PDL) vs product vs no-PDL, back-to-back
OUT=gpurun_out/r2_40
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  python tools/b2b.py 20 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_profull.so python tools/b2b.py 20 >> $OUT/b2b.jsonl
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_nopdl.so python tools/b2b.py 20 >> $OUT/b2b.jsonl
done
echo done > $OUT/DONE
