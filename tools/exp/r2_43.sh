# r2_43: BP3.0 N=7 ACCS (acc parked in T) with t kept in registers through S5
OUT=gpurun_out/r2_43
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_accs7tv.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
for i in 1 2 3; do
  for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
    HX_LIB_PATH=$PWD/$lib python tools/b2b.py 20 BP3.0:32 BP3.0:46 >> $OUT/b2b.jsonl
  done
done
echo done > $OUT/DONE
