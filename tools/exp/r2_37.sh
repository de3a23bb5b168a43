# r2_37: programmatic dependent launch for back-to-back device applies
OUT=gpurun_out/r2_37
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for rep in 1 2 3; do
  timeout 600 python bench.py --quick > $OUT/bench_pdl_$rep.json 2>> $OUT/bench.err
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_nopdl.so timeout 600 python bench.py --quick > $OUT/bench_nopdl_$rep.json 2>> $OUT/bench.err
done
echo done > $OUT/DONE
