# r2_46: exact per-thread register caps (__maxnreg__) for BP3.0 / BP3.5 vs __launch_bounds__
OUT=gpurun_out/r2_46
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_maxnreg.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0 or BP3.5" > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
for i in 1 2; do
  for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_maxnreg.so; do
    HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 10 --warmup 3 --bps BP3.5,BP3.0 --degrees 7..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
  done
done
echo done > $OUT/DONE
