# r2_19: HX_HOST_OVERLAP e2e (tests + bench); BP3.5 lean form (nothing live across barriers) at N=7..15
OUT=gpurun_out/r2_19
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hostpath.py tests/test_gpu_bench.py tests/test_gpu_capi_c.py -m gpu -q -p no:cacheprovider > $OUT/pytest_host.log 2>&1; echo "exit $?" >> $OUT/pytest_host.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
for v in lean lean_m1 lean_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.5" > $OUT/parity_$v.log 2>&1; echo "exit $?" >> $OUT/parity_$v.log
done
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.5 --degrees 7..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
