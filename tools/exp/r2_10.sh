# r2_10: BP3.0 high degrees: ACCS on/off x MINB 1/2/3 x serialized S4/S6 lines; no-HBM floors
OUT=gpurun_out/r2_10
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for v in m2ser m3ser nacc_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "test_degree_sweep_matches_oracle and BP3.0" > $OUT/parity_$v.log 2>&1; echo "exit $?" >> $OUT/parity_$v.log
done
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 9..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
