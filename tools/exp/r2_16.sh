# r2_16: BP3.0 N>=10 layouts weighted by pass counts (T/Z joint for ACCS degrees)
OUT=gpurun_out/r2_16
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_wt.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity_wt.log 2>&1; echo "exit $?" >> $OUT/parity_wt.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_wt.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 10..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_wt.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp3_kernel" -s 1 -c 1 -o $OUT/prof_wt12 python tools/profile_one.py bp3 28 12 > $OUT/ncu_wt.log 2>&1
echo done > $OUT/DONE
