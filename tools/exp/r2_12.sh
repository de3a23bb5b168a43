# r2_12: BP3.0 split-warp kernel (a warp pair per line) at N=7..15: load-group fences 1/2/4, MINB 1/2
OUT=gpurun_out/r2_12
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for v in split_g2 split_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity_$v.log 2>&1; echo "exit $?" >> $OUT/parity_$v.log
done
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 7..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
