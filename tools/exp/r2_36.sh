# r2_36: BP3.0 ACCS degrees (10, 12, 13, 15): t kept in registers through S5 vs re-read
OUT=gpurun_out/r2_36
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_tvreg.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 10..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
echo done > $OUT/DONE
