# r2_26: BP3.0 k-fastest S4/S6 i-line lanes at even m (ORD bit 8)
OUT=gpurun_out/r2_26
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_ki.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity_ki.log 2>&1; echo "exit $?" >> $OUT/parity_ki.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_ki.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 2..14 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
echo done > $OUT/DONE
