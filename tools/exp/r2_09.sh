# r2_09: BP3.0 ACCS (accumulator through shared memory) at N>=10 in the product;
# variants: ACCS from N=7 (MINB 2/3), MINB 2/3 at all N, BP3.5 MINB 2; no-HBM floor.
OUT=gpurun_out/r2_09
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "BP3.0" > $OUT/parity_default.log 2>&1; echo "exit $?" >> $OUT/parity_default.log
for v in accs7 accs7_m3 bp3_m2 bp3_m3 bp35_m2; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "test_degree_sweep_matches_oracle or golden" > $OUT/parity_$v.log 2>&1; echo "exit $?" >> $OUT/parity_$v.log
done
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_{accs7,accs7_m3,bp3_m3,noqws}.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.0:32 BP3.0:46 BP3.5:32 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_{bp3_m2,bp3_m3,bp35_m2}.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0,BP3.5 --degrees 9..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
