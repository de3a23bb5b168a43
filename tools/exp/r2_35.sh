# r2_35: BP3.0 N>=7 non-ACCS S5 with t / lam GwJ t through the own T line (frees registers for factor loads)
OUT=gpurun_out/r2_35
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_tvsmem.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_tvsmem.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.0:16 BP3.0:24 BP3.0:32 BP3.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 7..11 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
echo done > $OUT/DONE
