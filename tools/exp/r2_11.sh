# r2_11: BP3.0 factor ring (per-thread cp.async, FR t-slices ahead) depth 2/3/4 at N<=9; product = high-N ACCS/SER policy
OUT=gpurun_out/r2_11
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "BP3.0" > $OUT/parity_default.log 2>&1; echo "exit $?" >> $OUT/parity_default.log
for v in fr2 fr3 fr4; do
  HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "BP3.0" > $OUT/parity_$v.log 2>&1; echo "exit $?" >> $OUT/parity_$v.log
done
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib .so) BP3.0:32 BP3.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
done
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --degrees 1..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
