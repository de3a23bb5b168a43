# r2_28: BP1.0 c-fastest S3 lanes with (i, j, k) GwJ slot order (ORD bit 8) at the model-chosen degrees
OUT=gpurun_out/r2_28
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "BP1.0" > $OUT/parity_prod.log 2>&1; echo "exit $?" >> $OUT/parity_prod.log
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_cfast.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg.py -m gpu -q -p no:cacheprovider -k "BP1.0 or bp1" > $OUT/parity_cfast.log 2>&1; echo "exit $?" >> $OUT/parity_cfast.log
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_cfast.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP1.0 --degrees 2..14 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
echo done > $OUT/DONE
