set -x
OUT=gpurun_out/r2_01
mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu >> $OUT/nproc.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_hostpath.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "hostpath or host or full_size_device or BP1.0-7" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_coal.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib) BP1.0:32 BP1.0:16 BP1.0:46 >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
done
timeout 300 python tools/host_paths.py > $OUT/host_paths.json 2> $OUT/host_paths.err
