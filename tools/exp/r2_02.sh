# r2_02: GPU tests (all), bench, memcpy probe, BP1 E-sweep default vs coalesced-q/out hack
OUT=gpurun_out/r2_02
mkdir -p $OUT
gcc -O3 -mavx2 -pthread tools/memcpy_probe.c -o /tmp/memcpy_probe && /tmp/memcpy_probe > $OUT/memcpy_probe.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
cp gpurun_out/bench_details.json $OUT/ 2>/dev/null
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_coal.so; do
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py $(basename $lib) BP1.0:16 BP1.0:20 BP1.0:24 BP1.0:28 BP1.0:32 BP1.0:36 BP1.0:40 BP1.0:46 BP3.5:16 BP3.5:24 BP3.5:32 BP3.5:40 BP3.5:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
done
timeout 300 python tools/host_paths.py > $OUT/host_paths.json 2> $OUT/host_paths.err
