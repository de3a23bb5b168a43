# r2_03: t-first BP1.0 (coalesced k-line HBM stages, i-major GwJ), NT staging copies
OUT=gpurun_out/r2_03
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python tools/sweep.py new BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:40 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_coal.so timeout 300 python tools/sweep.py coal BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:40 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
timeout 300 python tools/host_paths.py > $OUT/host_paths.json 2> $OUT/host_paths.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp1_kernel" -s 1 -c 1 -o $OUT/prof_bp1 python tools/profile_one.py bp1 > $OUT/ncu_bp1.log 2>&1
