# r2_04: BP1.0 c-fastest j-lines, X (73,8) Y (153,17) at N=7
OUT=gpurun_out/r2_04
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg.py tests/test_gpu_helpers.py -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python tools/sweep.py new BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:40 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_coal.so timeout 300 python tools/sweep.py coal BP1.0:16 BP1.0:24 BP1.0:32 BP1.0:40 BP1.0:46 >> $OUT/esweep.jsonl 2>> $OUT/esweep.err
timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP1.0 --out $OUT/degree_sweep.jsonl > $OUT/degree_sweep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bp1_kernel" -s 1 -c 1 -o $OUT/prof_bp1 python tools/profile_one.py bp1 > $OUT/ncu_bp1.log 2>&1
