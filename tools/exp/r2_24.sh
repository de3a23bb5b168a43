# r2_24: launch-shape re-tune of BP3.5 / BP3.0 with the round-2 kernels; product BP1.0 after its re-tune
OUT=gpurun_out/r2_24
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP1.0,BP3.5,BP3.0 --out $OUT/prod.jsonl > /dev/null 2>> $OUT/sweep.err
for lib in paper_1711_00903_b200/variants/lib_bp35_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.5 --out $OUT/tune.jsonl > /dev/null 2>> $OUT/sweep.err
done
for lib in paper_1711_00903_b200/variants/lib_bp3_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.0 --out $OUT/tune.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
