# r2_18: BP3.5 register budget (MINB 1 / 3) at N >= 9
OUT=gpurun_out/r2_18
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 --bps BP3.5 --degrees 9..15 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
echo done > $OUT/DONE
