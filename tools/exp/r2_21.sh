# r2_21: BP3.0 launch shapes at N=1..3 (N=1 sits at 0.698)
OUT=gpurun_out/r2_21
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 10 --warmup 3 --bps BP3.0 --degrees 1..3 --out $OUT/sweep.jsonl > /dev/null 2>> $OUT/sweep.err
done
done
echo done > $OUT/DONE
