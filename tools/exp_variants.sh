#!/bin/bash
# Tuning experiment on the GPU box: parity + timing of every variant library.
#   bash tools/exp_variants.sh <tag> [pytest -k expr] [bps] [degrees]
OUT=gpurun_out/${1:-exp}
K=${2:-BP1.0}
BPS=${3:-BP1.0}
DEGREES=${4:-1..15}
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
for lib in paper_1711_00903_b200/libhexbench_b200.so paper_1711_00903_b200/variants/lib_*.so; do
  name=$(basename $lib .so)
  HX_LIB_PATH=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "$K" -p no:cacheprovider > "$OUT/parity_$name.log" 2>&1
  echo "exit $?" >> "$OUT/parity_$name.log"
  HX_LIB_PATH=$PWD/$lib timeout 300 python tools/sweep.py "$name" $(echo $BPS | tr ',' '\n' | sed 's/$/:32/') BP1.0:16 \
    >> "$OUT/n7.jsonl" 2> "$OUT/n7_$name.err"
  HX_LIB_PATH=$PWD/$lib timeout 900 python tools/degree_sweep.py --steps 8 --warmup 3 \
    --bps "$BPS" --degrees "$DEGREES" --out "$OUT/sweep.jsonl" > "$OUT/sweep_$name.log" 2>&1
done
echo done > "$OUT/DONE"
