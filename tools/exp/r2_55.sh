#!/bin/bash
# r2_55: per-degree S5 factor ring (N=11: 2 points, N=14: 1) in the product;
# BP3.0 N=7..15 config-4 sweep x2, and the same N=7 side-46 case under
# tools/b2b.py (40 applies, one event pair) vs degree_sweep (best of 3 x 10)
OUT=gpurun_out/r2_55
mkdir -p $OUT
for i in 1 2; do
  python tools/degree_sweep.py --bps BP3.0 --degrees 7..15 >> $OUT/sweep.jsonl
  python tools/b2b.py 40 BP3.0:46 BP3.0:32 >> $OUT/b2b.jsonl
  python tools/degree_sweep.py --bps BP3.0 --degrees 7 --steps 40 >> $OUT/sweep40.jsonl
done
