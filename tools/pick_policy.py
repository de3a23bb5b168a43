#!/usr/bin/env python3
"""Pick the fastest launch shape per (kernel, degree) from degree-sweep
autotuning runs and write tools/tune_policy.json for gen_layouts.py.

    python tools/pick_policy.py gpurun_out/tune01/tune.jsonl [more.jsonl ...]

Variant library names encode the shape: lib_t{target_threads}_m{min_blocks}.so.
"""
import collections
import json
import os
import re
import sys

BP = {"BP1.0": 10, "BP3.5": 35, "BP3.0": 30}


def main(paths):
    best = collections.defaultdict(dict)
    for path in paths:
        for line in open(path):
            r = json.loads(line)
            m = re.match(r"lib_t(\d+)_m(\d+)\.so", r["lib"])
            if not m:
                continue
            key = (BP[r["bp"]], r["degree"])
            shape = (int(m.group(1)), int(m.group(2)))
            best[key][shape] = max(best[key].get(shape, 0.0), r["gdof_per_s"])
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from gen_layouts import TARGET_THREADS, min_blocks
    policy = []
    for (bp, deg), shapes in sorted(best.items()):
        (t, mb), v = max(shapes.items(), key=lambda kv: kv[1])
        default = (TARGET_THREADS, min_blocks(bp, deg))
        # keep the default shape unless another is clearly (>2 %) faster
        if default in shapes and shapes[default] >= 0.98 * v:
            (t, mb), v = default, shapes[default]
        policy.append([bp, deg, t, mb])
        print(f"bp={bp} N={deg}: t{t}_m{mb} {v:.1f} GDOF/s")
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tune_policy.json")
    with open(out, "w") as fh:
        json.dump(policy, fh)
    print("wrote", out)


if __name__ == "__main__":
    main(sys.argv[1:])
