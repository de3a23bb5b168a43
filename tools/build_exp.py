#!/usr/bin/env python3
"""Build a diagnostic / experiment library with extra preprocessor defines
(never the product library):

    python tools/build_exp.py <name> [--layouts] DEF[=VAL] ...   ->  variants/lib_<name>.so

--layouts regenerates the layout table for the variant under the current
environment (e.g. HX_GEN_BP3_ACCS_MIN_N=7) instead of the committed one.

Select it at run time with HX_LIB_PATH (tools/sweep.py, tests)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_00903_b200 import build as native_build  # noqa: E402

if __name__ == "__main__":
    name, defs = sys.argv[1], [a for a in sys.argv[2:] if a != "--layouts"]
    if "--layouts" in sys.argv[2:]:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import gen_layouts
        hdr_dir = os.path.join(ROOT, "build", "variants", name)
        os.makedirs(hdr_dir, exist_ok=True)
        hdr = os.path.join(hdr_dir, "hx_layouts.h")
        pol = os.path.join(ROOT, "tools", "tune_policy.json")
        gen_layouts.main(hdr, gen_layouts.load_policy(pol) if os.path.exists(pol) else None)
        defs.append(f'HX_LAYOUTS_FILE="{hdr}"')
    defs = tuple(defs)
    out = os.path.join(ROOT, "paper_1711_00903_b200", "variants", f"lib_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    native_build.build(force=True, defines=defs, lib=out)
    print("built", out, flush=True)
