#!/usr/bin/env python3
"""Build tuning-variant libraries (never the product library).

Each variant is a generated layout table (tools/gen_layouts.py with a policy
override) compiled into paper_1711_00903_b200/variants/lib_<name>.so; select
one at run time with HX_LIB_PATH.  Names encode the BP1.0 shape so
tools/pick_policy.py can read them back:

    lib_t{T}_m{M}[_q{Q}].so   T target threads per CTA, M min resident CTAs
                              per SM (register budget), Q = 1: TMA q staging

    python tools/build_variants.py t256_m1_q1 t128_m4_q1 ...
"""
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import gen_layouts  # noqa: E402
from paper_1711_00903_b200 import build as native_build  # noqa: E402

VARIANTS = os.path.join(ROOT, "paper_1711_00903_b200", "variants")


BPS = {"bp1": gen_layouts.BP1, "bp35": gen_layouts.BP35, "bp3": gen_layouts.BP3}


def parse(name):
    """[bp1_|bp35_|bp3_]t<T>_m<M>[_q<Q>] -> (bps, T, M, Q); BP1.0 by default."""
    m = re.fullmatch(r"(?:(bp1|bp35|bp3)_)?t(\d+)_m(\d+)(?:_q(\d))?", name)
    if not m:
        raise SystemExit(f"bad variant name {name!r} (want [bpX_]t<T>_m<M>[_q<Q>])")
    bps = (BPS[m.group(1)],) if m.group(1) else (gen_layouts.BP1,)
    return bps, int(m.group(2)), int(m.group(3)), int(m.group(4) or 0)


def build_variant(name):
    """The variant's shape applies to the kernel its name selects (BP1.0 by
    default); the others keep the committed policy."""
    bps, t, mb, q = parse(name)
    pol_path = os.path.join(HERE, "tune_policy.json")
    policy = gen_layouts.load_policy(pol_path) if os.path.exists(pol_path) else {}
    for bp in bps:
        for deg in range(1, 16):
            policy[(bp, deg)] = (t, mb, q)
    hdr_dir = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(hdr_dir, exist_ok=True)
    hdr = os.path.join(hdr_dir, "hx_layouts.h")
    gen_layouts.main(hdr, policy)
    os.makedirs(VARIANTS, exist_ok=True)
    lib = os.path.join(VARIANTS, f"lib_{name}.so")
    native_build.build(force=True, defines=(f'HX_LAYOUTS_FILE="{hdr}"',), lib=lib)
    print("built", lib, flush=True)
    return lib


if __name__ == "__main__":
    for v in sys.argv[1:]:
        build_variant(v)
