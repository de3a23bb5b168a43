"""CPU: the generated shared-memory layouts (csrc/hx_layouts.h, from
tools/gen_layouts.py) are sound for every kernel and degree -- each tensor
phase maps its (k, j, i) points injectively into its element buffer, inside
the buffer, and a tile fits the 227 KB shared-memory limit.  A bad table would
alias shared memory silently, so this is checked on the committed header."""

import os
import re
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import gen_layouts  # noqa: E402

HEADER = os.path.join(ROOT, "paper_1711_00903_b200", "csrc", "hx_layouts.h")


def parse_header():
    text = open(HEADER).read()
    cfgs = {}
    pat = re.compile(
        r"struct Cfg<(\d+), (\d+)> \{\s*static constexpr int EPB = (\d+), NT = (\d+), MINB = (\d+);"
        r"\s*static constexpr int QS = (\d+);[^\n]*\n\s*static constexpr int ORD = (\d+);[^\n]*\n"
        r"\s*static constexpr int ACCS = (\d+), SER = (\d+);[^\n]*\n"
        r"\s*static constexpr int EBUF\[\d+\] = \{([^}]*)\};\s*static constexpr Lay L\[\d+\] = "
        r"\{(.*?)\};\n\};", re.S)
    for m in pat.finditer(text):
        bp, deg, epb, nt, minb, qs, ord_, accs, ser = (int(m.group(i)) for i in range(1, 10))
        ebuf = [int(x) for x in m.group(10).split(",")]
        lays = [tuple(int(v) for v in t.split(",")) for t in re.findall(r"\{([^{}]*)\}",
                                                                       m.group(11))]
        cfgs[(bp, deg)] = dict(epb=epb, nt=nt, minb=minb, qs=qs, ord=ord_, accs=accs,
                               ser=ser, ebuf=ebuf, lays=lays)
    return cfgs


CFGS = parse_header()


def test_header_has_every_kernel_and_degree():
    # 11: the element helpers (hx_interp.cu), BP1.0's former stage order
    assert set(CFGS) == {(bp, d) for bp in (10, 35, 30, 11) for d in range(1, 16)}


@pytest.mark.parametrize("key", sorted(CFGS))
def test_layout_injective_in_bounds_and_fits(key):
    bp, deg = key
    c = CFGS[key]
    n, m = deg + 1, deg + 2
    phases = gen_layouts.phases(bp, n, m, c["ord"])
    assert len(phases) == len(c["lays"])
    for (buf, dims, _pats), lay in zip(phases, c["lays"]):
        d0, d1, d2 = dims
        seen = set()
        for k in range(d0):
            for j in range(d1):
                for i in range(d2):
                    a = gen_layouts.kofs(lay, k) + j * lay[1] + i
                    assert a not in seen, (key, dims, lay, (k, j, i))
                    seen.add(a)
        assert max(seen) < c["ebuf"][buf], (key, dims, lay, c["ebuf"][buf])
    smem = sum(c["ebuf"]) * c["epb"] * 8 + (c["epb"] * n * c["qs"] * 8 + 16 if c["qs"] else 0)
    assert smem <= 227 * 1024, (key, smem)
    if c["accs"] and bp == 30:  # BP3.0: Z is written in place over T's k-lines
        assert c["lays"][5] == c["lays"][4], key
    assert c["ser"] == 0 or bp == 30, key
    assert c["accs"] == 0 or bp in (30, 35), key  # BP3.5: the lean kernel form
    assert c["nt"] % 32 == 0 and 32 <= c["nt"] <= 1024
