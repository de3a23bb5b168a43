#!/usr/bin/env python3
"""Generate paper_1711_00903_b200/csrc/hx_layouts.h.

Every kernel stage reads or writes whole 1-D lines of a per-element 3-D
tensor staged in shared memory; one thread owns one line.  For each tensor
"phase" this script picks the row stride S1 and slice stride S0 (element
(k, j, i) lives at k*S0 + j*S1 + i) and the per-element buffer stride EBUF
that minimise shared-memory wavefronts over the access patterns the phase
sees, under the usual model for 64-bit accesses: a warp request is served
as two half-warps, and within a half-warp the cost is the largest number of
distinct 8-byte words that fall in the same 8-byte bank pair (word mod 16).

Patterns: 0 = k-lines (lanes enumerate (j, i)), 1 = j-lines (lanes (k, i)),
2 = i-lines (lanes (k, j)); consecutive threads own consecutive lines, and
the lines of EPB elements are laid end to end.  Patterns 3, 4, 5 are the same
lines with the lane enumeration transposed (the first coordinate fastest):
3 = k-lines over (i, j) with j fastest, 4 = j-lines with k fastest, 5 = i-lines
with k fastest.  BP1.0 picks its j-line / i-line lane orders jointly with the
strides (``ORD``): with one order per pattern no padding can make both the
(k,i) j-lines and the (k,a) i-lines of X conflict-free (ncu r08: S2/S4 paid
1.86x wavefronts), with k fastest in both it can.
"""

import json
import os
import sys

BP1, BP35, BP3 = 10, 35, 30
INTERP = 11  # element helpers (hx_interp.cu): BP1.0's former (s, r, t) stage order
TARGET_THREADS = 256


def _degrees(env, default):
    v = os.environ.get(env)
    return default if v is None else {int(x) for x in v.split(",") if x.strip()}


# BP3.0 degrees whose S5 accumulator goes through shared memory (Z aliases
# T's layout; hx_bp3.cu kAccS) -- frees m doubles of registers across S6 --
# and whose S4 / S6 finish one line before loading the other (kSerial).
# Measured per degree (profiles/r2_10_bp3_high_degree.md): they pay where
# the register file, not shared memory, caps the resident CTAs.
BP3_ACCS = _degrees("HX_GEN_BP3_ACCS", {10, 12, 13, 15})
BP3_SER = _degrees("HX_GEN_BP3_SER", {10, 12, 13})
# BP3.5 degrees whose kernel keeps nothing in registers across a barrier
# (hx_bp35.cu kLean, emitted as ACCS): q, D_t q and the accumulator go
# through the thread's own k-line of buffer A (r2_19: N=11 0.855 -> 0.873,
# N=12 0.852 -> 0.943, N=13 0.747 -> 0.791 and N=14 0.788 -> 0.823 at MINB 2,
# N=15 0.815 -> 0.882; slower at N <= 10, where the registers are there).
BP35_LEAN = _degrees("HX_GEN_BP35_LEAN", set(range(11, 16)))
# BP1.0 degrees whose S3 lane order may be c-fastest with the GwJ slot
# stored (i, j, k) (ORD bit 8; hx_bp1.cu, hx_geom.cu), chosen by the model
# (picked at N = 4, 8, 10, 12; r2_28: N=4 0.79 -> 0.82, N=12 0.51 -> 0.52)
BP1_CFAST = _degrees("HX_GEN_BP1_CFAST", {2, 4, 6, 8, 10, 12, 14})
# BP3.0 degrees (even m) whose S4 / S6 i-line lane order may be k-fastest
# (ORD bit 8), chosen by the model against the default (r2_26: N=4 0.84 ->
# 0.87, N=6 0.90 -> 0.92, N=8 0.78 -> 0.79, N=10 0.70 -> 0.72)
BP3_KI = _degrees("HX_GEN_BP3_KI", {2, 4, 6, 8, 10, 12, 14})
# BP3.0 degrees whose S2 / S8 i-lines may take the k-paired lane order (ORD
# 4, combined with ORD 8 where that applies).  Round 1 measured it 1-2 %
# slower at N=7 (r11/r12); on the round-2 kernel: N=7 +0.2 % (r2_59: shared
# wavefronts 40.5 M -> 38.9 M, conflicts 4.6 M -> 2.8 M), N=4 0.902 -> 0.910,
# N=8 0.815 -> 0.821, N=10 0.724 -> 0.739 (ORD 12); N=12 -0.004 (r2_61)
BP3_ORD4 = _degrees("HX_GEN_BP3_ORD4", {4, 7, 8, 10})
# BP3.5 degrees whose S2 / S4 lines may take the k-fastest (ORD 2) or
# k-paired (ORD 4, k-paired layouts) lane order; the k-line stages touch HBM
# and keep i-fastest lanes.  Measured (r2_60, config 4): N=9 0.975 -> 0.985,
# N=11 0.875 -> 0.925, N=13 0.795 -> 0.868; flat at every other degree
BP35_ORD = _degrees("HX_GEN_BP35_ORD", {9, 11, 13})
# BP3.0 degrees whose layouts weight each access pattern by the number of
# passes that use it (phases()) instead of counting every pattern once
# (r2_16: N=10 0.687 -> 0.706, N=12 0.598 -> 0.613, equal elsewhere; at
# N <= 9 the weighted search returns the unweighted layouts).
BP3_WEIGHTED = _degrees("HX_GEN_BP3_WEIGHTED", set(range(10, 16)))


def lines(d, pat):
    d0, d1, d2 = d
    return {0: (d1 * d2, d0), 1: (d0 * d2, d1), 2: (d0 * d1, d2), 4: (d0 * d2, d1),
            5: (d0 * d1, d2), 6: (d0 * d1, d2), 7: (d0 * d2, d1)}[pat]


def kofs(lay, k):
    """Offset of slice k: plain (k * s0), or k-paired when sq > 0: slices 2h
    and 2h+1 sit sq apart inside a pair block of stride s0."""
    s0, _, sq = lay
    return k * s0 if sq == 0 else (k // 2) * s0 + (k % 2) * sq


def pair_coords(l, d0, d1):
    """Pattern 6 lane order over (k, a): k pairs outermost, then a, then the
    k parity fastest; an odd trailing slice is enumerated alone."""
    g = 2 * d1
    full = (d0 // 2) * g
    if l < full:
        kh, r = divmod(l, g)
        a, kl = divmod(r, 2)
        return 2 * kh + kl, a
    return d0 - 1, l - full


def addr(d, lay, pat, l, t):
    d0, d1, d2 = d
    s1 = lay[1]
    if pat == 0:
        j, i = divmod(l, d2)
        return kofs(lay, t) + j * s1 + i
    if pat == 1:
        k, i = divmod(l, d2)
        return kofs(lay, k) + t * s1 + i
    if pat == 7:
        k, i = pair_coords(l, d0, d2)
        return kofs(lay, k) + t * s1 + i
    if pat == 4:
        i, k = divmod(l, d0)
        return kofs(lay, k) + t * s1 + i
    if pat == 2:
        k, j = divmod(l, d1)
    elif pat == 5:
        j, k = divmod(l, d0)
    else:
        k, j = pair_coords(l, d0, d1)
    return kofs(lay, k) + j * s1 + t


def cost(d, lay, pats, epb, ebuf):
    """Modelled wavefronts; a pattern may carry a weight, (pattern, accesses
    per element relative to one pass)."""
    total = 0
    for pw in pats:
        pat, w = pw if isinstance(pw, tuple) else (pw, 1)
        nl, ln = lines(d, pat)
        tot_lines = nl * epb
        for w0 in range(0, tot_lines, 32):
            for t in range(ln):
                for h in (0, 16):
                    words = set()
                    for g in range(w0 + h, min(w0 + h + 16, tot_lines)):
                        e, l = divmod(g, nl)
                        words.add(e * ebuf + addr(d, lay, pat, l, t))
                    if not words:
                        continue
                    cnt = [0] * 16
                    for a in words:
                        cnt[a & 15] += 1
                    total += w * max(cnt)
    return total


def extent(d, lay):
    """Doubles spanned by one element's tensor under `lay`."""
    d0, d1, d2 = d
    return kofs(lay, d0 - 1) + (d1 - 1) * lay[1] + d2


_CACHE_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "build", "layout_cache.json")
_cache = None


def best_layout(d, pats, paired=False, wide=False):
    """Cheapest layout for one tensor phase (memoised in build/ -- the paired
    search evaluates ~1000 candidates)."""
    global _cache
    if _cache is None:
        try:
            with open(_CACHE_PATH) as fh:
                _cache = json.load(fh)
        except (OSError, ValueError):
            _cache = {}
    key = repr((tuple(d), tuple(pats), bool(paired))) + (" wide" if wide else "")
    if key not in _cache:
        _cache[key] = list(_best_layout(d, pats, paired, wide))
        os.makedirs(os.path.dirname(_CACHE_PATH), exist_ok=True)
        with open(_CACHE_PATH, "w") as fh:
            json.dump(_cache, fh)
    return tuple(_cache[key])


def _best_layout(d, pats, paired=False, wide=False):
    """wide: row strides up to d2 + 16 (BP1.0's Y needs s1 = 1 mod 16 with
    c-fastest j-lines, i.e. 17 at N=7; registers, not shared memory, bound
    its occupancy)."""
    d0, d1, d2 = d
    best = None
    for s1 in range(d2, d2 + (17 if wide else 4)):
        if not paired:
            cands = ((s0, s1, 0) for s0 in range(d1 * s1, d1 * s1 + 16))
        else:
            cands = ((s0, s1, sq) for sq in range(d1 * s1, d1 * s1 + 16)
                     for s0 in range(sq + d1 * s1, sq + d1 * s1 + 16))
        for lay in cands:
            c = cost(d, lay, pats, 1, 0)
            key = (c, extent(d, lay))
            if best is None or key < best[0]:
                best = (key, lay)
    return best[1]


def phases(bp, n, m, ord_=0):
    """(buffer id, dims, patterns) for every tensor phase of a kernel."""
    if bp == BP35:
        # A: S1 / S3 / S5 k-lines (0), S2 j-lines and i-lines; B: S2 / S4
        # i-lines; C: S2 / S4 j-lines.  ORD: lane order over (k, r) in S2 / S4
        # -- 0 r fastest (j-lines 1, i-lines 2), 2 k fastest (4, 5), 4
        # k-paired (7, 6)
        pj, pi = {0: (1, 2), 2: (4, 5), 4: (7, 6)}[ord_ & 6]
        return [(0, (n, n, n), (0, pj, pi)), (1, (n, n, n), (0, pi)),
                (2, (n, n, n), (0, pj))]
    if bp == BP1:
        # t-first stage order (hx_bp1.cu): X = (m, n, n) after the t
        # interpolation, read / written as k-lines by the HBM stages (pattern
        # 0: coalesced q loads and out stores) and as j-lines by S2 / S4;
        # Y = (m, m, n), j-lines and i-lines (S3, lanes (c, b) b fastest: the
        # GwJ loads of S3 are coalesced over that order).  ORD: lane order of
        # the j-line stages: 0 i fastest (pattern 1), 2 c fastest (4), 4
        # c-paired (7, with c-paired layouts).  With c fastest the address of
        # line L is congruent to a multiple of L mod 16 in every stage when
        # X = (73, 8) and Y = (153, 17) at N=7 (ncu r2_03: the i-fastest /
        # c-paired orders left 1.7x wavefronts in S3 or in S2 / S4).
        # ORD bit 8 (BP1_CFAST degrees): S3's lanes run c-fastest (pattern 5)
        # and the packed GwJ slot is stored (i, j, k) so its loads stay
        # contiguous -- with even m an even Y row stride otherwise leaves
        # the i-line starts on every other bank pair (model N=8: 1.71x).
        pj = {0: 1, 2: 4, 4: 7}[ord_ & 7]
        return [(0, (m, n, n), (0, pj)), (1, (m, m, n), (pj, 5 if ord_ & 8 else 2))]
    if bp == INTERP:
        # ORD: lane order of the i-line stages (S2, S4): 0 a fastest (pattern
        # 2), 2 k fastest (5), 4 k-paired (6, with k-paired layouts).  The
        # j-line and k-line stages also touch HBM and keep their coalesced
        # orders (k fastest there doubles the L1 tag requests: ncu r09).
        pi = {0: 2, 2: 5, 4: 6}[ord_]
        return [(0, (n, m, n), (1, pi)), (1, (n, m, m), (0, pi))]
    # BP3.0: ORD 4 = k-paired lane order in the i-line stages over the
    # (n, m, .) tensors (S2, S8: pattern 6).  The (m, m, m) stages S4 / S6 keep
    # theirs: with odd m the unpaired last slice costs more than it saves
    # (r11: 1.3-1.5x wavefronts there with pattern 6 / 7).
    # ORD bit 8: the i-line halves of S4 / S6 (over the (m, m, m) tensors T
    # and QR) enumerate their lines k-fastest (pattern 5): with even m an
    # even row stride confines i-line starts to every other bank pair, and
    # k-fastest lanes spread them again (model: N=8 1.28x -> 1.16x).
    pi = 6 if ord_ & 4 else 2
    pm = 5 if ord_ & 8 else 2
    if n - 1 in BP3_WEIGHTED:
        # patterns weighted by the passes each tensor sees (hx_bp3.cu): X is
        # written in S1 and S8, read in S2 and S9; QR / QS are read and
        # written by S5, read by S7 (k-lines) and touched three times by
        # S4 / S6 (i- resp. j-lines); T is written by S3 and read by S4 both
        # ways and by S5 (with ACCS also re-read, rewritten twice and read
        # by S7 -- ACCS degrees are searched jointly with Z, see plan())
        wt = 7 if n - 1 in BP3_ACCS else 2
        return [(0, (n, m, n), ((1, 2), (pi, 2))), (0, (m, m, m), ((0, 3), (pm, 3))),
                (1, (n, m, m), ((0, 1), (pi, 1))), (1, (m, m, m), ((0, 3), (1, 3))),
                (2, (m, m, m), ((0, wt), (1, 1), (pm, 1))), (2, (n, m, m), ((0, 1), (pi, 1)))]
    return [(0, (n, m, n), (1, pi)), (0, (m, m, m), (0, pm)),
            (1, (n, m, m), (0, pi)), (1, (m, m, m), (0, 1)),
            (2, (m, m, m), (0, 1, pm)), (2, (n, m, m), (0, pi))]


def q_stage_stride(n):
    """Slab stride (doubles) of BP1.0's TMA-staged q tile: every k-slab
    (n*n doubles, contiguous in HBM) is one bulk copy, so rows stay dense
    (s1 = n) and only the slab stride is free; it must keep 16-byte alignment
    (even) and S1 reads j-lines (pattern 1).  0 when n*n*8 is not a multiple
    of 16 (odd n): the bulk engine needs 16-byte sizes and addresses."""
    if n % 2:
        return 0
    d = (n, n, n)
    best = None
    for s0 in range(n * n, n * n + 16, 2):
        c = cost(d, (s0, n, 0), (1,), 1, 0)
        if best is None or c < best[0]:
            best = (c, s0)
    return best[1]


def plan(bp, deg, target=TARGET_THREADS, qstage=False):
    n, m = deg + 1, deg + 2
    lmax = n * n if bp == BP35 else m * m
    epb = max(1, target // lmax)
    nt = -(-epb * lmax // 32) * 32
    if bp in (BP1, INTERP) and target < lmax and target <= 128:
        # BP1.0 only: a CTA smaller than one element's line count walks over
        # the lines (for_lines); one element per tile
        nt = max(32, -(-target // 32) * 32)
    # BP3.0: ORD 4 only for the BP3_ORD4 degrees (N=7: +0.2 %, r2_59; round
    # 1 measured it 1-2 % slower, r11/r12), ORD 8 for BP3_KI
    ords = {BP1: (0, 2, 4), INTERP: (0, 2, 4)}.get(bp, (0,))
    if bp == BP3 and m % 2 == 0 and deg in BP3_KI:
        ords = (0, 8)
    if bp == BP3 and deg in BP3_ORD4:
        ords = ords + tuple(o | 4 for o in ords)
    if bp == BP35 and deg in BP35_ORD:
        ords = (0, 2, 4)
    if bp == BP1 and deg in BP1_CFAST:
        ords = ords + tuple(o | 8 for o in ords)
    best = None
    for o in ords:  # BP1.0: lane orders chosen jointly with the strides
        ph_o = phases(bp, n, m, o)
        lays_o = [best_layout(d, pats, paired=(6 in pats or 7 in pats), wide=(bp == BP1))
                  for _, d, pats in ph_o]
        c = sum(cost(d, lay, pats, 1, 0) for (_, d, pats), lay in zip(ph_o, lays_o))
        if best is None or c < best[0]:
            best = (c, o, ph_o, lays_o)
    _, ord_, ph, lays = best
    accs = int((bp == BP3 and deg in BP3_ACCS) or (bp == BP35 and deg in BP35_LEAN))
    ser = int(bp == BP3 and deg in BP3_SER)
    if accs and bp == BP3:
        lays = list(lays)
        if deg in BP3_WEIGHTED:
            # one layout for T and Z (Z written in place over T's k-lines)
            (_, dt, pt), (_, dz, pz) = ph[4], ph[5]
            d0, d1, d2 = dt
            cands = [(s0_, s1_, 0) for s1_ in range(d2, d2 + 4)
                     for s0_ in range(d1 * s1_, d1 * s1_ + 16)]
            lays[4] = min(cands, key=lambda l: (cost(dt, l, pt, 1, 0) + cost(dz, l, pz, 1, 0),
                                                extent(dt, l)))
        lays[5] = lays[4]  # Z written in place over T's k-lines
    nbuf = 1 + max(b for b, _, _ in ph)
    base = [0] * nbuf
    for (b, d, _), lay in zip(ph, lays):
        base[b] = max(base[b], max(extent(d, lay), d[0] * lay[0] if lay[2] == 0 else 0))
    qs = q_stage_stride(n) if (bp == INTERP and qstage) else 0
    # keep the tile inside the 227 KB shared-memory limit
    while epb > 1 and epb * (sum(base) + 16 * nbuf + n * qs) * 8 > 227 * 1024:
        epb -= 1
        nt = -(-epb * lmax // 32) * 32
    ebufs = []
    for b in range(nbuf):
        best = None
        for eb in range(base[b], base[b] + 16):
            c = sum(cost(d, lay, pats, epb, eb)
                    for (bb, d, pats), lay in zip(ph, lays) if bb == b)
            if best is None or c < best[0]:
                best = (c, eb)
        ebufs.append(best[1])
    return n, m, epb, nt, ph, lays, ebufs, qs, ord_, accs, ser


def min_blocks(bp, deg):
    """Second __launch_bounds__ argument (register budget).  Measured at N=7
    (gpurun sweeps sw01-sw03): BP3.5 and BP3.0 are fastest at 2 resident CTAs
    of 256 threads (<=128 registers); letting the compiler take ~160-200
    registers (1 CTA/SM) or squeezing to 3 CTAs/SM (spills) both lose 7-15 %.
    BP1.0 needs only ~60 registers and is left to the compiler."""
    if bp in (BP35, BP3) and deg <= 8:
        return 2
    return 1


def main(path, policy=None, verbose=False):
    """policy: {(bp, deg): (target_threads, min_blocks, qstage)}; defaults otherwise."""
    policy = policy or {}
    out = ["// Generated by tools/gen_layouts.py -- do not edit by hand.",
           "// Shared-memory strides per (kernel, degree): see that script for the",
           "// bank model.  Phase order follows the kernels' stage order.",
           "#pragma once", "", "namespace hx {", "",
           "// element (k, j, i) of a staged tensor lives at kofs(k) + j*s1 + i with",
           "// kofs(k) = k*s0, or (k/2)*s0 + (k%2)*sq for a k-paired layout (sq > 0)",
           "struct Lay {",
           "  int s0, s1, sq;",
           "  __host__ __device__ constexpr int kofs(int k) const {",
           "    return sq == 0 ? k * s0 : (k >> 1) * s0 + (k & 1) * sq;",
           "  }",
           "};", "",
           "template <int BP, int N> struct Cfg;", ""]
    for bp in (BP1, BP35, BP3, INTERP):
        for deg in range(1, 16):
            # the element helpers keep the shape policy tuned for the BP1.0
            # stage structure they share
            pol = policy.get((bp, deg)) or (policy.get((BP1, deg)) if bp == INTERP else None)
            target, minb, qst = pol or (TARGET_THREADS, min_blocks(bp, deg), 0)
            n, m, epb, nt, ph, lays, ebufs, qs, ord_, accs, ser = plan(bp, deg, target, bool(qst))
            out.append(f"template <> struct Cfg<{bp}, {deg}> {{")
            out.append(f"  static constexpr int EPB = {epb}, NT = {nt}, MINB = {minb};")
            out.append(f"  static constexpr int QS = {qs};  // TMA q-staging slab stride (0: off)")
            out.append(f"  static constexpr int ORD = {ord_};  // lane order (gen_layouts.phases): 0 default, 2 k-fast, 4 paired")
            out.append(f"  static constexpr int ACCS = {accs}, SER = {ser};  // BP3.0: S5 accumulator via shared memory (Z aliases T); serial S4/S6 lines")
            out.append("  static constexpr int EBUF[%d] = {%s};" % (
                len(ebufs), ", ".join(str(e) for e in ebufs)))
            out.append("  static constexpr Lay L[%d] = {%s};" % (
                len(lays), ", ".join("{%d, %d, %d}" % l for l in lays)))
            out.append("};")
            if verbose:
                sys.stderr.write(f"bp={bp} N={deg} epb={epb} nt={nt} ebuf={ebufs} lays={lays}\n")
    out += ["", "}  // namespace hx", ""]
    with open(path, "w") as fh:
        fh.write("\n".join(out))


def load_policy(path):
    """JSON list of [bp, deg, target_threads, min_blocks(, qstage)]
    (tools/tune_policy.json)."""
    import json
    with open(path) as fh:
        return {(int(r[0]), int(r[1])): (int(r[2]), int(r[3]), int(r[4]) if len(r) > 4 else 0)
                for r in json.load(fh)}


if __name__ == "__main__":
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    pol = os.path.join(here, "tune_policy.json")
    main(sys.argv[1] if len(sys.argv) > 1 else
         "paper_1711_00903_b200/csrc/hx_layouts.h",
         load_policy(sys.argv[2]) if len(sys.argv) > 2 else
         (load_policy(pol) if os.path.exists(pol) else None))
