#!/usr/bin/env python3
"""Latency anatomy of small applies (BASELINE config 1 is BP1.0 at E=4096):
time one apply for a range of element counts, L2-resident (back to back) and
with a 512 MB L2 flush before each launch.  One JSON line per (bp, E).

    python tools/small_e.py [bp] [E ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402


def main():
    bp = sys.argv[1] if len(sys.argv) > 1 else hx.BP1
    sizes = [int(x) for x in sys.argv[2:]] or [148, 444, 592, 1184, 1776, 2368, 3552, 4096,
                                                5328, 8192, 16384, 32768]
    big = hx.perturb_mesh(hx.build_cube_mesh(32, 2.0), amplitude=0.15, seed=7)
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    for n_el in sizes:
        mesh = hx.HexMesh(n_el, big.vertices[:n_el], big.extent)
        op = hx.make_operator(bp, 7, mesh, lam=1.0)
        q = torch.randn(n_el, op.n_p, dtype=torch.float64, device="cuda")
        out = torch.empty_like(q)
        res = {"bp": bp, "n_el": n_el}
        for mode in ("hot", "flushed"):
            times = []
            for it in range(25):
                if mode == "flushed":
                    flush.zero_()
                else:
                    torch.cuda._sleep(200_000)  # spacer: keep launch latency out
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                hx.apply_device(op, q, out)
                e.record()
                e.synchronize()
                if it >= 5:
                    times.append(s.elapsed_time(e) * 1e3)
            res[f"{mode}_us"] = statistics.median(times)
        nbytes = hx.traffic(bp, 7, n_el).bytes_per_element * n_el
        res["flushed_gb_per_s"] = nbytes / res["flushed_us"] / 1e3
        res["shape"] = {"epb": op.plan.elements_per_tile, "threads": op.plan.threads}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
