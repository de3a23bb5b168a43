"""Reporting integration: GPU timings in the JSON/CSV
schema of the reference's ``hexbench bench`` / ``hexbench roofline``
(cli.py:235-347), so tooling built on those reports keeps working.

    python -m paper_1711_00903_b200.report bench --bp 3.5 --degrees 7 --elements 32
    python -m paper_1711_00903_b200.report roofline --bp 1.0 --degrees 1..15 --elements 16
    python -m paper_1711_00903_b200.report calibrate --bytes 1073741824

Differences from the reference, all additive: ``wall_time_*`` are CUDA-event
times of device-resident applies, ``bandwidth_bytes_per_s`` is the measured
device copy bandwidth at the run's copy-equivalent size (``--bandwidth``
overrides), and the scratch roofline uses the measured shared-memory
bandwidth instead of the P100 ansatz; extra keys (``gdof_per_s``,
``achieved_bytes_per_s``, ``frac_of_bandwidth``, ``device``) ride along.
"""

import argparse
import csv
import json
import statistics
import sys

from . import perf

_BP_FLAG = {"1.0": perf.BP1, "3.5": perf.BP35, "3.0": perf.BP3}


def _degrees(text):
    if ".." in text:
        lo, hi = (int(x) for x in text.split(".."))
    else:
        lo = hi = int(text)
    if not 1 <= lo <= hi <= 15:
        raise argparse.ArgumentTypeError("--degrees must lie within 1..15")
    return list(range(lo, hi + 1))


def _spacer():
    """Queue ~100 us of GPU work before a timed launch so host launch latency
    is not timed (see bench.gpu_spacer)."""
    import torch
    torch.cuda._sleep(200_000)


def device_copy_bandwidth(nbytes, trials=10):
    """Mean read+write bandwidth of a D2D copy of nbytes."""
    import torch
    n = max(1, nbytes // 8)
    a = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    rates = []
    for _ in range(trials):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _spacer()
        s.record()
        b.copy_(a)
        e.record()
        e.synchronize()
        rates.append(2 * n * 8 / (s.elapsed_time(e) * 1e-3))
    return sum(rates) / len(rates)


def device_smem_bandwidth():
    import ctypes
    import torch
    from . import _native
    v = ctypes.c_double()
    _native.check(_native.lib().hx_measure_smem_bandwidth(
        ctypes.byref(v), torch.cuda.current_stream().cuda_stream))
    return v.value


def bench_runs(bps, degrees, side, variant="fused", lam=1.0, repeats=10, seed=0,
               bandwidth=None, perturb=False):
    """One reference-schema run entry per (bp, degree) (cli.py:262-284)."""
    import torch
    from .mesh import build_cube_mesh, perturb_mesh
    from .operators import AccessCounters, FieldVector, apply_device, make_operator, _charge

    mesh = build_cube_mesh(side, 2.0)
    if perturb:
        mesh = perturb_mesh(mesh, seed=seed)
    b_sh = device_smem_bandwidth()
    runs = []
    for bp in bps:
        for deg in degrees:
            op = make_operator(bp, deg, mesh, lam=lam, variant=variant)
            q = FieldVector.random(mesh.n_el, op.n_p, seed=seed).to_device().data
            out = torch.empty_like(q)
            apply_device(op, q, out)  # warm-up (cli.py:253)
            torch.cuda.synchronize()
            times = []
            for _ in range(repeats):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                _spacer()
                s.record()
                apply_device(op, q, out)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e) * 1e-3)
            counters = AccessCounters()
            _charge(op, counters)
            model = perf.traffic(bp, deg, mesh.n_el)
            b_gl = bandwidth if bandwidth is not None else \
                device_copy_bandwidth(model.copy_equivalent_bytes)
            med = statistics.median(times)
            nbytes = model.bytes_per_element * mesh.n_el
            entry = {
                "bp": bp, "degree": deg, "variant": variant, "elements": mesh.n_el,
                "wall_time_mean_s": sum(times) / len(times), "wall_time_median_s": med,
                "achieved_flops_per_s": counters.flops / med, "flops": counters.flops,
                "counted_global_bytes": counters.global_reads + counters.global_writes,
                "counted_scratch_bytes": counters.scratch_reads + counters.scratch_writes,
                "model_bytes": nbytes, "syncs": counters.syncs,
                "bandwidth_bytes_per_s": b_gl,
                "r_global_flops_per_s": perf.roofline_global(
                    b_gl, counters.flops, 8 * model.reads_doubles * mesh.n_el,
                    8 * model.writes_doubles * mesh.n_el),
                "gdof_per_s": mesh.n_el * op.n_p / med / 1e9,
                "achieved_bytes_per_s": nbytes / med,
                "frac_of_bandwidth": nbytes / med / b_gl,
                "shared_bandwidth_bytes_per_s": b_sh,
            }
            if bp != perf.BP35:
                entry["r_shared_flops_per_s"] = perf.roofline_shared(
                    b_sh, counters.flops, counters.scratch_reads, counters.scratch_writes)
            runs.append(entry)
            del op, q, out
            torch.cuda.empty_cache()
    return runs


def _machine():
    import platform
    import torch
    return f"{platform.platform()} / {torch.cuda.get_device_name(0)}"


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_1711_00903_b200.report")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, deg_default in (("bench", "7"), ("roofline", "1..15")):
        p = sub.add_parser(name)
        p.add_argument("--bp", choices=["1.0", "3.5", "3.0", "all"], default="all")
        p.add_argument("--degrees", type=_degrees, default=_degrees(deg_default))
        p.add_argument("--elements", type=int, default=8, help="elements per cube side")
        p.add_argument("--variant", choices=["baseline", "fused", "symfused"], default="fused")
        p.add_argument("--lambda", dest="lam", type=float, default=1.0)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--repeats", type=int, default=10)
        p.add_argument("--bandwidth", type=float, default=None, help="GB/s (else measured)")
        p.add_argument("--out", default=None)
        p.add_argument("--format", choices=["json", "csv"], default="json")
    p = sub.add_parser("calibrate")  # cli.py:85-88, 350-366
    p.add_argument("--bytes", type=int, default=1 << 27)
    p.add_argument("--repeats", type=int, default=10)
    p.add_argument("--out", default=None)
    p.add_argument("--format", choices=["json", "csv"], default="json")
    args = ap.parse_args(argv)
    if args.command == "calibrate":
        try:
            cal = perf.measure_stream_bandwidth(args.bytes, trials=args.repeats)
        except (MemoryError, ValueError) as exc:
            print(f"error: {exc}", file=sys.stderr)
            return 3 if isinstance(exc, MemoryError) else 2  # EXIT_RESOURCE / EXIT_USAGE
        payload = {"command": "calibrate", "bytes": cal.bytes_transferred,
                   "trial_times_s": cal.trial_times, "mean_bytes_per_s": cal.mean_bandwidth,
                   "theoretical_peak_bytes_per_s": cal.theoretical_peak, "machine": _machine()}
        header = ("trial", "time_s", "bytes_per_s")
        rows = [(i, t, cal.bytes_transferred / t) for i, t in enumerate(cal.trial_times)]
        return _emit(payload, header, rows, args)
    bps = list(perf.BENCHMARKS) if args.bp == "all" else [_BP_FLAG[args.bp]]
    bw = None if args.bandwidth is None else args.bandwidth * 1e9
    if args.command == "bench":
        runs = bench_runs(bps, args.degrees, args.elements, args.variant, args.lam,
                          args.repeats, args.seed, bw)
        payload = {"command": "bench",
                   "config": {"bp": args.bp, "degrees": args.degrees, "elements": args.elements,
                              "variant": args.variant, "lambda": args.lam,
                              "repeats": args.repeats, "seed": args.seed, "device": "cuda"},
                   "measured_bandwidth": None, "runs": runs, "machine": _machine()}
        header = ("bp", "degree", "variant", "elements", "wall_time_median_s",
                  "achieved_flops_per_s", "flops", "counted_global_bytes", "model_bytes",
                  "r_global_flops_per_s", "gdof_per_s", "frac_of_bandwidth")
        rows = [tuple(r.get(k) for k in header) for r in runs]
    else:
        n_el = args.elements ** 3
        b_gl = bw if bw is not None else device_copy_bandwidth(1 << 30)
        b_sh = device_smem_bandwidth()
        series = [perf.roofline_series(bp, args.degrees, n_el, b_gl, args.variant, b_sh)
                  for bp in bps]
        payload = {"command": "roofline", "n_el": n_el, "B_gl": b_gl, "B_sh": b_sh,
                   "series": [{"bp": s.bp, "points": [p.__dict__ for p in s.points]}
                              for s in series]}
        header = ("bp", "N", "F", "bytes", "R_global", "R_shared")
        rows = [(s.bp, p.degree, p.flops, p.bytes_moved, p.r_global, p.r_shared)
                for s in series for p in s.points]
    return _emit(payload, header, rows, args)


def _emit(payload, header, rows, args):
    if args.format == "csv":
        fh = sys.stdout if args.out is None else open(args.out, "w", newline="")
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)
        if args.out is not None:
            fh.close()
    else:
        text = json.dumps(payload, indent=2)
        if args.out is None:
            print(text)
        else:
            with open(args.out, "w") as fh:
                fh.write(text + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
