#!/usr/bin/env python3
"""Benchmark harness: GDOF/s and % of the empirical HBM roofline for the
BP1.0 / BP3.5 / BP3.0 FP64 element matvecs at N=7 (BASELINE.json metric).

One *step* = one apply of the operator over the whole synthetic element
batch resident in HBM.  Headline workload (N=1): BASELINE configs[1], BP3.5
N=7 E=32768 -- 1.21 GB of algorithmic traffic per apply, so the inputs are
larger than L2 between timed iterations.  BP1.0 (config 1, E=4096, 57 MB)
and BP3.0 (config 3, E=32768) are reported under ``per_bp``; the L2-resident
BP1.0 config is timed with an L2 flush before every apply.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL).  Each rank owns
its own E-element shard (weak scaling, no data-path collective); the
reported time is the max over ranks.  The JSON line ends with the compact
per-config ``per_bp`` table; the full secondary legs (CG, unfused baseline,
calibrations, host paths) go to gpurun_out/bench_details.json.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDOF/s and % empirical HBM roofline, BP1.0/3.5/3.0 FP64 N=7, 1/2/4/8 B200"
DEGREE = 7
LAM = 1.0
HEADLINE = ("BP3.5", 32)          # configs[1]: side 32 -> E = 32768
EXTRA = (("BP1.0", 16), ("BP3.0", 32), ("BP1.0", 32))
SAMPLE_EL = 2048                  # CPU-baseline sample of the oracle port (elements)
REF_SAMPLE_EL = 512               # ... of the reference itself (0.15 s per BP3.5 apply)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")  # pip-installed reference (hexbench)
DETAILS = os.path.join(ROOT, "gpurun_out", "bench_details.json")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every ~1 ms in a thread (the timed region of the headline is a few ms),
    nvidia-smi -lms 100 when NVML is unavailable."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons) from NVML
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(handle, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(handle, pynvml.NVML_CLOCK_SM)
                    mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(handle)
                    self.samples.append((sm, max_mhz, {r for r, b in bits.items() if mask & b}))
                    time.sleep(0.001)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # no NVML: fall back to nvidia-smi
            self.samples = []
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is None:
            self.stop.set()
            if self.thread is not None:
                self.thread.join(timeout=2)
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for s_mhz, m_mhz, rs in self.samples:
            sm.append(float(s_mhz))
            mx.append(float(m_mhz))
            reasons |= rs
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 2 + len(REASONS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for r, v in zip(REASONS, parts[2:]):
                if v.lower() == "active":
                    reasons.add(r)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one "
                         "rank per GPU (bench.py re-launches itself when WORLD_SIZE is unset)")
    # one rank per GPU; HX_BENCH_BACKEND=gloo (test only) lets several ranks
    # share one GPU to exercise the multi-rank code paths on a one-GPU box
    backend = os.environ.get("HX_BENCH_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if world > 1 and backend == "nccl" and world > ndev:
        raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, this node has {ndev}")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, ndev)
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (one per GPU, NCCL with
    its INIT log on so the communicator's N ranks are visible) and exit with
    its status.  Only rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def _reduce_device():
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value, world):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value, world):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def build_operator(bp, side, rank):
    import paper_1711_00903_b200 as hx

    mesh = hx.perturb_mesh(hx.build_cube_mesh(side, 2.0), amplitude=0.15, seed=7 + rank)
    op = hx.make_operator(bp, DEGREE, mesh, lam=LAM)
    return mesh, op


def gpu_spacer(flush=None):
    """Queue GPU work ahead of a timed launch so the start event is not
    reached before the host has enqueued the launch: a launch-latency gap
    (~10-20 us of Python + ctypes) would otherwise be timed as kernel time
    for the small configs.  With `flush` (a > L2 buffer) the spacer also
    evicts L2."""
    import torch

    if flush is not None:
        flush.add_(1.0)
    else:
        torch.cuda._sleep(200_000)  # ~100 us of GPU spin


def copy_bandwidth(nbytes, trials=10, flush=None):
    """Paper's empirical roofline: D2D copy of copy_equivalent_bytes, one
    warm-up, mean of `trials`; read+write bytes counted.
    Each trial is preceded by a GPU spacer (and an L2 flush when the kernel
    it calibrates was timed flushed), so host launch latency and L2 residency
    do not inflate or deflate the calibration."""
    import torch

    n = max(1, nbytes // 8)
    a = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    rates = []
    for _ in range(trials):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gpu_spacer(flush)
        s.record()
        b.copy_(a)
        e.record()
        e.synchronize()
        rates.append(2 * n * 8 / (s.elapsed_time(e) * 1e-3))
    del a, b
    return float(np.mean(rates)), float(np.max(rates))


def time_back_to_back(op, q, out, steps, warmup, reps=3):
    """ms per apply of `steps` applies queued back to back between one
    start and one stop event (best of `reps` runs): a stream of applies --
    the device path launches them as programmatic dependent launches, so one
    kernel's retiring CTAs overlap the next one's start.  Only for inputs
    larger than L2 (nothing is reused between applies)."""
    import torch
    import paper_1711_00903_b200 as hx

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gpu_spacer()
        s.record(stream)
        for _ in range(steps):
            hx.apply_device(op, q, out)
        e.record(stream)
        e.synchronize()
        ms = s.elapsed_time(e) / steps
        best = ms if best is None else min(best, ms)
    return best


def copy_bandwidth_back_to_back(nbytes, steps=20, reps=3):
    """The same-size D2D copy calibration for back-to-back timings: `steps`
    copies between one start and one stop event, best of `reps`."""
    import torch

    n = max(1, nbytes // 8)
    a = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    best = None
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gpu_spacer()
        s.record()
        for _ in range(steps):
            b.copy_(a)
        e.record()
        e.synchronize()
        rate = 2 * n * 8 / (s.elapsed_time(e) / steps * 1e-3)
        best = rate if best is None else max(best, rate)
    del a, b
    return best


def time_applies(op, q, out, steps, warmup, flush=None):
    """Per-launch CUDA-event times (ms) on the launching stream."""
    import torch
    import paper_1711_00903_b200 as hx

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        gpu_spacer(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        hx.apply_device(op, q, out)
        e.record(stream)
        times.append((s, e))
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in times]


def bp_report(bp, side, rank, steps, warmup, hbm_peak):
    import torch
    import paper_1711_00903_b200 as hx

    mesh, op = build_operator(bp, side, rank)
    q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
    out = torch.empty_like(q)
    t = hx.traffic(bp, DEGREE, mesh.n_el)
    bytes_per_apply = t.bytes_per_element * mesh.n_el
    flops = hx.flop_model(bp, "fused", DEGREE) * mesh.n_el
    l2_resident = bytes_per_apply < 256e6
    flush = torch.zeros(64 << 20, dtype=torch.float64, device="cuda") if l2_resident else None
    ms = time_applies(op, q, out, steps, warmup, flush)
    single_med = statistics.median(ms)
    mean = statistics.mean(ms)
    b_copy_mean, b_copy_best = copy_bandwidth(t.copy_equivalent_bytes, flush=flush)
    single = {"kernel_ms_median": single_med,
              "frac_of_measured_peak": bytes_per_apply / (single_med * 1e-3) / 1e9 / hbm_peak,
              "frac_of_copy_same_size": bytes_per_apply / (single_med * 1e-3) / b_copy_mean}
    if l2_resident:  # config 1: each apply after an L2 flush, one launch at a time
        med, timing = single_med, "single launches, L2 flushed before each"
    else:            # a stream of applies, as in the headline
        med = time_back_to_back(op, q, out, max(steps, 10), warmup)
        b_copy_mean = copy_bandwidth_back_to_back(t.copy_equivalent_bytes)
        timing = "back to back (one event pair around the applies)"
    rep = {
        "bp": bp, "degree": DEGREE, "n_el": mesh.n_el, "lam": LAM,
        "timing": timing, "single_launch": single,
        "kernel_ms_median": med, "kernel_ms_mean": mean,
        "gdof_per_s": mesh.n_el * op.n_p / (med * 1e-3) / 1e9,
        "gflop_per_s": flops / (med * 1e-3) / 1e9,
        "achieved_gb_per_s": bytes_per_apply / (med * 1e-3) / 1e9,
        "bytes_per_apply": bytes_per_apply,
        "frac_of_measured_peak": bytes_per_apply / (med * 1e-3) / 1e9 / hbm_peak,
        "b_copy_same_size_gb_per_s": b_copy_mean / 1e9,
        "b_copy_same_size_best_gb_per_s": b_copy_best / 1e9,
        "frac_of_copy_same_size": bytes_per_apply / (med * 1e-3) / b_copy_mean,
        "l2": "flushed before every apply" if l2_resident else "inputs larger than L2",
        "threads": op.plan.threads, "elements_per_tile": op.plan.elements_per_tile,
        "smem_bytes": op.plan.smem_bytes,
    }
    if l2_resident:
        hot = time_applies(op, q, out, steps, warmup, None)
        rep["l2_resident_back_to_back_gdof_per_s"] = \
            mesh.n_el * op.n_p / (statistics.median(hot) * 1e-3) / 1e9
    del op, q, out, flush
    torch.cuda.empty_cache()
    return rep


def port_cpu(sample_el=SAMPLE_EL, bp=HEADLINE[0], seconds=5.0):
    """Oracle port (numpy restatement of the reference apply) on a bounded
    sample of the headline workload, BLAS pinned to one thread."""
    import paper_1711_00903_b200 as hx
    from oracle import hexbench_oracle as orc
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None

    mesh = hx.perturb_mesh(hx.build_cube_mesh(HEADLINE[1], 2.0), amplitude=0.15, seed=7)
    sub = hx.HexMesh(sample_el, mesh.vertices[:sample_el], mesh.extent)
    rule = hx.gll_rule(DEGREE + 1) if bp == "BP3.5" else hx.gl_rule(DEGREE + 2)
    fac = hx.geometric_factors(sub, rule).data
    q = np.random.default_rng(0).standard_normal((sample_el, (DEGREE + 1) ** 3))
    interp = hx.interp_matrix(DEGREE).entries
    diff = (hx.diff_matrix_gll if bp == "BP3.5" else hx.diff_matrix_gl)(DEGREE).entries
    ctx = threadpool_limits(1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    try:
        orc.apply_chunked(bp, DEGREE, LAM, interp, diff, fac, q)
        reps, t0 = 0, time.perf_counter()
        while True:
            orc.apply_chunked(bp, DEGREE, LAM, interp, diff, fac, q)
            reps += 1
            el = time.perf_counter() - t0
            if el > seconds or reps >= 200:
                break
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    return {"value": sample_el * q.shape[1] / (el / reps) / 1e9, "unit": "GDOF/s", "cores": 1,
            "kind": "port",
            "sample": f"{bp} N={DEGREE} first {sample_el} elements of the E=32768 mesh, "
                      f"{reps} applies in {el:.1f} s (oracle/hexbench_oracle.py, numpy, "
                      "1 BLAS thread)"}


def reference_available():
    return os.path.isdir(os.path.join(REF_PATH, "hexbench"))


class ReferenceWorkload:
    """The unmodified reference package (pip-installed into baseline/_ref by
    tools/install_reference.sh) on a bounded sample of the headline mesh:
    its own HexMesh / make_operator / FieldVector / apply_operator
    (operators.py:118-143, :306-331), threads = the reference's own
    element-range thread pool.  The sample's corners are the first
    `sample_el` elements of perturb_mesh(build_cube_mesh(32, 2.0), 0.15,
    seed=7) -- built with this package's mesh module, which reproduces the
    reference's bit for bit (tests/test_oracle_golden.py), because the
    reference's own perturb_mesh of all 32768 elements alone takes minutes."""

    def __init__(self, sample_el, bp=HEADLINE[0]):
        import paper_1711_00903_b200 as hx
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        from hexbench import mesh as rmesh
        from hexbench import operators as rops
        full = hx.perturb_mesh(hx.build_cube_mesh(HEADLINE[1], 2.0), amplitude=0.15, seed=7)
        sub = rmesh.HexMesh(sample_el, np.array(full.vertices[:sample_el]), full.extent)
        self.rops = rops
        self.bp, self.sample_el = bp, sample_el
        self.op = rops.make_operator(bp, DEGREE, sub, lam=LAM)
        self.q = rops.FieldVector.random(sample_el, self.op.n_p, seed=0)
        self.dofs = sample_el * self.op.n_p

    def step(self, threads):
        self.rops.apply_operator(self.op, self.q, threads=threads)

    def rate(self, threads, seconds=3.0, min_reps=2):
        self.step(threads)  # warm-up
        reps, t0 = 0, time.perf_counter()
        while True:
            self.step(threads)
            reps += 1
            el = time.perf_counter() - t0
            if el > seconds and reps >= min_reps:
                break
        return self.dofs / (el / reps) / 1e9, reps, el


def reference_cpu(seconds=3.0):
    """cpu_baseline of our arm: the reference itself at threads=1 and
    threads=<host cores> on REF_SAMPLE_EL elements, plus the oracle port
    (one core).  Falls back to the port alone without baseline/_ref."""
    port = port_cpu(seconds=seconds)
    if not reference_available():
        port["note"] = "baseline/_ref missing: oracle port only"
        return port
    cores = os.cpu_count() or 1
    w = ReferenceWorkload(REF_SAMPLE_EL)
    v1, r1, e1 = w.rate(1, seconds)
    vt, rt, et = w.rate(cores, seconds)
    best_threads, best = (cores, vt) if vt >= v1 else (1, v1)
    return {"value": best, "unit": "GDOF/s", "cores": best_threads, "kind": "reference",
            "sample": f"{w.bp} N={DEGREE}: first {REF_SAMPLE_EL} elements of the E=32768 mesh "
                      "through the unmodified reference apply_operator (baseline/_ref); value = "
                      "the faster of threads=1 / threads=cores",
            "threads_1": {"value": v1, "cores": 1, "applies": r1, "seconds": round(e1, 2)},
            f"threads_{cores}": {"value": vt, "cores": cores, "applies": rt,
                                 "seconds": round(et, 2)},
            "port": {k: port[k] for k in ("value", "cores", "kind", "sample")}}


E2E_CHUNK_BYTES = 64 << 20  # uniform pipeline chunks for back-to-back steps (tune28)


def e2e_report(op, mesh, steps, warmup):
    """Same metric through the public host-buffer API: per step the H2D copy
    of q from pinned memory, the kernel and the D2H copy of out.  Steps are a
    stream of independent applies, so they use the library's opt-in
    back-to-back mode (hx_apply_host_ex with HX_HOST_OVERLAP: each call's
    uploads run under the previous call's downloads; the bench guarantees the
    mode's contract -- q is final, out is read only after the timed region,
    the workspace is this operator's).  The stream-ordered default mode (no
    cross-call overlap) is timed too and reported beside it."""
    import torch
    import paper_1711_00903_b200 as hx
    from paper_1711_00903_b200 import operators

    n = mesh.n_el * op.n_p
    q_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    q_pin.copy_(torch.from_numpy(np.random.default_rng(0).standard_normal(n)))
    o_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    qh, oh = q_pin.numpy(), o_pin.numpy()
    stream = torch.cuda.current_stream()

    def timed(chunk, overlap):
        work = operators._device_work(op, chunk)
        for _ in range(warmup):
            hx.apply_host(op, qh, oh, chunk_el=chunk, work=work, overlap=overlap)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps):
            hx.apply_host(op, qh, oh, chunk_el=chunk, work=work, overlap=overlap)
        e.record(stream)
        e.synchronize()
        del work
        return s.elapsed_time(e) / steps

    chunk = max(1, E2E_CHUNK_BYTES // (op.n_p * 8))
    ms = timed(chunk, True)
    default_chunk = operators.host_chunk_elements(op)
    ms_ordered = timed(default_chunk, False)
    return ms, {"value": None, "unit": "GDOF/s", "h2d_bytes_per_step": n * 8,
                "d2h_bytes_per_step": n * 8, "ms_per_step": ms,
                "path": "hx_apply_host_ex (C ABI), pinned host q/out, chunked 3-stream "
                        f"H2D/kernel/D2H pipeline, {chunk}-element chunks, HX_HOST_OVERLAP "
                        "(back-to-back steps pipelined)",
                "stream_ordered": {"value": mesh.n_el * op.n_p / (ms_ordered * 1e-3) / 1e9,
                                   "ms_per_step": ms_ordered,
                                   "path": f"hx_apply_host, {default_chunk}-element ramped "
                                           "chunks, each call after the previous one"}}


def e2e_api_report(op, mesh, steps, warmup):
    """The call a reference user makes: apply_operator(op, FieldVector(numpy))
    on a plain pageable numpy array (reference operators.py:306), through
    hx_apply_host_staged; host-synchronous, timed by wall clock per call."""
    import torch
    import paper_1711_00903_b200 as hx

    fv = hx.FieldVector(mesh.n_el, op.n_p,
                        np.random.default_rng(0).standard_normal((mesh.n_el, op.n_p)))
    for _ in range(warmup):
        hx.apply_operator(op, fv)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out = hx.apply_operator(op, fv)
        ts.append(time.perf_counter() - t0)
        del out
    ms = statistics.median(ts) * 1e3
    return {"value": mesh.n_el * op.n_p / (ms * 1e-3) / 1e9, "unit": "GDOF/s",
            "ms_per_step": ms, "h2d_bytes_per_step": fv.data.nbytes,
            "d2h_bytes_per_step": fv.data.nbytes,
            "path": "apply_operator(op, FieldVector(pageable numpy)) -> hx_apply_host_staged "
                    "(pinned staging ring, host copy threads), median wall clock"}


def pcie_bandwidth(nbytes, trials=5):
    """Pinned host<->device copy rates (GB/s) at the e2e step size: H2D alone,
    D2H alone, and the time of both directions concurrently (the PCIe bound
    of one e2e step)."""
    import torch

    n = nbytes // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_in = torch.empty(n, dtype=torch.float64, device="cuda")
    d_out = torch.zeros(n, dtype=torch.float64, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = float("inf")
        for _ in range(trials):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def both():
        with torch.cuda.stream(s_in):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s_out):
            h_out.copy_(d_out, non_blocking=True)

    t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
    t_both = timed(both)
    return {"h2d_gb_per_s": nbytes / t_h2d / 1e9, "d2h_gb_per_s": nbytes / t_d2h / 1e9,
            "bidirectional_ms": t_both * 1e3}


# CG vector passes per iteration beyond the matvec's Table-1 bytes: the
# direction update fused into the matvec's load adds r read + p write (the
# p read is the matvec's q read); the update reads x, p, r, Ap, writes x, r
CG_VECTOR_PASSES = 8
CG_VECTOR_PASSES_UNFUSED = 9  # + hx_cg_direction's own p read (p rw, r read)


def cg_report(op, mesh, iters=20, warmup=3):
    """CG iteration throughput (paper_1711_00903_b200/cg.py): the direction
    update fused into the matvec + <p,Ap> (hx_apply_energy_dir), the update --
    2 kernels per iteration plus 2 tiny reduces, no host synchronisation.
    HBM traffic per iteration = the matvec's Table-1 bytes + 8 vector passes;
    the unfused form (separate hx_cg_direction pass) is timed beside it."""
    import torch
    import paper_1711_00903_b200 as hx
    from paper_1711_00903_b200.cg import CGWorkspace, cg_iterations

    b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    w = CGWorkspace(b)

    def timed(k, fused):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        cg_iterations(op, b, k, w, fuse_direction=fused)
        e.record()
        e.synchronize()
        return s.elapsed_time(e)

    res = {}
    for fused in (True, False):
        timed(warmup, fused)
        # subtract the per-call setup (copies + one dot) measured separately
        res[fused] = (timed(iters, fused) - timed(0, fused)) / iters
    ms = res[True]
    mv = hx.traffic(op.bp, op.degree).bytes_per_element
    per_el = mv + CG_VECTOR_PASSES * 8 * op.n_p
    gbs = per_el * op.n_el / (ms * 1e-3) / 1e9
    unf = mv + CG_VECTOR_PASSES_UNFUSED * 8 * op.n_p
    return {"bp": op.bp, "degree": op.degree, "n_el": op.n_el, "ms_per_iteration": ms,
            "gdof_iterations_per_s": op.n_el * op.n_p / (ms * 1e-3) / 1e9,
            "hbm_bytes_per_iteration": per_el * op.n_el, "achieved_gb_per_s": gbs,
            "kernels_per_iteration": 4,
            "unfused_direction": {"ms_per_iteration": res[False],
                                  "hbm_bytes_per_iteration": unf * op.n_el,
                                  "achieved_gb_per_s": unf * op.n_el / (res[False] * 1e-3) / 1e9,
                                  "kernels_per_iteration": 5}}


def cg_assembled_report(side=32, iters=20, warmup=3):
    """Assembled CG (cg.cg_solve_assembled: Poisson, BP3.5 N=7 on the
    unperturbed side^3 cube mesh, Dirichlet mask): direction update fused into
    the matvec + <p,Ap>, the gather-scatter of A p, the update.  Same 8 vector
    passes per iteration as the element-local CG; the DSS gathers re-read
    shared-node neighbours (L2 hits)."""
    import torch
    import paper_1711_00903_b200 as hx
    from paper_1711_00903_b200.cg import CGWorkspace, cg_iterations_assembled

    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(hx.BP35, DEGREE, mesh, lam=0.0)
    b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    w = CGWorkspace(b)

    def timed(k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        cg_iterations_assembled(op, side, b, k, w)
        e.record()
        e.synchronize()
        return s.elapsed_time(e)

    timed(warmup)
    ms = (timed(iters) - timed(0)) / iters
    per_el = hx.traffic(op.bp, op.degree).bytes_per_element + CG_VECTOR_PASSES * 8 * op.n_p
    unique = (side * DEGREE + 1) ** 3
    small = small_mesh_cg_graph()
    return {"bp": op.bp, "degree": op.degree, "n_el": op.n_el, "side": side,
            "global_dofs": unique, "ms_per_iteration": ms,
            "gdof_iterations_per_s": op.n_el * op.n_p / (ms * 1e-3) / 1e9,
            "global_gdof_iterations_per_s": unique / (ms * 1e-3) / 1e9,
            "hbm_bytes_per_iteration": per_el * op.n_el,
            "achieved_gb_per_s": per_el * op.n_el / (ms * 1e-3) / 1e9,
            "kernels_per_iteration": 7, "small_mesh_cuda_graph": small}


def small_mesh_cg_graph(side=8, iters=200):
    """Launch-bound regime: assembled CG on a side-8 cube (512 elements, N=7),
    eager (~8 launches per iteration from Python) vs the iteration blocks
    captured once as a CUDA graph (AssembledCG(graph=True)).  Wall
    clock per iteration, including the host reads of the residual every 10
    iterations."""
    import time

    import torch
    import paper_1711_00903_b200 as hx
    from paper_1711_00903_b200.cg import AssembledCG

    mesh = hx.build_cube_mesh(side, 2.0)
    op = hx.make_operator(hx.BP35, DEGREE, mesh, lam=0.0)
    b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    res = {}
    for name, graph in (("eager", False), ("graph", True)):
        solver = AssembledCG(op, side, graph=graph)  # the graph is captured here, once
        solver.solve(b, tol=0.0, maxiter=20)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.solve(b, tol=0.0, maxiter=iters)
        torch.cuda.synchronize()
        res[f"{name}_us_per_iteration"] = (time.perf_counter() - t0) / iters * 1e6
    res["n_el"] = mesh.n_el
    res["speedup"] = res["eager_us_per_iteration"] / res["graph_us_per_iteration"]
    return res


def unfused_pass_bytes(bp, deg=DEGREE):
    """HBM bytes per element of the unfused pass structure (hx_baseline.cu):
    every pass reads its input tensor and writes its output (the += passes
    also read the output), pointwise steps read their operands and factors."""
    n, m = deg + 1, deg + 2
    interp = (n**3 + n * m * n) + (n * m * n + n * m * m) + (n * m * m + m**3)
    project = (m**3 + m * n * m) + (m * n * m + m * n * n) + (m * n * n + n**3)

    def chain(p):  # 3 D passes, chain rule (4 in + 7 factors, 4 out), 3 D^T += passes
        return 6 * p**3 + 15 * p**3 + 9 * p**3
    doubles = {"BP1.0": interp + 3 * m**3 + project, "BP3.5": chain(n),
               "BP3.0": interp + chain(m) + project}[bp]
    return 8 * doubles


def baseline_report(steps=5, warmup=2, side=32):
    """Fused kernels vs the unfused Kernel-1-style path (apply_baseline:
    one launch per contraction pass, intermediates in HBM -- the paper's
    reference kernel, and the reference's variant="baseline"
    access pattern) at N=7, E=32768: the K1 -> fused speed-up on B200.  The
    baseline's HBM traffic is its pass structure (unfused_pass_bytes); the
    reference's own baseline counters (perf.element_counters(bp, "baseline",
    N)) count every term's operand read and are reported beside it."""
    import torch
    import paper_1711_00903_b200 as hx
    from paper_1711_00903_b200.operators import apply_baseline_device, baseline_workspace

    res = {}
    for bp in hx.BENCHMARKS:
        mesh, op = build_operator(bp, side, 0)
        q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
        out = torch.empty_like(q)
        work = baseline_workspace(op)

        def timed(fn):
            for _ in range(warmup):
                fn()
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(steps)]
            for s, e in ev:
                s.record()
                fn()
                e.record()
            torch.cuda.synchronize()
            return statistics.median(s.elapsed_time(e) for s, e in ev)

        t_base = timed(lambda: apply_baseline_device(op, q, out, work))
        t_fused = timed(lambda: hx.apply_device(op, q, out))
        c = hx.element_counters(bp, "baseline", DEGREE)
        counted = (c["global_reads"] + c["global_writes"]) * mesh.n_el
        passes = unfused_pass_bytes(bp) * mesh.n_el
        res[bp] = {"n_el": mesh.n_el, "baseline_ms": t_base, "fused_ms": t_fused,
                   "speedup_fused_over_baseline": t_base / t_fused,
                   "baseline_gdof_per_s": mesh.n_el * op.n_p / (t_base * 1e-3) / 1e9,
                   "baseline_pass_bytes": passes,
                   "baseline_achieved_gb_per_s": passes / (t_base * 1e-3) / 1e9,
                   "reference_baseline_counted_global_bytes": counted,
                   "baseline_launches": {"BP1.0": 7, "BP3.5": 7, "BP3.0": 13}[bp]}
        del op, q, out, work
        torch.cuda.empty_cache()
    return res


def kernel_profile(bp):
    """Per-launch counters of the kernel from the committed ncu capture
    (profiles/kernels.json, written by tools/ncu_summary.py), per element."""
    path = os.path.join(ROOT, "profiles", "kernels.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        k = json.load(fh).get(f"{KERNEL[bp]}<{DEGREE}>")
    return k


KERNEL = {"BP1.0": "bp1_kernel", "BP3.5": "bp35_kernel", "BP3.0": "bp3_kernel"}
SMEM_WAVEFRONT_BYTES = 128  # one shared-memory wavefront: 32 banks x 4 B per cycle


def smem_roofline(rep, b_smem):
    """Shared-memory roofline of one per_bp entry: the kernel's measured
    shared-memory wavefronts per element (ncu) x 128 B, over the kernel time,
    against the measured LDS bandwidth (north_star (4); the paper's B_sh,
    PAPER.md:476-487)."""
    k = kernel_profile(rep["bp"])
    if not k or not b_smem:
        return None
    wf = k["smem_wavefronts"] / k["n_el"]
    nbytes = wf * SMEM_WAVEFRONT_BYTES * rep["n_el"]
    achieved = nbytes / (rep["kernel_ms_median"] * 1e-3)
    return {"smem_bytes_per_element": wf * SMEM_WAVEFRONT_BYTES,
            "smem_gb_per_s": achieved / 1e9, "smem_roofline_frac": achieved / b_smem,
            "ncu": k.get("source")}


def run_ours(args):
    import torch
    import paper_1711_00903_b200 as hx

    rank, world, local = dist_setup(args)
    hbm_peak, peak_kind = load_peaks()
    bp, side = HEADLINE
    mesh, op = build_operator(bp, side, rank)
    q = hx.FieldVector.random(mesh.n_el, op.n_p, seed=0).to_device().data
    out = torch.empty_like(q)
    t = hx.traffic(bp, DEGREE, mesh.n_el)
    bytes_per_apply = t.bytes_per_element * mesh.n_el
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        hx.apply_device(op, q, out)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        # the K applies back to back between one event pair: the timed region
        # holds nothing but our kernels (programmatic dependent launches, so
        # one apply's retiring CTAs overlap the next one's start)
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        gpu_spacer()  # the first launch is queued before the start event is reached
        start.record(stream)
        for _ in range(args.steps):
            hx.apply_device(op, q, out)
        stop.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    total_ms = max_over_ranks(start.elapsed_time(stop), world)
    ms_per_step = total_ms / args.steps
    kernel_ms = ms_per_step  # average launch duration over the timed region
    # one launch at a time (GPU spacer before each, per-launch events): the
    # per-launch fill / drain the back-to-back stream hides, for reference
    single_ms = max_over_ranks(statistics.median(
        time_applies(op, q, out, max(5, min(args.steps, 20)), 1)), world)
    dofs_all = sum_over_ranks(mesh.n_el * op.n_p, world)
    value = dofs_all / (ms_per_step * 1e-3) / 1e9
    achieved = bytes_per_apply / (kernel_ms * 1e-3) / 1e9

    barrier(world)
    e2e_ms, e2e = e2e_report(op, mesh, args.steps, max(3, args.warmup))  # same K as `value`
    e2e_ms = max_over_ranks(e2e_ms, world)
    e2e["value"] = dofs_all / (e2e_ms * 1e-3) / 1e9
    e2e["ms_per_step"] = e2e_ms
    full = rank == 0 and not args.quick
    details = {}
    if full:
        pcie = pcie_bandwidth(e2e["h2d_bytes_per_step"])
        details["pcie"] = pcie
        e2e["frac_of_pcie_bound"] = pcie["bidirectional_ms"] / e2e_ms
        api = e2e_api_report(op, mesh, args.steps, max(3, args.warmup))
        api["vs_pinned_e2e"] = api["ms_per_step"] / e2e_ms
        # like for like: one isolated, stream-ordered pinned call per step
        api["vs_pinned_isolated"] = api["ms_per_step"] / e2e["stream_ordered"]["ms_per_step"]
        e2e["api"] = {k: api[k] for k in ("value", "ms_per_step", "vs_pinned_e2e",
                                          "vs_pinned_isolated")}
        details["e2e_api"] = api
    b_smem = None
    if full:
        import ctypes
        from paper_1711_00903_b200 import _native
        bsh = ctypes.c_double()
        _native.check(_native.lib().hx_measure_smem_bandwidth(
            ctypes.byref(bsh), torch.cuda.current_stream().cuda_stream))
        b_smem = bsh.value
        details["calibration"] = {
            "b_smem_measured_gb_per_s": b_smem / 1e9,
            "b_smem_paper_ansatz_gb_per_s": hx.shared_bandwidth_ansatz(148, 32, 4, 1.965) / 1e9,
            "note": "measured LDS.64 bandwidth (hx_measure_smem_bandwidth) replaces the "
                    "paper's B_sh ansatz (PAPER.md:476-487)"}
        details["cg"] = cg_report(op, mesh)
        details["cg_assembled"] = cg_assembled_report()
        details["unfused_baseline"] = baseline_report()

    traffic = None
    prof = kernel_profile(bp)
    if prof:
        traffic = prof["dram_bytes"] / prof["n_el"] * mesh.n_el

    per_bp = {}
    cpu = None
    del op, q, out
    torch.cuda.empty_cache()
    if full and world == 1:
        for xbp, xside in ((bp, side),) + EXTRA:
            r = bp_report(xbp, xside, 0, args.steps, args.warmup, hbm_peak)
            sm = smem_roofline(r, b_smem)
            if sm:
                r.update(sm)
            details.setdefault("per_bp", {})[f"{xbp} E={r['n_el']}"] = r
            per_bp[f"{xbp} E={r['n_el']}"] = {
                k: (round(r[k], 4) if isinstance(r.get(k), float) else r.get(k))
                for k in ("gdof_per_s", "frac_of_measured_peak", "frac_of_copy_same_size",
                          "kernel_ms_median", "smem_roofline_frac")}
        cpu = reference_cpu()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: perturb_mesh(build_cube_mesh(32, 2.0), 0.15, seed=7+rank), "
                    "q = FieldVector.random(seed=0), device-generated geometric factors",
            "config": arm_config(bp, mesh.n_el, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                         "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                         if peak_kind == "measured" else "fallback 6650 GB/s",
                         "kernel": f"bp35_kernel<{DEGREE}>",
                         "algorithmic_bytes_per_element": t.bytes_per_element,
                         "kernel_ms": kernel_ms,
                         "timing": "K applies back to back, one CUDA event pair on the "
                                   "launching stream; kernel_ms = region / K",
                         "single_launch_kernel_ms": single_ms},
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "gflop_per_s": hx.flop_model(bp, "fused", DEGREE) * dofs_all / (DEGREE + 1) ** 3
                           / (ms_per_step * 1e-3) / 1e9,
        }
        if details:
            line["details"] = summarize_details(details)
            os.makedirs(os.path.dirname(DETAILS), exist_ok=True)
            with open(DETAILS, "w") as fh:
                json.dump(details, fh, indent=1)
        line["per_bp"] = per_bp  # last: the driver keeps the tail of the line
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def summarize_details(d):
    """A few headline numbers of the secondary legs for the JSON line (the
    full legs are in gpurun_out/bench_details.json)."""
    out = {"file": os.path.relpath(DETAILS, ROOT)}
    if "calibration" in d:
        out["b_smem_gb_per_s"] = round(d["calibration"]["b_smem_measured_gb_per_s"], 1)
    if "cg" in d:
        out["cg_ms_per_iteration"] = round(d["cg"]["ms_per_iteration"], 4)
    if "cg_assembled" in d:
        out["cg_assembled_ms_per_iteration"] = round(d["cg_assembled"]["ms_per_iteration"], 4)
    if "unfused_baseline" in d:
        out["fused_speedup_over_unfused"] = {
            k: round(v["speedup_fused_over_baseline"], 2)
            for k, v in d["unfused_baseline"].items()}
    return out


def arm_config(bp, n_el, world):
    """The `config` both arms report (same workload, same keys)."""
    return {"workload": f"{bp} N={DEGREE} E={n_el} per GPU (BASELINE configs[1])",
            "bp": bp, "degree": DEGREE, "n_el_per_gpu": n_el, "lam": LAM,
            "l2": "inputs larger than L2 (1.21 GB per apply)",
            "parallelism": f"element partition x{world}, no data-path collective"}


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the path
    -- the unmodified hexbench package pip-installed into baseline/_ref --
    through its public apply_operator with its element-range thread pool on
    all host cores, each step a bounded sample of the headline workload;
    rank 0 only.  Without baseline/_ref: the oracle port, threads over
    element ranges."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    bp = HEADLINE[0]
    if reference_available():
        sample = 1024
        w = ReferenceWorkload(sample)
        # the reference's element-range thread pool is GIL-bound: time its
        # faster setting (threads = 1 or all cores), so the arm is its best
        probe = {t: w.rate(t, seconds=1.0, min_reps=1)[0] for t in sorted({1, cores})}
        threads = max(probe, key=probe.get)
        for _ in range(args.warmup):
            w.step(threads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            w.step(threads)
        el = time.perf_counter() - t0
        ms = el / args.steps * 1e3
        value = w.dofs / (ms * 1e-3) / 1e9
        kind = "reference"
        cores = threads
        desc = (f"bounded sample: first {sample} of the 32768 elements per step through the "
                f"unmodified reference apply_operator(op, q, threads={threads}) (baseline/_ref, "
                "hexbench 0.1.0); threads = the faster of 1 / all host cores "
                f"({', '.join(f'{t}: {v:.4f} GDOF/s' for t, v in probe.items())})")
    else:
        value, ms, desc = port_reference_steps(args, cores)
        kind = "port"
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "impl": "reference",
        "data": "synthetic: same mesh / q generator as the GPU arm",
        "config": arm_config(bp, HEADLINE[1] ** 3, 1),
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def port_reference_steps(args, cores):
    """Fallback reference arm: the oracle port on all host cores (4096-element
    sample per step, one BLAS thread per worker thread)."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_1711_00903_b200 as hx
    from oracle import hexbench_oracle as orc

    bp, side = HEADLINE
    sample = 4096
    mesh = hx.perturb_mesh(hx.build_cube_mesh(side, 2.0), amplitude=0.15, seed=7)
    sub = hx.HexMesh(sample, mesh.vertices[:sample], mesh.extent)
    fac = hx.geometric_factors(sub, hx.gll_rule(DEGREE + 1)).data
    diff = hx.diff_matrix_gll(DEGREE).entries
    q = np.random.default_rng(0).standard_normal((sample, (DEGREE + 1) ** 3))
    chunks = np.linspace(0, sample, cores + 1).astype(int)
    spans = [(lo, hi) for lo, hi in zip(chunks[:-1], chunks[1:]) if hi > lo]
    pool = ThreadPoolExecutor(max_workers=cores)

    def step():
        list(pool.map(lambda r: orc.apply(bp, DEGREE, LAM, None, diff, fac[r[0]:r[1]],
                                          q[r[0]:r[1]]), spans))

    import contextlib
    try:
        from threadpoolctl import threadpool_limits
        limits = threadpool_limits(1)
    except ImportError:
        limits = contextlib.nullcontext()
    with limits:
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    return (sample * q.shape[1] / (ms * 1e-3) / 1e9, ms,
            f"bounded sample: first {sample} of the {mesh.n_el} elements per step, {cores} "
            "threads over element ranges (1 BLAS thread each), oracle/hexbench_oracle.py")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--quick", action="store_true",
                    help="headline only (skip per-BP reports and the CPU baseline)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
