"""Measurement contract: Table-1 traffic, the FLOP convention, rooflines and
the analytic access counters.

These are the *algorithmic* numbers the harness divides by measured kernel
times (reference ``perf.py:79-117``, ``PAPER.md:439-487``).  The access
counters mirror the per-element charging sequence of reference
``operators.py:146-200`` / ``:271-293``; they are value-independent and
exactly linear in the element count, so they are charged once per element
and scaled, never by touching the data.
"""

from dataclasses import dataclass, field

BP1 = "BP1.0"
BP35 = "BP3.5"
BP3 = "BP3.0"
BENCHMARKS = (BP1, BP35, BP3)
VARIANTS = ("baseline", "fused", "symfused")

DOUBLE = 8

# P100 defaults of the paper's shared-bandwidth ansatz (reference perf.py:12-18)
DEFAULT_PEAK_BANDWIDTH = 549e9
DEFAULT_SM_COUNT = 56
DEFAULT_SIMD_WIDTH = 32
DEFAULT_WORD_BYTES = 4
DEFAULT_CLOCK_GHZ = 1.328


@dataclass(frozen=True)
class TrafficModel:
    """Minimum per-element doubles moved to/from main memory (Table 1)."""

    bp: str
    degree: int
    n_el: int
    reads_doubles: int
    writes_doubles: int

    @property
    def total_doubles(self):
        return self.reads_doubles + self.writes_doubles

    @property
    def bytes_per_element(self):
        return DOUBLE * self.total_doubles

    @property
    def copy_equivalent_bytes(self):
        # a copy of T/2 doubles moves the same read+write total
        return DOUBLE * self.n_el * self.total_doubles // 2


def traffic(bp, degree, n_el=1):
    """Table 1 (reference perf.py:79-93)."""
    if bp not in BENCHMARKS:
        raise ValueError(f"unknown benchmark {bp!r}")
    if not 1 <= degree <= 15:
        raise ValueError("degree must be in 1..15")
    n3 = (degree + 1) ** 3
    m3 = (degree + 2) ** 3
    reads = {BP1: n3 + m3, BP35: 8 * n3, BP3: n3 + 7 * m3}[bp]
    return TrafficModel(bp, degree, n_el, reads, n3)


def flop_model(bp, variant, degree):
    """Closed-form FLOPs per element (reference perf.py:96-117): multiply-add
    = 2, pointwise scale = 1, chain rule = 15/point, lambda + combine = 5."""
    if bp not in BENCHMARKS:
        raise ValueError(f"unknown benchmark {bp!r}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    n, m = degree + 1, degree + 2
    interp = 2 * (m * n ** 3 + m ** 2 * n ** 2 + m ** 3 * n)
    if bp == BP1:
        return 2 * interp + m ** 3
    if bp == BP35:
        return 12 * n ** 4 + 20 * n ** 3
    return 2 * interp + 12 * m ** 4 + 20 * m ** 3


# nominal B200 HBM3e bandwidth (the calibration's `theoretical_peak`)
B200_PEAK_BANDWIDTH = 8.0e12


@dataclass(frozen=True)
class BandwidthCalibration:
    """Result of :func:`measure_stream_bandwidth` (reference perf.py:46-51)."""

    bytes_transferred: int
    trial_times: list
    mean_bandwidth: float
    theoretical_peak: float = DEFAULT_PEAK_BANDWIDTH


def measure_stream_bandwidth(nbytes, trials=10, device=None):
    """Streaming-bandwidth calibration (reference perf.py:120-143).

    Same contract as the reference -- at least 1 MiB and 3 trials
    (``ValueError``), ``MemoryError`` when the buffers cannot be allocated,
    one untimed warm-up pass, ``mean_bandwidth`` = mean of the per-trial
    ``bytes_transferred / time`` -- but the copy is a device-to-device copy
    of ``nbytes`` on the GPU the operators run on (the reference copies host
    memory), timed with CUDA events behind a GPU spacer so host launch
    latency is not timed.  ``bytes_transferred`` counts the bytes copied (one
    way), as the reference does; the copy moves twice that through HBM, the
    convention ``TrafficModel.copy_equivalent_bytes`` accounts for.
    """
    if nbytes < 1 << 20:
        raise ValueError("use at least 1 MiB for a meaningful measurement")
    if trials < 3:
        raise ValueError("need at least 3 trials")
    import torch
    count = nbytes // 8
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    try:
        src = torch.randn(count, dtype=torch.float64, device=dev)
        dst = torch.empty_like(src)
    except torch.OutOfMemoryError as exc:
        raise MemoryError("could not allocate calibration buffers") from exc
    with torch.cuda.device(dev):
        dst.copy_(src)  # warm-up
        times = []
        for _ in range(trials):
            start = torch.cuda.Event(enable_timing=True)
            stop = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # spacer: the copy is queued before `start`
            start.record()
            dst.copy_(src)
            stop.record()
            stop.synchronize()
            times.append(start.elapsed_time(stop) * 1e-3)
    rates = [8 * count / t for t in times]
    return BandwidthCalibration(8 * count, times, float(sum(rates) / len(rates)),
                                B200_PEAK_BANDWIDTH)


def roofline_global(b_gl, flops, d_r, d_w):
    if b_gl <= 0 or flops <= 0:
        raise ValueError("bandwidth and FLOPs must be positive")
    if d_r + d_w <= 0:
        raise ValueError("byte traffic must be positive")
    return b_gl * flops / (d_r + d_w)


def shared_bandwidth_ansatz(sm_count=DEFAULT_SM_COUNT, simd_width=DEFAULT_SIMD_WIDTH,
                            word_bytes=DEFAULT_WORD_BYTES, clock_ghz=DEFAULT_CLOCK_GHZ):
    if min(sm_count, simd_width, word_bytes, clock_ghz) <= 0:
        raise ValueError("all ansatz inputs must be positive")
    return sm_count * simd_width * word_bytes * clock_ghz * 1e9


def roofline_shared(b_sh, flops, s_r, s_w):
    if b_sh <= 0 or flops <= 0:
        raise ValueError("bandwidth and FLOPs must be positive")
    if s_r + s_w <= 0:
        raise ValueError("scratch traffic must be positive")
    return b_sh * flops / (s_r + s_w)


@dataclass(frozen=True)
class RooflinePoint:
    degree: int
    flops: int
    bytes_moved: int
    r_global: float
    r_shared: float = None

    @property
    def bound(self):
        return self.r_global if self.r_shared is None else min(self.r_global, self.r_shared)


@dataclass(frozen=True)
class RooflineSeries:
    bp: str
    variant: str
    n_el: int
    bandwidth: float
    shared_bandwidth: float
    points: list = field(default_factory=list)


def scratch_traffic(bp, variant, degree):
    """Per-element scratch bytes (reads, writes) of one apply -- reference
    perf.py:172-178 re-runs a one-element apply to read its counters; the
    counters are value-independent, so they are charged analytically here."""
    c = element_counters(bp, variant, degree)
    return c["scratch_reads"], c["scratch_writes"]


def roofline_series(bp, degrees, n_el, b_gl, variant="fused", b_sh=None):
    """Model series across degrees (reference perf.py:181-201): the global
    roofline from Table 1 and, for the interpolation-bearing benchmarks, the
    scratch roofline from the modelled scratch traffic.  Feed it the
    measured B_copy and B_smem of the device (bench.py's calibration)."""
    with_shared = b_sh is not None and bp != BP35
    points = []
    for degree in degrees:
        t = traffic(bp, degree, n_el)
        flops = flop_model(bp, variant, degree) * n_el
        r_gl = roofline_global(b_gl, flops, 8 * t.reads_doubles * n_el,
                               8 * t.writes_doubles * n_el)
        r_sh = None
        if with_shared:
            s_r, s_w = scratch_traffic(bp, variant, degree)
            r_sh = roofline_shared(b_sh, flop_model(bp, variant, degree), s_r, s_w)
        points.append(RooflinePoint(degree, flops, t.bytes_per_element * n_el, r_gl, r_sh))
    return RooflineSeries(bp, variant, n_el, b_gl, b_sh if with_shared else None, points)


# ---------------------------------------------------------------------------
# analytic access counters
# ---------------------------------------------------------------------------

COUNTER_FIELDS = ("global_reads", "global_writes", "scratch_reads",
                  "scratch_writes", "interp_matrix_reads", "flops", "syncs")


class _Tally(dict):
    def __init__(self):
        super().__init__({k: 0 for k in COUNTER_FIELDS})


def _contract(c, variant, out_points, terms, interp, in_global, out_global):
    c["flops"] += 2 * out_points * terms
    uses = out_points * terms
    loads = (uses + 1) // 2 if (interp and variant == "symfused") else uses
    c["scratch_reads"] += DOUBLE * loads
    if interp:
        c["interp_matrix_reads"] += DOUBLE * loads
    c["global_reads" if in_global else "scratch_reads"] += DOUBLE * uses
    c["global_writes" if out_global else "scratch_writes"] += DOUBLE * out_points


def _pointwise(c, points, fpp, tensor_reads, factor_reads, writes, in_global, out_global):
    c["flops"] += fpp * points
    c["global_reads"] += DOUBLE * factor_reads * points
    c["global_reads" if in_global else "scratch_reads"] += DOUBLE * tensor_reads * points
    c["global_writes" if out_global else "scratch_writes"] += DOUBLE * writes * points


def _interp(c, v, n, m, gb, in_global, out_global):
    _contract(c, v, m * n * n, n, True, in_global, gb)
    _contract(c, v, m * m * n, n, True, gb, gb)
    _contract(c, v, m * m * m, n, True, gb, out_global)


def _project(c, v, n, m, gb, in_global, out_global):
    _contract(c, v, m * n * m, m, True, in_global, gb)
    _contract(c, v, m * n * n, m, True, gb, gb)
    _contract(c, v, n * n * n, m, True, gb, out_global)


def _diff_chain(c, v, q, gb):
    p = q ** 3
    for _ in range(3):
        _contract(c, v, p, q, False, gb, gb)
    _pointwise(c, p, 15, 3, 6, 3, gb, gb)
    for _ in range(3):
        _contract(c, v, p, q, False, gb, gb)
    _pointwise(c, p, 5, 1, 1, 0, gb, gb)


def element_counters(bp, variant, degree):
    """Counter increments of one element apply, replaying the charge sequence
    of reference operators.py:271-293 (no arithmetic on data)."""
    if bp not in BENCHMARKS:
        raise ValueError(f"unknown benchmark {bp!r}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    n, m = degree + 1, degree + 2
    gb = variant == "baseline"
    c = _Tally()

    def staging(points):
        if not gb:
            c["global_reads"] += DOUBLE * points
            c["scratch_writes"] += DOUBLE * points

    def boundaries(count, slices):
        c["syncs"] += count * slices + 1 if gb else count

    staging(n ** 3)
    if bp == BP1:
        _interp(c, variant, n, m, gb, gb, gb)
        _pointwise(c, m ** 3, 1, 1, 1, 1, gb, gb)
        _project(c, variant, n, m, gb, gb, True)
        boundaries(5, m)
    elif bp == BP35:
        _diff_chain(c, variant, n, gb)
        c["global_writes"] += DOUBLE * n ** 3
        boundaries(1, n)
    else:
        _interp(c, variant, n, m, gb, gb, gb)
        _diff_chain(c, variant, m, gb)
        _project(c, variant, n, m, gb, gb, True)
        boundaries(7, m)
    return dict(c)
