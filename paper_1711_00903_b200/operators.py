"""Drop-in operator API for BP1.0 / BP3.5 / BP3.0 (reference ``operators.py``).

Same names, signatures, validation and error types as the reference
(``make_operator`` operators.py:118-143, ``apply_operator`` :306-331,
``apply_bp*`` :334-349, ``FieldVector`` :67-91, ``OperatorInstance`` :94-115,
``AccessCounters`` :41-64).  What changes is underneath:

* ``make_operator`` builds the 1-D matrices on the host (tiny) and the
  geometric factors on the device, straight into the packed layout the
  kernels stream (``hx_geometric_factors``);
* ``apply_operator`` is one fused sm_100a kernel launch through the C ABI
  (``hx_apply`` for device-resident torch tensors, ``hx_apply_host`` for
  host numpy arrays, with the PCIe copies pipelined against the kernel);
* counters are charged analytically per element (``perf.element_counters``),
  identical to the reference's instrumented values;
* ``threads`` is accepted for signature compatibility; results are
  independent of it by construction (the reference guarantees the same,
  operators.py:309-311).

There is no CPU execution path: without the native library every apply
raises ``NativeLibraryError``.
"""

import threading
from dataclasses import dataclass, field, fields

import numpy as np

from . import _native
from .basis import check_degree, diff_matrix_gl, diff_matrix_gll, interp_matrix
from .mesh import DegenerateGeometryError, GeometricFactors
from .perf import BENCHMARKS, BP1, BP3, BP35, VARIANTS, element_counters
from .quadrature import gl_rule, gll_rule

DOUBLE = 8
_BP_ID = {BP1: _native.HX_BP1, BP35: _native.HX_BP35, BP3: _native.HX_BP3}


class UnsupportedVariantError(ValueError):
    """A variant was requested for a benchmark that lacks it."""


@dataclass
class AccessCounters:
    """Modelled byte / FLOP / barrier totals (reference operators.py:41-64)."""

    global_reads: int = 0
    global_writes: int = 0
    scratch_reads: int = 0
    scratch_writes: int = 0
    interp_matrix_reads: int = 0
    flops: int = 0
    syncs: int = 0

    def merge(self, other):
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(other, f.name))


def _is_torch(x):
    return type(x).__module__.startswith("torch")


@dataclass(frozen=True)
class FieldVector:
    """Element-blocked field, (n_el, n_p) float64, point order (k, j, i).

    ``data`` may be a numpy array (host) or a torch float64 tensor (device
    resident); shape and size checks follow reference operators.py:75-79.
    """

    n_el: int
    n_p: int
    data: object = field(repr=False)

    def __post_init__(self):
        d = self.data
        if _is_torch(d):
            import torch
            if d.dtype != torch.float64:
                d = d.to(torch.float64)
            if d.numel() != self.n_el * self.n_p:
                raise ValueError("data length must be n_el * n_p")
            d = d.reshape(self.n_el, self.n_p)
        else:
            d = np.asarray(d, dtype=float)
            if d.size != self.n_el * self.n_p:
                raise ValueError("data length must be n_el * n_p")
            d = d.reshape(self.n_el, self.n_p)
        object.__setattr__(self, "data", d)

    @classmethod
    def constant(cls, n_el, n_p, value=1.0):
        return cls(n_el, n_p, np.full(n_el * n_p, float(value)))

    @classmethod
    def random(cls, n_el, n_p, seed=0):
        rng = np.random.default_rng(seed)
        return cls(n_el, n_p, rng.standard_normal(n_el * n_p))

    @property
    def on_device(self):
        return _is_torch(self.data) and self.data.is_cuda

    def flat(self):
        return self.data.reshape(-1)

    def to_device(self, device=None):
        import torch
        dev = torch.device("cuda") if device is None else torch.device(device)
        d = self.data if _is_torch(self.data) else torch.from_numpy(np.ascontiguousarray(self.data))
        return FieldVector(self.n_el, self.n_p, d.to(dev))

    def to_host(self):
        d = self.data.detach().cpu().numpy() if _is_torch(self.data) else self.data
        return FieldVector(self.n_el, self.n_p, d)


@dataclass(frozen=True)
class OperatorInstance:
    bp: str
    degree: int
    lam: float
    interp: object  # OperatorMatrix or None
    diff: object
    factors: object  # GeometricFactors (device-backed, host view on demand)
    variant: str
    n_el: int
    plan: object = field(default=None, repr=False, compare=False)
    device_factors: object = field(default=None, repr=False, compare=False)
    device: object = field(default=None, repr=False, compare=False)

    @property
    def n_q(self):
        return self.degree + 1

    @property
    def n_q_gl(self):
        return self.degree + 2

    @property
    def n_p(self):
        return self.n_q ** 3


def _stream(device):
    import torch
    return ctypes_stream(torch.cuda.current_stream(device))


def ctypes_stream(s):
    return s.cuda_stream


def _validate(bp, degree, variant, lam):
    """Reference operators.py:120-129, same order and messages."""
    if bp not in BENCHMARKS:
        raise ValueError(f"unknown benchmark {bp!r}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if variant == "symfused" and bp == BP35:
        raise UnsupportedVariantError(
            "symfused exploits the interpolation matrix; BP3.5 has none")
    if lam < 0:
        raise ValueError("lambda must be non-negative")
    check_degree(degree)


def make_operator(bp, degree, mesh, lam=0.0, variant="fused", device=None, factors=None):
    """Assemble matrices and device-resident geometric factors.

    ``factors`` (optional) is a reference-layout ``(n_el, 7, m, m, m)`` array or
    ``GeometricFactors`` to upload instead of generating them on the device
    (used to feed the reference's exact factors into parity tests).
    """
    _validate(bp, degree, variant, lam)
    import torch

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    if bp == BP1:
        interp, diff, rule = interp_matrix(degree), None, gl_rule(degree + 2)
    elif bp == BP35:
        interp, diff, rule = None, diff_matrix_gll(degree), gll_rule(degree + 1)
    else:
        interp, diff, rule = interp_matrix(degree), diff_matrix_gl(degree), gl_rule(degree + 2)
    plan = _native.Plan(_BP_ID[bp], degree, float(lam),
                        None if interp is None else interp.entries,
                        None if diff is None else diff.entries, rule.nodes, rule.weights)
    n_el = mesh.n_el
    packed = torch.empty(max(n_el, 1) * plan.elem_stride, dtype=torch.float64, device=dev)
    stream = _stream(dev)
    with torch.cuda.device(dev):
        if factors is None:
            verts = torch.from_numpy(np.array(mesh.vertices, dtype=np.float64)).to(dev)
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            _native.check(_native.lib().hx_geometric_factors(
                plan.handle, _native.ptr(verts), n_el, 0, _native.ptr(packed),
                _native.ptr(flag), stream), "hx_geometric_factors")
            if int(flag.item()) & _native.HX_FLAG_DEGENERATE:
                raise DegenerateGeometryError("non-positive Jacobian determinant")
        else:
            ref = factors.data if isinstance(factors, GeometricFactors) else factors
            ref = np.ascontiguousarray(ref, dtype=np.float64).reshape(n_el, 7, -1)
            src = torch.from_numpy(ref).to(dev)
            _native.check(_native.lib().hx_repack_factors(
                plan.handle, _native.ptr(src), n_el, _native.ptr(packed), 1, stream),
                "hx_repack_factors")
            verts = None
    q = rule.n

    def host_view():
        with torch.cuda.device(dev):
            if factors is not None:
                return np.array(ref).reshape(n_el, 7, q, q, q)
            full = torch.empty(max(n_el, 1) * 7 * plan.slot_stride, dtype=torch.float64,
                               device=dev)
            s = _stream(dev)
            v = torch.from_numpy(np.array(mesh.vertices, dtype=np.float64)).to(dev)
            _native.check(_native.lib().hx_geometric_factors(
                plan.handle, _native.ptr(v), n_el, 1, _native.ptr(full), None, s))
            out = torch.empty(n_el * 7 * q ** 3, dtype=torch.float64, device=dev)
            _native.check(_native.lib().hx_repack_factors(
                plan.handle, _native.ptr(full), n_el, _native.ptr(out), 0, s))
            return out.cpu().numpy().reshape(n_el, 7, q, q, q)

    geo = GeometricFactors(rule.kind, q, rule.weights, loader=host_view)
    return OperatorInstance(bp, degree, float(lam), interp, diff, geo, variant, n_el,
                            plan=plan, device_factors=packed, device=dev)


def _charge(op, counters):
    if counters is None:
        return
    per = element_counters(op.bp, op.variant, op.degree)
    for k, v in per.items():
        setattr(counters, k, getattr(counters, k) + v * op.n_el)


def apply_device(op, q, out, flag=None, stream=None):
    """Raw device apply: ``out = A q`` for torch CUDA tensors, asynchronous on
    ``stream`` (default: torch's current stream), no allocation, no sync.
    This is what the harness times."""
    import torch
    if torch.cuda.current_device() != op.device.index:
        with torch.cuda.device(op.device):
            return apply_device(op, q, out, flag, stream)
    if stream is None:
        stream = _stream(op.device)
    _native.check(_native.lib().hx_apply(
        op.plan.handle, _native.ptr(q), _native.ptr(op.device_factors), _native.ptr(out),
        op.n_el, _native.ptr(flag), stream), "hx_apply")


def _check_out(op, q, out):
    """A caller-supplied ``out`` must be what the kernels write without a
    copy: C-contiguous float64 of shape (n_el, n_p), the same kind as ``q``
    (a CUDA tensor on op.device for device data, host memory for host data),
    and not ``q`` itself."""
    shape = (op.n_el, op.n_p)
    if q.on_device:
        import torch
        if not (_is_torch(out) and out.is_cuda):
            raise ValueError("out must be a CUDA tensor when q is device-resident")
        if out.device != op.device:
            raise ValueError(f"out is on {out.device}, the operator on {op.device}")
        if out.dtype != torch.float64 or tuple(out.shape) != shape or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous float64 tensor of shape {shape}")
        if out.data_ptr() == q.data.data_ptr():
            raise ValueError("out must not alias q")
    else:
        if not isinstance(out, np.ndarray):
            raise ValueError("out must be a numpy array when q is host data")
        if out.dtype != np.float64 or out.shape != shape or not out.flags.c_contiguous \
                or not out.flags.writeable:
            raise ValueError(f"out must be a writeable C-contiguous float64 array of shape {shape}")
        if np.shares_memory(out, q.data):
            raise ValueError("out must not alias q")


def apply_operator(op, q, counters=None, threads=1, out=None):
    """Apply a benchmark operator to a field vector (reference operators.py:306-331).

    Returns a new FieldVector of the same kind as ``q`` (host numpy in, host
    numpy out; device tensor in, device tensor out).  Raises ValueError on a
    shape mismatch, a device mismatch or non-finite input, like the
    reference.  Without ``out`` the non-finite test is fused into the kernel's
    loads and the (never returned) result is discarded on error; with a
    caller-supplied ``out`` (an extension: the reference has none) q is
    scanned first, as the reference does (operators.py:317-318), so ``out``
    is left untouched on bad input.
    """
    if q.n_el != op.n_el or q.n_p != op.n_p:
        raise ValueError("field vector shape does not match operator")
    import torch

    dev = op.device
    if q.on_device and q.data.device != dev:
        raise ValueError(f"field vector is on {q.data.device}, the operator on {dev}")
    if out is not None:
        _check_out(op, q, out)
    with torch.cuda.device(dev):
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        stream = _stream(dev)
        if q.on_device:
            src = q.data.contiguous()
            if out is not None:
                _native.check(_native.lib().hx_check_finite(
                    _native.ptr(src), src.numel(), _native.ptr(flag), stream), "hx_check_finite")
                if int(flag.item()) & _native.HX_FLAG_NONFINITE:
                    raise ValueError("field vector contains non-finite values")
            dst = torch.empty_like(src) if out is None else out
            apply_device(op, src, dst, flag, stream)
            result = FieldVector(op.n_el, op.n_p, dst)
        else:
            src = np.ascontiguousarray(q.data, dtype=np.float64)
            if out is not None and not _native.lib().hx_host_all_finite(
                    _native.ptr(src), src.size):
                raise ValueError("field vector contains non-finite values")
            dst = _pinned_empty(src.shape) if out is None else out
            _apply_numpy(op, src, dst, flag, stream)
            result = FieldVector(op.n_el, op.n_p, dst)
        if int(flag.item()) & _native.HX_FLAG_NONFINITE:
            raise ValueError("field vector contains non-finite values")
    _charge(op, counters)
    return result


DEFAULT_CHUNK_BYTES = 32 << 20  # r42: best for isolated pinned calls
STAGED_CHUNK_BYTES = 16 << 20   # pageable input: host copy of chunk c+1 overlaps chunk c


def host_chunk_elements(op, chunk_bytes=DEFAULT_CHUNK_BYTES):
    return max(1, min(op.n_el, chunk_bytes // (op.n_p * DOUBLE)))


def _device_work(op, chunk_el):
    import torch
    nbytes = _native.lib().hx_apply_host_workspace(op.plan.handle, chunk_el)
    return torch.empty(nbytes // DOUBLE, dtype=torch.float64, device=op.device)


def _apply_host(op, src, dst, flag, stream, chunk_el=None, work=None, overlap=False):
    if op.n_el == 0:
        return dst
    if chunk_el is None:
        chunk_el = host_chunk_elements(op)
    if work is None:
        work = _device_work(op, chunk_el)
    _native.check(_native.lib().hx_apply_host_ex(
        op.plan.handle, _native.ptr(src), _native.ptr(op.device_factors), _native.ptr(dst),
        op.n_el, chunk_el, _native.ptr(work), _native.ptr(flag),
        _native.HX_HOST_OVERLAP if overlap else 0, stream), "hx_apply_host_ex")
    return dst


def _pinned_empty(shape):
    """Uninitialised page-locked float64 host array (torch's caching host
    allocator: repeated calls reuse the blocks), so apply_operator's result
    comes straight back over PCIe with no host copy or page faults."""
    import torch
    return torch.empty(int(np.prod(shape)), dtype=torch.float64,
                       pin_memory=True).numpy().reshape(shape)


# Page-locked staging ring of hx_apply_host_staged, cached per size; one user
# at a time.
_staging = {}
_staging_lock = threading.Lock()


def _staging_buffer(op, chunk_el):
    import torch
    need = _native.lib().hx_apply_host_staging_bytes(op.plan.handle, chunk_el) // DOUBLE
    buf = _staging.get("buf")
    if buf is None or buf.numel() < need:
        buf = torch.empty(need, dtype=torch.float64, pin_memory=True)
        _staging["buf"] = buf
    return buf


def _apply_numpy(op, src, dst, flag, stream, chunk_el=None):
    """apply_operator's host path: hx_apply_host_staged, which streams
    pageable arrays through a pinned ring with host worker threads (page-
    locked ones go straight to the copy engines).  Host-synchronous."""
    if op.n_el == 0:
        return dst
    if chunk_el is None:
        chunk_el = host_chunk_elements(op, STAGED_CHUNK_BYTES)
    work = _device_work(op, chunk_el)
    with _staging_lock:
        stage = _staging_buffer(op, chunk_el)
        _native.check(_native.lib().hx_apply_host_staged(
            op.plan.handle, _native.ptr(src), _native.ptr(op.device_factors),
            _native.ptr(dst), op.n_el, chunk_el, _native.ptr(work), _native.ptr(stage),
            _native.ptr(flag), stream), "hx_apply_host_staged")
    return dst


def apply_host(op, src, dst, flag=None, stream=None, chunk_el=None, work=None, overlap=False):
    """End-to-end apply on host arrays through ``hx_apply_host`` (asynchronous on
    ``stream``; pass page-locked arrays for full copy/compute overlap).

    ``overlap=True`` (HX_HOST_OVERLAP) pipelines back-to-back calls: the call
    does not wait for earlier work on ``stream``, its uploads and kernels run
    under the previous call's downloads.  Only for streaming callers that
    guarantee ``src`` is final, nobody touches ``src`` / ``dst`` until the
    stream passes the call, and ``work`` belongs to this operator alone
    (include/hexbench_b200.h, hx_apply_host_ex)."""
    if stream is None:
        stream = _stream(op.device)
    return _apply_host(op, src, dst, flag, stream, chunk_el, work, overlap)


def baseline_workspace(op):
    """Device scratch for apply_baseline (4 GL-point tensors per element)."""
    import torch

    nbytes = _native.lib().hx_apply_baseline_workspace(op.plan.handle, op.n_el)
    return torch.empty(max(1, nbytes // DOUBLE), dtype=torch.float64, device=op.device)


def apply_baseline_device(op, q, out, work, flag=None, stream=None):
    """Raw unfused apply (asynchronous, no allocation, no sync): see
    apply_baseline."""
    if stream is None:
        stream = _stream(op.device)
    _native.check(_native.lib().hx_apply_baseline(
        op.plan.handle, _native.ptr(q), _native.ptr(op.device_factors), _native.ptr(out),
        op.n_el, _native.ptr(work), _native.ptr(flag), stream), "hx_apply_baseline")


def apply_baseline(op, q, out=None, stream=None):
    """Unfused apply on device tensors: the paper's Kernel-1 structure
     -- one launch per contraction pass, intermediates through
    HBM, the pass order of operators.py:208-268 -- i.e. what the reference's
    ``variant="baseline"`` counters describe.  Same result as the fused
    kernels up to rounding; exists so the fused kernels can be measured
    against it (bench.py).  ``q``: (n_el, n_p) float64 CUDA tensor."""
    import torch

    if tuple(q.shape) != (op.n_el, op.n_p):
        raise ValueError("field vector shape does not match operator")
    out = torch.empty_like(q) if out is None else out
    flag = torch.zeros(1, dtype=torch.int32, device=q.device)
    apply_baseline_device(op, q, out, baseline_workspace(op), flag, stream)
    if int(flag.item()) & _native.HX_FLAG_NONFINITE:
        raise ValueError("field vector contains non-finite values")
    return out


def apply_bp1(op, q, counters=None, threads=1):
    if op.bp != BP1:
        raise ValueError("operator is not BP1.0")
    return apply_operator(op, q, counters, threads)


def apply_bp35(op, q, counters=None, threads=1):
    if op.bp != BP35:
        raise ValueError("operator is not BP3.5")
    return apply_operator(op, q, counters, threads)


def apply_bp3(op, q, counters=None, threads=1):
    if op.bp != BP3:
        raise ValueError("operator is not BP3.0")
    return apply_operator(op, q, counters, threads)


def _interp_entries(interp):
    mat = interp.entries if hasattr(interp, "entries") else np.asarray(interp, dtype=float)
    mat = np.ascontiguousarray(mat, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1] + 1:
        raise ValueError("interp must be an (N+2) x (N+1) GLL -> GL matrix")
    check_degree(mat.shape[1] - 1)
    return mat


def _interp_elements(x, interp, project):
    """Shared body of interpolate_to_gl / project_to_gll: one batched kernel
    launch (``hx_interp_elements``) over every element tensor in ``x``."""
    import torch

    mat = _interp_entries(interp)
    m, n = mat.shape
    src_n, dst_n = (m, n) if project else (n, m)
    on_dev = _is_torch(x)
    shape = tuple(x.shape)
    if len(shape) < 3 or shape[-3:] != (src_n,) * 3:
        raise ValueError(
            f"expected element tensors of shape (..., {src_n}, {src_n}, {src_n}), got {shape}")
    batch = shape[:-3]
    n_el = int(np.prod(batch)) if batch else 1
    if on_dev:
        if not x.is_cuda:
            raise ValueError("torch tensors must live on a CUDA device")
        dev = x.device
        src = x.to(torch.float64).contiguous().view(n_el, src_n ** 3)
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
        src = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).reshape(
            n_el, src_n ** 3)).to(dev)
    with torch.cuda.device(dev):
        dst = torch.empty((n_el, dst_n ** 3), dtype=torch.float64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        _native.check(_native.lib().hx_interp_elements(
            n - 1, _native.ptr(mat), int(project), _native.ptr(src), _native.ptr(dst), n_el,
            _native.ptr(flag), _stream(dev)), "hx_interp_elements")
        if int(flag.item()) & _native.HX_FLAG_NONFINITE:
            raise ValueError("element tensor contains non-finite values")
    dst = dst.view(*batch, dst_n, dst_n, dst_n)
    return dst if on_dev else dst.cpu().numpy()


def interpolate_to_gl(q_e, interp):
    """Pure interpolation of element tensors from GLL to GL nodes (reference
    operators.py:352-356): ``(..., n, n, n) -> (..., m, m, m)``, contracting
    axes 1, 2, 0 of each element with ``interp`` (an OperatorMatrix or an
    (N+2) x (N+1) array).  numpy in -> numpy out (through the device);
    a torch CUDA tensor stays on its device.  Any number of leading batch
    axes: one kernel launch for all of them."""
    return _interp_elements(q_e, interp, project=False)


def project_to_gll(t_e, interp):
    """Transpose interpolation of element tensors from GL back to GLL
    (reference operators.py:359-364): ``(..., m, m, m) -> (..., n, n, n)``."""
    return _interp_elements(t_e, interp, project=True)
