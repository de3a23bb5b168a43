"""Conjugate gradients on the element matvecs -- the operator's real caller
(the paper's benchmarks are the inner kernel of a CG
Poisson solve).  The reference package has no solver; this
module is new and exercises the multi-GPU dot-product path.

Per iteration, all on the device and without a host synchronisation:

  1. Ap = A p and <p, A p>      one fused kernel (hx_apply_energy)
  2. alpha, x, r, <r, r>        hx_cg_update
  3. beta, p                    hx_cg_direction

Under torch.distributed each rank owns a contiguous element range
(shard.partition) and the two scalars are all-reduced (8 bytes each, NCCL)
after steps 1 and 2.  The residual is read back every ``check_every``
iterations only.
"""

from dataclasses import dataclass, field

from . import _native
from .operators import _stream


@dataclass
class CGResult:
    x: object
    iterations: int
    converged: bool
    residual_norms: list = field(default_factory=list)  # ||r|| at each check


def _allreduce(t, group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


class CGWorkspace:
    """Device scratch of one solve: vectors p, r, Ap and the scalar slots."""

    def __init__(self, like):
        import torch
        self.p = torch.empty_like(like)
        self.r = torch.empty_like(like)
        self.ap = torch.empty_like(like)
        npart = _native.lib().hx_energy_partials()
        self.partials = torch.empty(npart, dtype=torch.float64, device=like.device)
        self.npart = npart
        # separate one-element tensors so each can be all-reduced on its own
        self.rr = [torch.zeros(1, dtype=torch.float64, device=like.device) for _ in range(2)]
        self.pap = torch.zeros(1, dtype=torch.float64, device=like.device)


def cg_solve(op, b, x0=None, tol=1e-10, maxiter=500, check_every=10, group=None, work=None):
    """Solve A x = b for a device-resident right-hand side.

    ``op`` is an OperatorInstance (or this rank's ShardedOperator.op); ``b`` a
    float64 CUDA tensor of shape (op.n_el, op.n_p).  Converged when
    ||r|| <= tol * ||b|| (checked every ``check_every`` iterations).
    """
    import torch

    L = _native.lib()
    ptr = _native.ptr
    dev = op.device
    n = b.numel()
    stream = _stream(dev)
    w = work if work is not None else CGWorkspace(b)
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    if x0 is None:
        w.r.copy_(b)
    else:  # r = b - A x0
        _native.check(L.hx_apply(op.plan.handle, ptr(x), ptr(op.device_factors), ptr(w.ap),
                                 op.n_el, ptr(flag), stream), "hx_apply")
        torch.sub(b, w.ap, out=w.r)
    w.p.copy_(w.r)
    cur = 0
    _native.check(L.hx_dot(ptr(w.r), ptr(w.r), n, ptr(w.partials), w.npart, ptr(w.rr[cur]),
                           stream), "hx_dot")
    _allreduce(w.rr[cur], group)
    bb = torch.zeros(1, dtype=torch.float64, device=dev)
    _native.check(L.hx_dot(ptr(b), ptr(b), n, ptr(w.partials), w.npart, ptr(bb), stream))
    _allreduce(bb, group)
    target = tol * float(bb.sqrt().item())
    norms = [float(w.rr[cur].sqrt().item())]
    if norms[0] <= target:
        return CGResult(x, 0, True, norms)
    it = 0
    converged = False
    while it < maxiter:
        nxt = 1 - cur
        _native.check(L.hx_apply_energy(op.plan.handle, ptr(w.p), ptr(op.device_factors),
                                        ptr(w.ap), op.n_el, ptr(w.partials), w.npart,
                                        ptr(w.pap), ptr(flag), stream), "hx_apply_energy")
        _allreduce(w.pap, group)
        _native.check(L.hx_cg_update(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), n, ptr(w.rr[cur]),
                                     ptr(w.pap), ptr(w.partials), w.npart, ptr(w.rr[nxt]),
                                     stream), "hx_cg_update")
        _allreduce(w.rr[nxt], group)
        it += 1
        if it % check_every == 0 or it == maxiter:
            norms.append(float(w.rr[nxt].sqrt().item()))
            if norms[-1] <= target:
                converged = True
                break
        _native.check(L.hx_cg_direction(ptr(w.p), ptr(w.r), n, ptr(w.rr[nxt]), ptr(w.rr[cur]),
                                        stream), "hx_cg_direction")
        cur = nxt
    if int(flag.item()) & _native.HX_FLAG_NONFINITE:
        raise ValueError("non-finite values during the CG solve")
    return CGResult(x, it, converged, norms)


def cg_iterations(op, b, iterations, work, stream=None):
    """Run exactly ``iterations`` CG steps from x = 0 without convergence
    checks or host synchronisation (the harness times this)."""
    import torch

    L = _native.lib()
    ptr = _native.ptr
    n = b.numel()
    stream = _stream(op.device) if stream is None else stream
    x = torch.zeros_like(b)
    w = work
    w.r.copy_(b)
    w.p.copy_(b)
    cur = 0
    L.hx_dot(ptr(w.r), ptr(w.r), n, ptr(w.partials), w.npart, ptr(w.rr[cur]), stream)
    for _ in range(iterations):
        nxt = 1 - cur
        L.hx_apply_energy(op.plan.handle, ptr(w.p), ptr(op.device_factors), ptr(w.ap),
                          op.n_el, ptr(w.partials), w.npart, ptr(w.pap), None, stream)
        L.hx_cg_update(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), n, ptr(w.rr[cur]), ptr(w.pap),
                       ptr(w.partials), w.npart, ptr(w.rr[nxt]), stream)
        L.hx_cg_direction(ptr(w.p), ptr(w.r), n, ptr(w.rr[nxt]), ptr(w.rr[cur]), stream)
        cur = nxt
    return x


# ---- assembled system on the structured cube mesh --------------------------
#
# The element operators above are block-diagonal (unassembled).  The Poisson /
# Helmholtz problem a CG solver actually targets couples elements through
# their shared nodes: A_G = Q^T A_L Q with Q the scatter from global nodes to
# element-local copies.  On the build_cube_mesh(side, extent) numbering
# (mesh.py:44-56) Q Q^T is a fixed-order gather (hx_dss), and CG runs on
# continuous element-local representatives (see csrc/hx_dss.cu).


def gather_scatter(u, side, degree, mask_boundary=False, out=None, stream=None):
    """``out = mask . Q Q^T u`` on device: every element-local copy of a global
    node receives the (bit-identical) sum over all its copies."""
    import torch

    if out is None:
        out = torch.empty_like(u)
    _check_cube(u, side, degree)
    stream = _stream(u.device) if stream is None else stream
    _native.check(_native.lib().hx_dss(_native.ptr(u), _native.ptr(out), side, degree,
                                       int(bool(mask_boundary)), stream), "hx_dss")
    return out


def _check_cube(u, side, degree):
    if u.numel() != side ** 3 * (degree + 1) ** 3:
        raise ValueError(f"vector has {u.numel()} entries, the side-{side} cube mesh at degree "
                         f"{degree} has {side ** 3 * (degree + 1) ** 3}")


def cg_solve_assembled(op, side, b, tol=1e-10, maxiter=1000, check_every=10,
                       mask_boundary=True, work=None):
    """Solve the assembled system ``mask Q^T A_L Q x = mask Q^T b`` by CG.

    ``op`` is an OperatorInstance on build_cube_mesh(side, extent) (perturbing
    the corners breaks conformity, so use the unperturbed mesh); ``b`` is an
    element-local load vector (for instance the BP1.0 mass matvec of a nodal
    source).  Boundary nodes carry homogeneous Dirichlet conditions when
    ``mask_boundary`` (needed for BP3.5 / BP3.0 with lam = 0).  Returns a
    CGResult whose ``x`` is continuous (every copy of a global node holds the
    same value).  Per iteration: the fused matvec + <p, A p>, then one update
    kernel that gathers A p across element copies on the fly (the assembled
    vector is never stored), then the direction update.
    """
    import torch

    L = _native.lib()
    ptr = _native.ptr
    deg = op.degree
    _check_cube(b, side, deg)
    if op.n_el != side ** 3:
        raise ValueError("operator mesh is not the side^3 cube mesh")
    dev = op.device
    stream = _stream(dev)
    n = b.numel()
    mask = int(bool(mask_boundary))
    w = work if work is not None else CGWorkspace(b)
    x = torch.zeros_like(b)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    gather_scatter(b, side, deg, mask_boundary, out=w.r, stream=stream)
    w.p.copy_(w.r)
    cur = 0
    _native.check(L.hx_dot_dss(ptr(w.r), ptr(w.r), side, deg, ptr(w.partials), w.npart,
                               ptr(w.rr[cur]), stream), "hx_dot_dss")
    target = tol * float(w.rr[cur].sqrt().item())
    norms = [float(w.rr[cur].sqrt().item())]
    if norms[0] == 0.0:
        return CGResult(x, 0, True, norms)
    it = 0
    converged = False
    while it < maxiter:
        nxt = 1 - cur
        _native.check(L.hx_apply_energy(op.plan.handle, ptr(w.p), ptr(op.device_factors),
                                        ptr(w.ap), op.n_el, ptr(w.partials), w.npart,
                                        ptr(w.pap), ptr(flag), stream), "hx_apply_energy")
        _native.check(L.hx_cg_update_dss(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), side, deg, mask,
                                         ptr(w.rr[cur]), ptr(w.pap), ptr(w.partials), w.npart,
                                         ptr(w.rr[nxt]), stream), "hx_cg_update_dss")
        it += 1
        if it % check_every == 0 or it == maxiter:
            norms.append(float(w.rr[nxt].sqrt().item()))
            if norms[-1] <= target:
                converged = True
                break
        _native.check(L.hx_cg_direction(ptr(w.p), ptr(w.r), n, ptr(w.rr[nxt]), ptr(w.rr[cur]),
                                        stream), "hx_cg_direction")
        cur = nxt
    if int(flag.item()) & _native.HX_FLAG_NONFINITE:
        raise ValueError("non-finite values during the CG solve")
    return CGResult(x, it, converged, norms)


def cg_iterations_assembled(op, side, b, iterations, work, mask_boundary=True, stream=None):
    """``iterations`` assembled-CG steps from x = 0 with no convergence checks
    or host synchronisation (the harness times this)."""
    import torch

    L = _native.lib()
    ptr = _native.ptr
    deg = op.degree
    n = b.numel()
    stream = _stream(op.device) if stream is None else stream
    mask = int(bool(mask_boundary))
    x = torch.zeros_like(b)
    w = work
    gather_scatter(b, side, deg, mask_boundary, out=w.r, stream=stream)
    w.p.copy_(w.r)
    cur = 0
    L.hx_dot_dss(ptr(w.r), ptr(w.r), side, deg, ptr(w.partials), w.npart, ptr(w.rr[cur]), stream)
    for _ in range(iterations):
        nxt = 1 - cur
        L.hx_apply_energy(op.plan.handle, ptr(w.p), ptr(op.device_factors), ptr(w.ap),
                          op.n_el, ptr(w.partials), w.npart, ptr(w.pap), None, stream)
        L.hx_cg_update_dss(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), side, deg, mask,
                           ptr(w.rr[cur]), ptr(w.pap), ptr(w.partials), w.npart,
                           ptr(w.rr[nxt]), stream)
        L.hx_cg_direction(ptr(w.p), ptr(w.r), n, ptr(w.rr[nxt]), ptr(w.rr[cur]), stream)
        cur = nxt
    return x
