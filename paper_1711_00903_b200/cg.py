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
