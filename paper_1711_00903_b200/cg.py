"""Conjugate gradients on the element matvecs -- the operator's real caller
(the paper's benchmarks are the inner kernel of a CG
Poisson solve).  The reference package has no solver; this
module is new and exercises the multi-GPU dot-product path.

Per iteration, all on the device and without a host synchronisation:

  1. beta, p = r + beta p,      one fused kernel (hx_apply_energy_dir): the
     Ap = A p and <p, A p>      direction update rides the matvec's first load
  2. alpha, x, r, <r, r>        hx_cg_update

Every iteration has the same form: the solve starts from p = 0 with the
previous <r, r> slot set to 1, so the first direction is p = r + rr * 0 = r
exactly.  ``fuse_direction=False`` runs step 1 as hx_cg_direction followed
by hx_apply_energy -- the same arithmetic, bit for bit (tests/test_gpu_cg.py).

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


def _host_staged(t, group):
    """gloo (the CPU test backend) takes host tensors: stage device data
    through the host there; NCCL works on the device tensors directly."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _allreduce(t, group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if _host_staged(t, group):
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _direction_apply(op, w, ap, cur, flag, strm, fused):
    """Step 1: p = r + (rr[cur] / rr[1 - cur]) p, then ap = A p, pap = <p, A p>."""
    L, ptr = _native.lib(), _native.ptr
    if fused:
        _native.check(L.hx_apply_energy_dir(op.plan.handle, ptr(w.p), ptr(w.r), ptr(w.rr[cur]),
                                            ptr(w.rr[1 - cur]), ptr(op.device_factors), ptr(ap),
                                            op.n_el, ptr(w.partials), w.npart, ptr(w.pap),
                                            ptr(flag), strm), "hx_apply_energy_dir")
        return
    _native.check(L.hx_cg_direction(ptr(w.p), ptr(w.r), w.p.numel(), ptr(w.rr[cur]),
                                    ptr(w.rr[1 - cur]), strm), "hx_cg_direction")
    _native.check(L.hx_apply_energy(op.plan.handle, ptr(w.p), ptr(op.device_factors), ptr(ap),
                                    op.n_el, ptr(w.partials), w.npart, ptr(w.pap), ptr(flag),
                                    strm), "hx_apply_energy")


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

    def start(self):
        """p = 0 and the previous <r, r> slot = 1: the first (uniform) step's
        direction update yields p = r exactly (rr[0] must hold <r, r>)."""
        self.p.zero_()
        self.rr[1].fill_(1.0)


def cg_solve(op, b, x0=None, tol=1e-10, maxiter=500, check_every=10, group=None, work=None,
             graph=False, fuse_direction=True):
    """Solve A x = b for a device-resident right-hand side.

    ``op`` is an OperatorInstance (or this rank's ShardedOperator.op); ``b`` a
    float64 CUDA tensor of shape (op.n_el, op.n_p).  Converged when
    ||r|| <= tol * ||b|| (checked every ``check_every`` iterations).
    ``graph=True`` (single process): the iterations between two checks run as
    one captured CUDA graph (see AssembledCG); same iterates bit for bit, the
    iteration count rounded up to whole blocks.  ``fuse_direction``: see the
    module docstring.
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
    cur = 0
    _native.check(L.hx_dot(ptr(w.r), ptr(w.r), n, ptr(w.partials), w.npart, ptr(w.rr[cur]),
                           stream), "hx_dot")
    _allreduce(w.rr[cur], group)
    w.start()
    bb = torch.zeros(1, dtype=torch.float64, device=dev)
    _native.check(L.hx_dot(ptr(b), ptr(b), n, ptr(w.partials), w.npart, ptr(bb), stream))
    _allreduce(bb, group)
    target = tol * float(bb.sqrt().item())
    norms = [float(w.rr[cur].sqrt().item())]
    if norms[0] <= target:
        return CGResult(x, 0, True, norms)
    it = 0
    converged = False

    def step(c, strm):
        nx = 1 - c
        _direction_apply(op, w, w.ap, c, flag, strm, fuse_direction)
        _allreduce(w.pap, group)
        _native.check(L.hx_cg_update(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), n, ptr(w.rr[c]),
                                     ptr(w.pap), ptr(w.partials), w.npart, ptr(w.rr[nx]),
                                     strm), "hx_cg_update")
        _allreduce(w.rr[nx], group)
        return nx

    import torch.distributed as dist
    if graph and not (dist.is_available() and dist.is_initialized()):
        k = check_every + (check_every % 2)

        def block():
            c, strm = 0, _stream(dev)
            for _ in range(k):
                c = step(c, strm)

        run = block  # first block eager (first-launch setup), then captured
        while it < maxiter:
            run()
            it += k
            norms.append(float(w.rr[0].sqrt().item()))
            if norms[-1] <= target:
                converged = True
                break
            if run is block:
                run = _graphed(block)
    else:
        while it < maxiter:
            nxt = step(cur, stream)
            it += 1
            if it % check_every == 0 or it == maxiter:
                norms.append(float(w.rr[nxt].sqrt().item()))
                if norms[-1] <= target:
                    converged = True
                    break
            cur = nxt
    if int(flag.item()) & _native.HX_FLAG_NONFINITE:
        raise ValueError("non-finite values during the CG solve")
    return CGResult(x, it, converged, norms)


def cg_iterations(op, b, iterations, work, stream=None, fuse_direction=True):
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
    cur = 0
    L.hx_dot(ptr(w.r), ptr(w.r), n, ptr(w.partials), w.npart, ptr(w.rr[cur]), stream)
    w.start()
    for _ in range(iterations):
        nxt = 1 - cur
        _direction_apply(op, w, w.ap, cur, None, stream, fuse_direction)
        L.hx_cg_update(ptr(x), ptr(w.p), ptr(w.r), ptr(w.ap), n, ptr(w.rr[cur]), ptr(w.pap),
                       ptr(w.partials), w.npart, ptr(w.rr[nxt]), stream)
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
#
# Multi-GPU: rank r owns the reference chunking's element range [lo, hi)
# (shard.partition).  The gathered vector (A p) additionally needs the
# elements that share a node with the range -- at most side^2 + side + 1
# either side, owned by the neighbouring ranks -- so each iteration exchanges
# those halos with the two neighbours (point-to-point send/recv, NCCL over
# NVLink on GPUs) between the matvec and the update kernel.  Every copy of a
# shared node then sums the same values in the same order on every rank, so
# the ranks' representatives stay bitwise consistent.


def _check_cube(u, n_el, degree):
    if u.numel() != n_el * (degree + 1) ** 3:
        raise ValueError(f"vector has {u.numel()} entries, expected {n_el} elements of "
                         f"{(degree + 1) ** 3} nodes")


class AssembledShard:
    """This rank's piece of the assembled cube-mesh system: own elements
    [lo, hi) plus the halo range [base, top) the gather-scatter reads."""

    def __init__(self, side, degree, rank=0, world_size=1, group=None):
        from .shard import partition

        self.side, self.degree = side, degree
        self.rank, self.world_size, self.group = rank, world_size, group
        n_el = side ** 3
        parts = partition(n_el, world_size)
        self.lo, self.hi = parts[rank]
        self.halo = side * side + side + 1
        if world_size > 1 and min(h - l for l, h in parts) < self.halo:
            raise ValueError(f"every rank needs >= side^2 + side + 1 = {self.halo} elements "
                             f"(the halo must come from the direct neighbours)")
        self.base = max(0, self.lo - self.halo)
        self.top = min(n_el, self.hi + self.halo)
        self.n_own = self.hi - self.lo
        self.n_pad = self.top - self.base

    def padded(self, like):
        """Zeroed (n_pad, n_p) buffer on like's device."""
        import torch
        return torch.zeros((self.n_pad, like.shape[-1]), dtype=like.dtype, device=like.device)

    def own(self, pad):
        """View of the own elements inside a padded buffer."""
        return pad[self.lo - self.base: self.hi - self.base]

    def exchange(self, pad):
        """Fill the halo rows of ``pad`` from the neighbouring ranks (their own
        rows), sending ours to them.  No-op on one rank."""
        if self.world_size == 1:
            return
        import torch.distributed as dist

        o0, o1 = self.lo - self.base, self.hi - self.base
        n_send = min(self.halo, self.n_own)
        # (peer, receive view, send view): halo below from / own head to rank-1,
        # halo above from / own tail to rank+1
        links = []
        if self.rank > 0:
            links.append((self.rank - 1, pad[:o0], pad[o0:o0 + n_send]))
        if self.rank < self.world_size - 1:
            links.append((self.rank + 1, pad[o1:], pad[o1 - n_send:o1]))
        staged = _host_staged(pad, self.group)
        ops, recvs = [], []
        for peer, rview, sview in links:
            rbuf = rview.new_empty(rview.shape, device="cpu") if staged else rview
            if rbuf is not rview or not rview.is_contiguous():
                recvs.append((rview, rbuf))
            sbuf = sview.cpu() if staged else sview.contiguous()
            ops.append(dist.P2POp(dist.irecv, rbuf, peer, self.group))
            ops.append(dist.P2POp(dist.isend, sbuf, peer, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for rview, rbuf in recvs:
            rview.copy_(rbuf)


def gather_scatter(u, side, degree, mask_boundary=False, out=None, stream=None, shard=None):
    """``out = mask . Q Q^T u`` on device: every element-local copy of a global
    node receives the (bit-identical) sum over all its copies.  With a
    ``shard``, ``u`` is the rank's padded buffer (halos already exchanged)
    and ``out`` covers the own elements."""
    import torch

    sh = shard or AssembledShard(side, degree)
    _check_cube(u, sh.n_pad, degree)
    if out is None:
        out = torch.empty((sh.n_own, u.shape[-1]), dtype=u.dtype, device=u.device)
    stream = _stream(u.device) if stream is None else stream
    _native.check(_native.lib().hx_dss(_native.ptr(u), _native.ptr(out), side, degree,
                                       int(bool(mask_boundary)), sh.lo, sh.hi, sh.base,
                                       stream), "hx_dss")
    return out


def _global_sum(t, sh):
    if sh.world_size > 1:
        _allreduce(t, sh.group)


class _AssembledState:
    def __init__(self, op, side, b, mask_boundary, work, shard):
        import torch

        self.sh = shard or AssembledShard(side, op.degree)
        if op.n_el != self.sh.n_own:
            raise ValueError("operator does not cover this rank's element range")
        _check_cube(b, self.sh.n_own, op.degree)
        self.mask = int(bool(mask_boundary))
        self.w = work if work is not None else CGWorkspace(b)
        self.ap_pad = self.sh.padded(b)      # A p with halos
        self.x = torch.zeros_like(b)


def _assembled_setup(op, side, b, st, stream):
    """r = mask dss(b) (b exchanged through the halo buffer), <r, r>, p = 0
    (CGWorkspace.start: the first step's direction update gives p = r)."""
    L, ptr, sh, w = _native.lib(), _native.ptr, st.sh, st.w
    sh.own(st.ap_pad).copy_(b)
    sh.exchange(st.ap_pad)
    gather_scatter(st.ap_pad, side, op.degree, st.mask, out=w.r, stream=stream, shard=sh)
    _native.check(L.hx_dot_dss(ptr(w.r), ptr(w.r), side, op.degree, sh.lo, sh.hi,
                               ptr(w.partials), w.npart, ptr(w.rr[0]), stream), "hx_dot_dss")
    _global_sum(w.rr[0], sh)
    w.start()


def _assembled_step(op, side, st, cur, stream, flag=None, fused=True):
    """One CG iteration (direction update fused into the matvec); returns the
    index of the new <r, r> slot.  A p is assembled in place over the
    halo-padded buffer by the separable face passes, then read by the masked
    update (hx_cg_update_assembled)."""
    L, ptr, sh, w = _native.lib(), _native.ptr, st.sh, st.w
    nxt = 1 - cur
    _direction_apply(op, w, sh.own(st.ap_pad), cur, flag, stream, fused)
    _global_sum(w.pap, sh)
    sh.exchange(st.ap_pad)
    _native.check(L.hx_cg_update_assembled(ptr(st.x), ptr(w.p), ptr(w.r), ptr(st.ap_pad), side,
                                           op.degree, st.mask, sh.lo, sh.hi, sh.base, sh.top,
                                           ptr(w.rr[cur]), ptr(w.pap), ptr(w.partials), w.npart,
                                           ptr(w.rr[nxt]), stream), "hx_cg_update_assembled")
    _global_sum(w.rr[nxt], sh)
    return nxt


def _graphed(block):
    """Capture ``block`` (a sequence of launches on torch's current stream)
    into a CUDA graph and return its replay: a launch-bound loop (small
    meshes: ~10 us of Python + ctypes per launch against a few us of GPU
    work) becomes one graph launch per block."""
    import torch

    side_stream = torch.cuda.Stream()
    side_stream.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side_stream):
        with torch.cuda.graph(graph, stream=side_stream):
            block()
    torch.cuda.current_stream().wait_stream(side_stream)
    return graph.replay


class AssembledCG:
    """Reusable assembled-CG solver for ``mask Q^T A_L Q x = mask Q^T b`` on
    build_cube_mesh(side, extent) (see cg_solve_assembled).  Owns the device
    state; with ``graph=True`` (one GPU) the ``check_every`` iterations
    between two convergence checks are captured once, at construction, as a
    CUDA graph and every solve replays it -- bitwise the same iterates as the
    eager loop, one graph launch per block instead of ~7 launches per
    iteration (small meshes are launch-bound).  With a graph the iteration
    count is rounded up to whole blocks."""

    def __init__(self, op, side, mask_boundary=True, check_every=10, shard=None, graph=False,
                 work=None, fuse_direction=True):
        import torch

        self.op, self.side, self.check_every = op, side, check_every
        self.fused = fuse_direction
        self.dev = op.device
        like = torch.zeros((op.n_el, op.n_p), dtype=torch.float64, device=self.dev)
        self.st = _AssembledState(op, side, like, mask_boundary, work, shard)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.k = check_every + (check_every % 2)  # even: the rr slots return to slot 0
        self.replay = None
        if graph and self.st.sh.world_size == 1:
            # one eager block first (first-launch setup of every kernel), on a
            # throw-away right-hand side, then capture
            g = torch.Generator(device=self.dev).manual_seed(0)
            warm = torch.randn(like.shape, dtype=torch.float64, device=self.dev, generator=g)
            _assembled_setup(op, side, warm, self.st, _stream(self.dev))
            self._block()
            self.replay = _graphed(self._block)

    def _block(self):
        c = 0
        strm = _stream(self.dev)
        for _ in range(self.k):
            c = _assembled_step(self.op, self.side, self.st, c, strm, self.flag, self.fused)

    def solve(self, b, tol=1e-10, maxiter=1000):
        """Solve for the (rank's) element-local load vector ``b``; returns a
        CGResult (``x`` is the solver's own buffer: copy it to keep it)."""
        op, side, st = self.op, self.side, self.st
        w = st.w
        stream = _stream(self.dev)
        _check_cube(b, st.sh.n_own, op.degree)
        st.x.zero_()
        self.flag.zero_()
        _assembled_setup(op, side, b, st, stream)
        norm0 = float(w.rr[0].sqrt().item())
        target = tol * norm0
        norms = [norm0]
        if norm0 == 0.0:
            return CGResult(st.x, 0, True, norms)
        it, cur, converged = 0, 0, False
        if self.replay is not None:
            while it < maxiter:
                self.replay()
                it += self.k
                norms.append(float(w.rr[0].sqrt().item()))
                if norms[-1] <= target:
                    converged = True
                    break
        else:
            while it < maxiter:
                nxt = _assembled_step(op, side, st, cur, stream, self.flag, self.fused)
                it += 1
                if it % self.check_every == 0 or it == maxiter:
                    norms.append(float(w.rr[nxt].sqrt().item()))
                    if norms[-1] <= target:
                        converged = True
                        break
                cur = nxt
        if int(self.flag.item()) & _native.HX_FLAG_NONFINITE:
            raise ValueError("non-finite values during the CG solve")
        return CGResult(st.x, it, converged, norms)


def cg_solve_assembled(op, side, b, tol=1e-10, maxiter=1000, check_every=10,
                       mask_boundary=True, work=None, shard=None, graph=False,
                       fuse_direction=True):
    """Solve the assembled system ``mask Q^T A_L Q x = mask Q^T b`` by CG.

    ``op`` is an OperatorInstance on build_cube_mesh(side, extent) (perturbing
    the corners breaks conformity, so use the unperturbed mesh) -- or, with a
    ``shard`` (AssembledShard), this rank's ShardedOperator.op on its element
    range; ``b`` is the (rank's) element-local load vector, e.g. the BP1.0
    mass matvec of a nodal source.  Boundary nodes carry homogeneous Dirichlet
    conditions when ``mask_boundary`` (needed for BP3.5 / BP3.0 with
    lam = 0).  Returns a CGResult whose ``x`` is continuous (every copy of a
    global node holds the same value).  Per iteration: the fused matvec +
    <p, A p>, the halo exchange (multi-GPU), the gather-scatter of A p in
    place with three per-axis face passes, the update (plain read of the
    assembled A p, masked, multiplicity-weighted <r, r>); the direction
    update rides the next matvec (``fuse_direction``, module docstring).
    ``graph=True``: see AssembledCG (capturing costs ~40 ms, so
    reuse an AssembledCG for repeated solves)."""
    solver = AssembledCG(op, side, mask_boundary, check_every, shard, graph, work,
                         fuse_direction)
    return solver.solve(b, tol, maxiter)


def cg_iterations_assembled(op, side, b, iterations, work, mask_boundary=True, shard=None,
                            fuse_direction=True):
    """``iterations`` assembled-CG steps from x = 0 with no convergence checks
    or host synchronisation (the harness times this)."""
    stream = _stream(op.device)
    st = _AssembledState(op, side, b, mask_boundary, work, shard)
    _assembled_setup(op, side, b, st, stream)
    cur = 0
    for _ in range(iterations):
        cur = _assembled_step(op, side, st, cur, stream, None, fuse_direction)
    return st.x
