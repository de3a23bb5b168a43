"""Element partitioning across GPUs (one process per GPU, torch.distributed).

The three matvecs are block-diagonal -- "no communication is required
between elements" -- so a rank owns a contiguous element range
and applies its operator with no data-path collective.  The partition is the
reference's own chunking, ``np.linspace(0, E, G+1).astype(int)``
(operators.py:324-325), so a gathered multi-GPU result is bitwise identical
to the single-GPU one (the analogue of the thread-invariance criterion,
test_acceptance.py:210-224).

The only collective is the optional CG-style inner product: per-rank partial
sums reduced with one 8-byte NCCL all-reduce (``global_dot``).
"""

import numpy as np

from .mesh import HexMesh


def partition(n_el, world_size):
    """Contiguous [lo, hi) element range of every rank (reference chunking)."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    b = np.linspace(0, n_el, world_size + 1).astype(int)
    return [(int(lo), int(hi)) for lo, hi in zip(b[:-1], b[1:])]


def shard_mesh(mesh, rank, world_size):
    lo, hi = partition(mesh.n_el, world_size)[rank]
    return HexMesh(hi - lo, mesh.vertices[lo:hi], mesh.extent), (lo, hi)


def global_dot(u, v, group=None):
    """<u, v> over all ranks: local float64 dot, then all_reduce(SUM).
    u, v are torch tensors on the rank's device (or CPU under gloo)."""
    import torch
    import torch.distributed as dist

    part = torch.dot(u.reshape(-1), v.reshape(-1)).reshape(1)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part


def gather_field(local, n_el_total, world_size, group=None):
    """All-gather per-rank (n_local, n_p) blocks into the global (E, n_p) array
    in rank order (ranges from ``partition``)."""
    import torch
    import torch.distributed as dist

    ranges = partition(n_el_total, world_size)
    width = max(hi - lo for lo, hi in ranges)
    n_p = local.shape[1]
    pad = torch.zeros((width, n_p), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world_size)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: hi - lo] for b, (lo, hi) in zip(bufs, ranges)])


class ShardedOperator:
    """This rank's share of a global operator: make_operator on the local
    element range, on the rank's GPU."""

    def __init__(self, bp, degree, mesh, lam=0.0, variant="fused", rank=0, world_size=1,
                 device=None):
        from .operators import make_operator

        self.rank, self.world_size = rank, world_size
        self.n_el_total = mesh.n_el
        local, self.range = shard_mesh(mesh, rank, world_size)
        self.op = make_operator(bp, degree, local, lam=lam, variant=variant, device=device)

    def apply_device(self, q_local, out_local, flag=None, stream=None):
        from .operators import apply_device

        apply_device(self.op, q_local, out_local, flag, stream)
