#!/usr/bin/env python3
"""BASELINE config 5: element-partitioned strong and weak scaling of all three
BPs at N=7 with the CG-style NCCL dot all-reduce, one process per GPU.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node G \
        --master-addr 127.0.0.1 --master-port 29511 tools/scaling.py [--out f]

strong: the side-92 cube (E = 778,688, 398.7 M DOF) split over the G ranks by
the reference's chunking (shard.partition); weak: 46^3 = 97,336 elements per
rank.  Per apply: the rank's fused kernel with <q, A q> fused
in (hx_apply_energy), then the 8-byte all-reduce (NCCL over NVLink) -- timed
on the device as the max over ranks.  One JSON line per (mode, bp) on rank 0.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1711_00903_b200 as hx  # noqa: E402
from paper_1711_00903_b200 import _native  # noqa: E402
from paper_1711_00903_b200.operators import _stream  # noqa: E402
from paper_1711_00903_b200.shard import ShardedOperator  # noqa: E402

DEG = 7


def max_over_ranks(v):
    dev = "cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run(mode, bp, rank, world, steps, warmup, strong_side=92, weak_side=46):
    if mode == "strong":
        mesh = hx.perturb_mesh(hx.build_cube_mesh(strong_side, 2.0), amplitude=0.15, seed=7)
        sh = ShardedOperator(bp, DEG, mesh, lam=1.0, rank=rank, world_size=world)
        op, total_el = sh.op, mesh.n_el
    else:
        mesh = hx.perturb_mesh(hx.build_cube_mesh(weak_side, 2.0), amplitude=0.15, seed=7 + rank)
        op, total_el = hx.make_operator(bp, DEG, mesh, lam=1.0), mesh.n_el * world
    q = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
    out = torch.empty_like(q)
    L = _native.lib()
    npart = L.hx_energy_partials()
    partials = torch.empty(npart, dtype=torch.float64, device="cuda")
    energy = torch.zeros(1, dtype=torch.float64, device="cuda")
    stream = _stream(op.device)

    def step():
        # A q and <q, A q> in one kernel (the dot is evaluated from the
        # kernel's quadrature-point values: no extra pass over q or A q),
        # then the 8-byte all-reduce across ranks
        _native.check(L.hx_apply_energy(op.plan.handle, _native.ptr(q),
                                        _native.ptr(op.device_factors), _native.ptr(out),
                                        op.n_el, _native.ptr(partials), npart,
                                        _native.ptr(energy), None, stream))
        if dist.is_initialized():
            if dist.get_backend() == "gloo":
                h = energy.cpu()
                dist.all_reduce(h)
                energy.copy_(h)
            else:
                dist.all_reduce(energy)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(s.elapsed_time(e) / steps)
    # the all-reduce alone (8 bytes), for the record
    torch.cuda._sleep(200_000)
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    part = torch.ones(1, dtype=torch.float64,
                      device="cpu" if dist.is_initialized() and dist.get_backend() == "gloo"
                      else "cuda")
    s2.record()
    for _ in range(steps):
        if dist.is_initialized():
            dist.all_reduce(part)
    e2.record()
    torch.cuda.synchronize()
    ar_us = max_over_ranks(s2.elapsed_time(e2) / steps * 1e3)
    nbytes = hx.traffic(bp, DEG, total_el).bytes_per_element * total_el
    rec = {"mode": mode, "bp": bp, "degree": DEG, "gpus": world, "n_el_total": total_el,
           "n_el_per_gpu_max": max_over_ranks(op.n_el), "dofs": total_el * op.n_p,
           "ms_per_apply_with_dot": ms, "gdof_per_s": total_el * op.n_p / (ms * 1e-3) / 1e9,
           "hbm_gb_per_s_total": nbytes / (ms * 1e-3) / 1e9,
           "gflop_per_s": hx.flop_model(bp, "fused", DEG) * total_el / (ms * 1e-3) / 1e9,
           "allreduce_8B_us": ar_us}
    del op, q, out
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default="strong,weak")
    ap.add_argument("--out", default=None)
    ap.add_argument("--strong-side", type=int, default=92)
    ap.add_argument("--weak-side", type=int, default=46)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1 or "MASTER_ADDR" in os.environ:
        backend = os.environ.get("HX_BENCH_BACKEND", "nccl")  # gloo: test-only, ranks share a GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    fh = open(args.out, "a") if (args.out and rank == 0) else None
    for mode in args.modes.split(","):
        for bp in hx.BENCHMARKS:
            rec = run(mode, bp, rank, world, args.steps, args.warmup, args.strong_side,
                      args.weak_side)
            if rank == 0:
                line = json.dumps(rec)
                print(line, flush=True)
                if fh:
                    fh.write(line + "\n")
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
