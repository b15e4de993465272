"""Scenario sharding across ranks (one process per GPU).

Each rank owns the contiguous scenario group `partition(N, world)[rank]`
(reference: partition, proj/core/src/executor.cpp:7-19) and one bipm_ctx on
its GPU.  The exchange is an all-reduce of device buffers inside the C++
solver: NCCL over NVLink/NVSwitch in production (`backend="nccl"`), or a
host-staged gloo all-reduce (`backend="gloo"`), which lets tests run several
ranks on one GPU.
"""
from __future__ import annotations

import numpy as np

from . import _native as nat

_OPS = {0: "SUM", 1: "MAX", 2: "MIN"}


def gloo_allreduce(group=None):
    """In-place all-reduce of a float64 numpy array with torch.distributed."""
    import torch
    import torch.distributed as dist

    def fn(arr: np.ndarray, op: int) -> None:
        t = torch.from_numpy(arr)
        dist.all_reduce(t, op=getattr(dist.ReduceOp, _OPS[int(op)]), group=group)

    return fn


def sharded_context(problem: nat.Problem, world: int, rank: int, device: int = 0,
                    backend: str = "nccl") -> nat.Context:
    lo, hi = nat.partition(problem.N, world)[rank]
    ctx = nat.Context(problem, device=device, lo=lo, hi=hi)
    if world > 1:
        if backend == "nccl":
            import torch.distributed as dist
            box = [nat.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            ctx.set_nccl(box[0], world, rank)
        elif backend == "gloo":
            ctx.set_host_comm(gloo_allreduce(), world, rank)
        else:
            raise ValueError(f"unknown backend {backend}")
    return ctx
