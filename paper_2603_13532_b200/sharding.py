"""Summand sharding across GPUs.

The two summand loops of the reference (src/sketch.cpp:103-143 and :155-169) are
independent per summand, so each rank owns a contiguous block of summands, builds
the partial sketches Y and the partial projected core h for it, and the library
sums them with ncclAllReduce inside ts_krp_sum (after stages C and F2).  The QR,
ST-HOSVD and output GEMM run replicated; every rank returns the same result.
"""
from __future__ import annotations

from typing import Sequence, Tuple

from .tucksum import Engine


def shard_range(count: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block [begin, end) of `count` summands for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad world/rank")
    begin = count * rank // world
    end = count * (rank + 1) // world
    return begin, end


def shard(items: Sequence, world: int, rank: int):
    b, e = shard_range(len(items), world, rank)
    return items[b:e]


def init_nccl_engine(device: int, rank: int, world: int) -> Engine:
    """Creates the rank's Engine and joins the library's NCCL communicator.

    The 128-byte ncclUniqueId is produced on rank 0 and broadcast with
    torch.distributed (plumbing only; the all-reduces run inside the library on
    the engine's stream)."""
    import torch.distributed as dist

    eng = Engine(device)
    if world > 1:
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.init_nccl(obj[0], world, rank)
    return eng


def gloo_allreduce(buf):
    """Host all-reduce hook over torch.distributed (e.g. gloo): sums the numpy
    buffer over the ranks in place."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(buf)
    dist.all_reduce(t)


def init_host_engine(device: int, rank: int, world: int) -> Engine:
    """The rank's Engine with the host all-reduce hook (ts_ctx_set_host_allreduce)
    over the default torch.distributed group instead of NCCL: the same sharded
    ts_krp_sum orchestration, exchanges through host memory."""
    eng = Engine(device)
    if world > 1:
        eng.set_host_allreduce(gloo_allreduce, world, rank)
    return eng
