"""Multi-GPU bookkeeping for the spike-wave step.

The path shards only by independent images (inference configs C2, C5): each rank owns a slice of
the batch (strong scaling) or a whole batch of its own (weak scaling, what bench.py reports), and
there is no data-path collective -- the only communication is a barrier and the max / sum of the
per-rank timings and unit counts.  Sequential plasticity (C1, C3, C4) does not shard: each rank runs
an independent replica.  One process per GPU, launched by torchrun; NCCL on GPUs, gloo on CPU (tests).
"""
from __future__ import annotations

import os
from typing import Tuple

import torch
import torch.distributed as dist


def env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl", device=None) -> None:
    rank, world, _ = env()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) slice of ``total`` independent images for ``rank`` (sizes differ by
    at most one; every image is owned by exactly one rank)."""
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def _reduce(x: float, op, device) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, device="cpu") -> float:
    """Max over ranks (the job's time is the slowest rank's device time)."""
    return _reduce(x, dist.ReduceOp.MAX, device)


def sum_over_ranks(x: float, device="cpu") -> float:
    """Sum over ranks (images processed by the whole job)."""
    return _reduce(x, dist.ReduceOp.SUM, device)


def barrier() -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def job_throughput(units_this_rank: int, time_s_this_rank: float, device="cpu") -> float:
    """Whole-job throughput: units of all ranks / max-over-ranks time (bench.py's ``value``)."""
    units = sum_over_ranks(units_this_rank, device)
    t = max_over_ranks(time_s_this_rank, device)
    return units / t if t > 0 else float("nan")
