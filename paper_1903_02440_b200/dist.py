"""Multi-GPU bookkeeping for the spike-wave step.

Inference (C2, C5) shards by independent images: each rank owns a slice of the batch (strong
scaling) or a whole batch of its own (weak scaling, what bench.py reports); the only communication is
a barrier, the max / sum of the per-rank timings and unit counts, and an optional all-gather of the
per-image decisions (gather_decisions).  Sequential plasticity (C1, C3, C4) cannot shard by image
(each image's weights depend on the previous update): FeatureShardedSTDP splits the FEATURES of
the plastic layer over ranks instead, with one all-reduce(MIN) of packed inhibition keys per image
(SURVEY.md §8(e), f4).  One process per GPU, launched by torchrun; NCCL on GPUs, gloo on CPU (tests).
"""
from __future__ import annotations

import os
from typing import Callable, Optional, Tuple

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


def gather_decisions(decision: torch.Tensor) -> torch.Tensor:
    """All-gather of the per-image results of every rank (equal batch per rank), rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return decision
    world = dist.get_world_size()
    out = torch.empty((world,) + tuple(decision.shape), dtype=decision.dtype, device=decision.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, decision.contiguous())
    else:  # gloo has no all_gather_into_tensor
        dist.all_gather(list(out.unbind(0)), decision.contiguous())
    return out.reshape((-1,) + tuple(decision.shape[1:]))


def all_reduce_min(keys: torch.Tensor) -> torch.Tensor:
    """In-place MIN over ranks of the packed position keys (no-op on one process)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
    return keys


class GpuOps:
    """The libsnn calls one feature-sharded step makes (the product path; tests may substitute
    reference ops with the same signatures to exercise the orchestration on CPU)."""

    def __init__(self):
        from . import snn
        self.snn = snn

    def conv_fire(self, lat_in, w, pad, T, theta):
        return self.snn.conv_fire(lat_in, w, pad, T, theta)

    def position_keys(self, lat, v, f_offset):
        return self.snn.position_keys(lat, v, f_offset)

    def k_winners_keys(self, keys, F, k, r):
        return self.snn.k_winners_keys(keys, F, k, r)

    def stdp_update_shard(self, w, lat_in, pad, lat_out, winners, count, rates, f_offset):
        return self.snn.stdp_update(w, lat_in, pad, lat_out, winners, count, rates["a_plus"], rates["a_minus"],
                                    rates["lb"], rates["ub"], rates["stabilizer"], f_offset=f_offset)


class FeatureShardedSTDP:
    """f4: sequential STDP of one finite-threshold conv layer (conv+fire -> pointwise inhibition ->
    k-WTA -> STDP, image by image) with the layer's F features split over ``world`` ranks.

    Rank g holds w[f0:f1] (``shard(F, g, world)``).  Per image, ``keys`` runs the rank's conv and
    reduces each position to its best packed key (lat, v desc, f); the keys are MIN-reduced over
    ranks (``reduce``, default NCCL/gloo all-reduce); ``apply`` runs the k-WTA on the reduced map --
    the same on every rank -- and updates the rank's own winners.  Bit-identical to the one-GPU step
    (snn_inhibit + snn_k_winners + snn_stdp_update) because the inhibition minimum over all features
    is the minimum over ranks of the per-rank minima."""

    def __init__(self, spec, w_full: torch.Tensor, T: int, k: int, r: int, rates: dict, rank: int = 0,
                 world: int = 1, ops=None, reduce: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
        self.spec, self.T, self.k, self.r, self.rates = spec, T, k, r, rates
        self.F = int(w_full.shape[0])
        self.f0, self.f1 = shard(self.F, rank, world)
        self.w = w_full[self.f0:self.f1].clone().contiguous()
        self.ops = ops if ops is not None else GpuOps()
        self.reduce = reduce if reduce is not None else all_reduce_min
        self._lat = None

    def keys(self, lat_in: torch.Tensor) -> torch.Tensor:
        """lat_in [1, C, H, W] -> this rank's position keys [1, Ho, Wo] (before the reduction)."""
        s = self.spec
        self._lat, v = self.ops.conv_fire(lat_in, self.w, s.pad, self.T, s.theta)
        return self.ops.position_keys(self._lat, v, self.f0)

    def apply(self, lat_in: torch.Tensor, keys: torch.Tensor):
        """k-WTA on the reduced keys, then STDP of this rank's winners; returns (winners, count)."""
        win, cnt = self.ops.k_winners_keys(keys, self.F, self.k, self.r)
        self.ops.stdp_update_shard(self.w, lat_in[0], self.spec.pad, self._lat[0], win[0], cnt, self.rates, self.f0)
        return win, cnt

    def step(self, lat_in: torch.Tensor):
        return self.apply(lat_in, self.reduce(self.keys(lat_in)))
