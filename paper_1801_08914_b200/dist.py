"""Multi-process plumbing of the weak-scaling run (bench.py under torchrun).

The hot path shards by independent meshes (replicas) or by cells with no
data-path exchange, so the only collectives are control-plane:
a barrier around the timed region and the max-over-ranks of the device time.
These helpers are backend-agnostic (NCCL on the GPU box, gloo in the CPU
tests, tests/test_dist_cpu.py).
"""
from __future__ import annotations

import os
from typing import Sequence

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def replica_seed(base: int, rank: int) -> int:
    """Seed of a rank's replica inputs: distinct per rank, reproducible."""
    return base + 7919 * rank


def shard(n_units: int, world_size: int, rank: int) -> range:
    """Contiguous, balanced share of n_units (cells, slabs or meshes) for a rank."""
    q, r = divmod(n_units, world_size)
    lo = rank * q + min(rank, r)
    return range(lo, lo + q + (1 if rank < r else 0))


def _device() -> torch.device:
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def reduce_max(values: Sequence[float] | float):
    """Element-wise max over ranks (identity without a process group)."""
    scalar = not isinstance(values, (list, tuple))
    vals = [float(values)] if scalar else [float(v) for v in values]
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor(vals, dtype=torch.float64, device=_device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = [float(v) for v in t.cpu()]
    return vals[0] if scalar else vals


def reduce_sum(values: Sequence[float] | float):
    scalar = not isinstance(values, (list, tuple))
    vals = [float(values)] if scalar else [float(v) for v in values]
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor(vals, dtype=torch.float64, device=_device())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        vals = [float(v) for v in t.cpu()]
    return vals[0] if scalar else vals


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
