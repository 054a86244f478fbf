"""Frame sharding over ranks: frames are independent, so rank r of
W owns the contiguous global frame indices [r B, (r+1) B) and generates its
own shard from the per-frame seeds -- no input scatter and no data-path
collective.  The only collectives are the barrier around the timed region and
the max / sum reductions of the per-rank timings and counts (NCCL on GPUs,
gloo in the CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def frame_range(rank: int, world: int, frames_per_rank: int):
    """Weak scaling: every rank decodes frames_per_rank frames of its own contiguous slice."""
    assert 0 <= rank < world
    first = rank * frames_per_rank
    return first, frames_per_rank


def frame_range_strong(rank: int, world: int, total_frames: int):
    """Strong scaling: the job's total_frames split into contiguous slices whose sizes differ by
    at most one frame (the first total % world ranks take one more)."""
    assert 0 <= rank < world and total_frames >= 0
    base, extra = divmod(total_frames, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def _red_device(device):
    # NCCL reduces device tensors; gloo (CPU tests, functional multi-rank runs) host tensors
    return device if dist.get_backend() == "nccl" else None


def max_over_ranks(value: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_red_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_red_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(device=None):
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None and device.type == "cuda" and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()
