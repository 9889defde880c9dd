"""Multi-GPU plumbing for the stream-sharded path: one process per GPU, each
owning its own sensor streams; no collective on the data path. torch.distributed
is used only to line ranks up and to take the max of the timed regions
(the slowest rank defines the job's time)."""
from __future__ import annotations

import os


def env():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def stream_range(streams_per_rank: int, rank: int):
    """Global ids of the streams a rank owns (weak scaling: a fixed count per
    GPU, contiguous blocks)."""
    return range(rank * streams_per_rank, (rank + 1) * streams_per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed seconds); identity when not
    distributed."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: float, world: int, max_seconds: float) -> float:
    """Whole-job units/s: every rank's units over the slowest rank's time."""
    return units_per_rank * world / max_seconds
