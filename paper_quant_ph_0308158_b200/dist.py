"""Host-side multi-process helpers (one process per GPU, torch.distributed).

The path partitions by output range -- the paper's "continuous portions"
 and "trade-off between number of parallel processors and size of
memory": rank r owns outputs [start_r, start_r + count_r) and needs
all of k1 (replicated).  bench.py runs one independent replica per GPU
("scaling": "weak"); `output_shards` is the strong-scaling partition used
with the ``*_range`` calls.  No data-path collective: the only collectives
are the timing reduction (max over ranks) and barriers.
"""
from __future__ import annotations

import os


def env_rank() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def output_shards(N: int, world: int, align: int = 1024) -> list[tuple[int, int]]:
    """Split [0, N) into `world` contiguous ranges, boundaries aligned to
    `align` entries where possible (whole 1024-entry walk tiles), covering
    [0, N) exactly once, in rank order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = -(-N // align)                     # ceil
    out = []
    for r in range(world):
        a = (units * r) // world * align
        b = (units * (r + 1)) // world * align
        a, b = min(a, N), min(b, N)
        out.append((a, b - a))
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the bench's per-step time)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
