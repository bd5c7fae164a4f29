"""Multi-GPU work split for the sharded configs.

Batch GS targets and OSPR jobs are independent, so every rank owns whole
units and there is no data-path collective; the only collective is the final
gather of per-unit errors to rank 0 (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, start + count) of `total` units for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def unit_seeds(first_unit: int, count: int, seed0: int = 1) -> np.ndarray:
    """Seeds of units first_unit .. first_unit+count-1 (BASELINE: seed = 1 + t)."""
    return np.arange(seed0 + first_unit, seed0 + first_unit + count, dtype=np.uint64)


def gather_to_root(values, dist, world: int, rank: int):
    """Gather equally-sized 1-D tensors to rank 0 in rank order (None elsewhere)."""
    import torch
    if world == 1:
        return values
    out = [torch.empty_like(values) for _ in range(world)] if rank == 0 else None
    dist.gather(values, out, dst=0)
    return torch.cat(out) if rank == 0 else None
