"""Multi-GPU host logic: one process per GPU (torchrun), torch.distributed
only as plumbing.

The batched configs shard independent images across ranks with no data-path
collective; timing is taken on the device and reduced as
the max over ranks.  A single huge image (BASELINE configs[3]) is split into
row bands; a rank renders its band from the points whose disks reach it
(halo of the cutoff radius) and the partial gradients of points shared by two
bands are summed across ranks.  Pure index logic lives here so it can be
tested on CPU with the gloo backend.
"""
from __future__ import annotations

import math

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) of `total` units for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def band_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Row band [r0, r1) of an output frame for `rank`."""
    return shard_range(height, world, rank)


def band_point_mask(pos_y: np.ndarray, r0: int, r1: int, cutoff: float) -> np.ndarray:
    """Points whose closed ball of radius `cutoff` can touch a pixel row in
    [r0, r1): |mu_y - y| <= cutoff for some integer y in the band."""
    lo = r0 - cutoff - 1.0
    hi = (r1 - 1) + cutoff + 1.0
    return (pos_y >= lo) & (pos_y <= hi)


def halo_points(pos_y: np.ndarray, height: int, world: int, cutoff: float) -> np.ndarray:
    """Number of bands each point contributes to (>1: its gradient is a sum of
    per-band partials and needs the cross-rank reduction)."""
    n = np.zeros(pos_y.shape[0], np.int32)
    for r in range(world):
        r0, r1 = band_rows(height, world, r)
        n += band_point_mask(pos_y, r0, r1, cutoff)
    return n


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar across ranks (the timing rule of the bench)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(array, device=None):
    """In-place SUM all-reduce of a tensor (halo-gradient reduction)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(array, op=dist.ReduceOp.SUM)
    return array


def weak_scaling_units(batch_per_rank: int, world: int) -> int:
    """Images processed by the whole job when every rank runs a fixed batch."""
    return batch_per_rank * world


def strong_scaling_batch(global_batch: int, world: int, rank: int) -> int:
    s, e = shard_range(global_batch, world, rank)
    return e - s


def bands_cover(height: int, world: int) -> bool:
    rows = [band_rows(height, world, r) for r in range(world)]
    return rows[0][0] == 0 and rows[-1][1] == height and all(
        rows[k][1] == rows[k + 1][0] for k in range(world - 1))


def ceil_div(a: int, b: int) -> int:
    return -(-a // b) if b else math.inf
