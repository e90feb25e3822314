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


def default_halo(cutoff: float) -> float:
    """Rows beyond a band a point may sit and still reach it: the cutoff
    (closed ball, bin_grid.cpp:98) plus one row of slack."""
    return float(cutoff) + 1.0


def band_point_mask(pos_y: np.ndarray, r0: int, r1: int, halo: float) -> np.ndarray:
    """Points a band keeps: mu_y in [r0 - halo, r1 - 1 + halo].  With the
    default halo (cutoff + 1) that is every point whose closed ball can touch
    a pixel row in [r0, r1) (|mu_y - y| <= cutoff for an integer y there);
    a wider halo also keeps the candidates of far nearest-point fallbacks."""
    lo = r0 - halo
    hi = (r1 - 1) + halo
    return (pos_y >= lo) & (pos_y <= hi)


def halo_points(pos_y: np.ndarray, height: int, world: int, halo: float) -> np.ndarray:
    """Number of bands each point belongs to (>1: its gradient is a sum of
    per-band partials and needs the cross-rank reduction)."""
    n = np.zeros(pos_y.shape[0], np.int32)
    for r in range(world):
        r0, r1 = band_rows(height, world, r)
        n += band_point_mask(pos_y, r0, r1, halo)
    return n


def band_points(pos_y: np.ndarray, r0: int, r1: int, halo: float) -> np.ndarray:
    """Ascending indices of the points a rank keeps for rows [r0, r1).  The
    ascending order keeps the reference's per-pixel summation order
    (engine.cpp:59-72 sums in ascending point index) and its nearest-point
    tie rule (smallest index, bin_grid.cpp:114-164)."""
    return np.nonzero(band_point_mask(pos_y, r0, r1, halo))[0]


def shared_points(pos_y: np.ndarray, height: int, world: int, halo: float) -> np.ndarray:
    """Ascending indices of the points kept by two or more bands: the only
    gradients that need a cross-rank reduction."""
    return np.nonzero(halo_points(pos_y, height, world, halo) > 1)[0]


class BandPlan:
    """One rank's share of a single huge image (BASELINE configs[3]): its row
    band, the points it renders (with their band-local positions: y shifted
    by -r0, exact in fp32 for integer r0 within the frame) and where the
    globally shared points sit in its local arrays."""

    def __init__(self, pos: np.ndarray, height: int, world: int, rank: int, cutoff: float,
                 halo: float | None = None):
        self.r0, self.r1 = band_rows(height, world, rank)
        self.cutoff = float(cutoff)
        self.halo = default_halo(cutoff) if halo is None else float(halo)
        if self.halo < default_halo(cutoff):
            raise ValueError("halo must be >= cutoff + 1")
        self.idx = band_points(pos[:, 1], self.r0, self.r1, self.halo)
        self.shared = shared_points(pos[:, 1], height, world, self.halo)
        # local slot of each shared point on this rank (-1: not in this band)
        where = np.full(pos.shape[0], -1, np.int64)
        where[self.idx] = np.arange(self.idx.size)
        self.shared_local = where[self.shared]
        # points this rank owns outright (in no other band)
        owned = np.ones(self.idx.size, bool)
        owned[self.shared_local[self.shared_local >= 0]] = False
        self.owned_local = np.nonzero(owned)[0]

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    def halo_needed(self, pos: np.ndarray, fb_pixels: np.ndarray, fb_nearest: np.ndarray,
                    width: int) -> float:
        """The halo under which this band's nearest-point fallbacks are the
        full frame's (bin_grid.cpp:114-164: argmin over ALL points, ties to
        the smallest index).  `fb_pixels` are band-local pixel ids (r * W + c)
        of the band's fallback pixels and `fb_nearest` the band-local point
        each one chose.  A point the band does not keep lies more than
        m = min(y - (r0 - halo), (r1 - 1 + halo) - y) rows from pixel row y,
        so a local choice at distance d <= m is the global one (ties
        included: every point at distance <= m is kept).  Returns the current
        halo when every choice is certified, else the smallest halo that
        certifies the worst one (plus one row)."""
        if len(fb_pixels) == 0:
            return self.halo
        fb_pixels = np.asarray(fb_pixels, np.int64)
        near = self.idx[np.asarray(fb_nearest, np.int64)]
        qx = (fb_pixels % width).astype(np.float64)
        qy = (fb_pixels // width + self.r0).astype(np.float64)
        p = np.asarray(pos, np.float64)[near]
        d = np.sqrt((qx - p[:, 0]) ** 2 + (qy - p[:, 1]) ** 2)
        inner = np.minimum(qy - self.r0, (self.r1 - 1) - qy)  # rows to the band edge
        m = inner + self.halo
        # certified with a relative guard for the f64 distance itself
        bad = d * (1.0 + 1e-12) + 1e-9 > m
        if not bad.any():
            return self.halo
        return float(np.ceil(np.max(d[bad] - inner[bad])) + 1.0)

    def local_positions(self, pos: np.ndarray) -> np.ndarray:
        p = np.array(pos[self.idx], dtype=pos.dtype, copy=True)
        p[:, 1] -= p.dtype.type(self.r0)
        return p

    def shared_partials(self, d_col: np.ndarray, d_pos: np.ndarray) -> np.ndarray:
        """[len(shared), C + 2] partial gradients of the shared points (zeros
        for the ones outside this band), the buffer the ranks SUM-reduce."""
        C = d_col.shape[1]
        buf = np.zeros((self.shared.size, C + 2), d_col.dtype)
        have = self.shared_local >= 0
        buf[have, :C] = d_col[self.shared_local[have]]
        buf[have, C:] = d_pos[self.shared_local[have]]
        return buf

    def assemble(self, d_col: np.ndarray, d_pos: np.ndarray, reduced: np.ndarray, n: int):
        """Full-size gradients as this rank holds them: its owned points and
        every shared point (reduced); other ranks' owned points stay zero."""
        C = d_col.shape[1]
        g_col = np.zeros((n, C), d_col.dtype)
        g_pos = np.zeros((n, 2), d_pos.dtype)
        own = self.idx[self.owned_local]
        g_col[own] = d_col[self.owned_local]
        g_pos[own] = d_pos[self.owned_local]
        g_col[self.shared] = reduced[:, :C]
        g_pos[self.shared] = reduced[:, C:]
        return g_col, g_pos


def resolve_band_plan(pos: np.ndarray, width: int, height: int, world: int, rank: int,
                      cutoff: float, probe, reduce_max=None, max_rounds: int = 4) -> "BandPlan":
    """The band plan whose nearest-point fallbacks equal the full frame's.

    `probe(plan)` renders the band (the device forward on the plan's local
    points) and returns (band-local fallback pixel ids, band-local nearest
    point of each).  Every rank certifies its fallbacks (BandPlan.halo_needed);
    the halo is the max over ranks (`reduce_max`, identity for one process) so
    that all ranks agree on the kept and shared point sets.  One widening
    certifies every fallback: the widened halo keeps the previous choice and
    puts the band edge beyond it, and a closer point found there is closer
    still."""
    reduce_max = reduce_max or (lambda v: v)
    halo = default_halo(cutoff)
    for _ in range(max_rounds):
        plan = BandPlan(pos, height, world, rank, cutoff, halo)
        fb_pix, fb_near = probe(plan)
        need = float(reduce_max(plan.halo_needed(pos, fb_pix, fb_near, width)))
        if need <= halo:
            return plan
        halo = need
    raise RuntimeError("band halo did not converge")


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
