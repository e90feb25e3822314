"""Multi-GPU driver of the hot path: one process
per GPU, the package's device API on each, ``torch.distributed`` (NCCL over
NVLink) as plumbing only.

Two decompositions, both mirroring the reference's single-image contract
(engine.cpp:107-176 forward, 238-309 backward) per shard:

* ``BatchShards`` — batched configs (BASELINE configs[1], [2], [4]): images
  are independent, each rank renders and differentiates its own images, no
  collective on the data path (weak scaling).  ``gather`` collects results on
  one rank when a caller wants them there (timed separately: it moves far
  more bytes than the step computes).
* ``BandSplit`` — one huge image (configs[3]): rank k renders the row band
  [r0, r1) from the points a band keeps (``dist.BandPlan``: every point whose
  disk reaches the band, plus whatever far nearest-point fallbacks need,
  certified by ``dist.resolve_band_plan``), and the partial gradients of the
  points kept by several bands are SUM-reduced with one NCCL all-reduce of a
  compact [shared, C + 2] buffer.  Band images are bit-identical to the
  full-frame rows (same points in the same ascending order, y shifted by an
  integer); shared gradients are sums of per-band partials.

Launch: ``torchrun --nproc-per-node N`` (or ``launch()`` below) with
RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the env.  A
single process (no env) is a group of one.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np

from . import Context, forward_counts  # noqa: F401  (re-export for callers)
from . import dist as gdist


def _torch():
    import torch
    import torch.distributed as tdist
    return torch, tdist


class Group:
    """This process's GPU, its ``Context`` on a dedicated stream, and the
    process group (NCCL) when there is more than one rank."""

    def __init__(self, backend: str = "nccl"):
        torch, tdist = _torch()
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        if self.world > 1 and not tdist.is_initialized():
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                tdist.init_process_group("nccl", init_method="env://",
                                         device_id=torch.device("cuda", self.local))
            else:
                tdist.init_process_group(backend, init_method="env://")
        self.device = torch.device("cuda", self.local) if backend == "nccl" else None
        self._ctx = None
        self._stream = None

    # ---- device plumbing (lazy: CPU tests use only the collectives) ----
    @property
    def stream(self):
        if self._stream is None:
            torch, _ = _torch()
            torch.cuda.set_device(self.local)
            self._stream = torch.cuda.Stream(device=self.device)
        return self._stream

    @property
    def ctx(self) -> Context:
        if self._ctx is None:
            self._ctx = Context(self.local)
            self._ctx.set_stream(self.stream.cuda_stream)
        return self._ctx

    # ---- collectives ----
    def barrier(self) -> None:
        _, tdist = _torch()
        if self.world > 1:
            tdist.barrier()

    def max_over_ranks(self, value: float) -> float:
        """Max of a scalar across ranks (device times: the slowest rank)."""
        torch, tdist = _torch()
        if self.world == 1:
            return float(value)
        t = torch.tensor([float(value)], device=self.device)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def sum_(self, tensor):
        """In-place SUM all-reduce (on this group's stream for NCCL)."""
        torch, tdist = _torch()
        if self.world > 1:
            if self.device is not None:
                with torch.cuda.stream(self.stream):
                    tdist.all_reduce(tensor, op=tdist.ReduceOp.SUM)
            else:
                tdist.all_reduce(tensor, op=tdist.ReduceOp.SUM)
        return tensor

    def close(self) -> None:
        _, tdist = _torch()
        if self._ctx is not None:
            self._ctx.synchronize()
        if self.world > 1 and tdist.is_initialized():
            tdist.destroy_process_group()


class BatchShards:
    """Batch sharding: rank k owns images [b0, b1) of a global batch (or a
    fixed per-rank batch under weak scaling) and runs the reference's
    forward + backward on them with no cross-rank traffic."""

    def __init__(self, group: Group, width: int, height: int, sigma: float, cutoff: float,
                 fallback: str = "nearest"):
        self.g = group
        self.width, self.height = int(width), int(height)
        self.sigma, self.cutoff = float(sigma), float(cutoff)
        self.fallback = 0 if fallback == "nearest" else 1

    def local_range(self, global_batch: int) -> tuple[int, int]:
        return gdist.shard_range(global_batch, self.g.world, self.g.rank)

    def forward(self, pos, col, image):
        """gmi_forward on this rank's device arrays (B x N x 2, B x N x C,
        image B x H x W x C) -> ForwardCache."""
        B, N, C = int(col.shape[0]), int(col.shape[1]), int(col.shape[2])
        return self.g.ctx.forward_device(pos, col, B, N, C, self.width, self.height,
                                         self.sigma, self.cutoff, self.fallback, image)

    def backward(self, pos, col, cache, upstream, d_col, d_pos) -> None:
        B, N, C = int(col.shape[0]), int(col.shape[1]), int(col.shape[2])
        self.g.ctx.backward_device(pos, col, B, N, C, self.width, self.height, self.sigma,
                                   self.cutoff, self.fallback, cache, upstream, d_col, d_pos)

    def step(self, pos, col, upstream, image, d_col, d_pos, forward_only: bool = False):
        cache = self.forward(pos, col, image)
        if not forward_only:
            self.backward(pos, col, cache, upstream, d_col, d_pos)
        return cache

    def gather(self, tensor, dst: int = 0):
        """All ranks' shards of `tensor` (equal shapes) stacked on rank `dst`
        (None elsewhere): the optional result collection of SURVEY §8e."""
        torch, tdist = _torch()
        if self.g.world == 1:
            return tensor
        parts = [torch.empty_like(tensor) for _ in range(self.g.world)] if self.g.rank == dst else None
        with torch.cuda.stream(self.g.stream):
            tdist.gather(tensor, parts, dst=dst)
        return torch.cat(parts, 0) if parts is not None else None


class BandSplit:
    """One huge image split into row bands across the ranks (configs[3]).

    Every rank holds the full point set on the host (the plan needs every
    y); it keeps its band's points on the device and renders rows [r0, r1).
    ``step`` = band forward + band backward + the NCCL SUM of the shared
    points' partial gradients."""

    def __init__(self, group: Group, positions: np.ndarray, colors: np.ndarray, width: int,
                 height: int, sigma: float, cutoff: float, fallback: str = "nearest"):
        torch, _ = _torch()
        self.g = group
        self.width, self.height = int(width), int(height)
        self.sigma, self.cutoff = float(sigma), float(cutoff)
        self.fallback = 0 if fallback == "nearest" else 1
        pos = np.ascontiguousarray(positions, np.float32)
        col = np.ascontiguousarray(colors, np.float32)
        self.N_full, self.C = pos.shape[0], col.shape[1]
        dev = group.device

        def upload(plan):
            with torch.cuda.stream(group.stream):
                lp = torch.from_numpy(plan.local_positions(pos)).to(dev).unsqueeze(0).contiguous()
                lc = torch.from_numpy(col[plan.idx]).to(dev).unsqueeze(0).contiguous()
            return lp, lc

        def probe(plan):
            # the band forward on the plan's points: its fallback pixels and
            # the band-local nearest point each chose
            if self.fallback != 0:
                return np.zeros(0, np.int64), np.zeros(0, np.int64)
            lp, lc = upload(plan)
            with torch.cuda.stream(group.stream):
                img = torch.empty(1, plan.rows, self.width, self.C, device=dev)
            cache = group.ctx.forward_device(lp, lc, 1, int(plan.idx.size), self.C, self.width,
                                             plan.rows, self.sigma, self.cutoff, 0, img)
            group.ctx.synchronize()
            _, flag, near = cache.pixels()
            fb = np.nonzero(flag[0].ravel())[0]
            return fb, near[0].ravel()[fb]

        reduce_max = group.max_over_ranks if group.world > 1 else None
        self.plan = gdist.resolve_band_plan(pos, self.width, self.height, group.world, group.rank,
                                            self.cutoff, probe, reduce_max)
        self.pos, self.col = upload(self.plan)
        self.N = int(self.plan.idx.size)
        with torch.cuda.stream(group.stream):
            sl = torch.from_numpy(self.plan.shared_local).to(dev)
            self._li = sl.clamp(min=0)
            self._have = (sl >= 0).float().unsqueeze(1)
            self.shared_buf = torch.zeros(self.plan.shared.size, self.C + 2, device=dev)
            self.image = torch.empty(1, self.plan.rows, self.width, self.C, device=dev)
            self.d_col = torch.empty(1, self.N, self.C, device=dev)
            self.d_pos = torch.empty(1, self.N, 2, device=dev)
        group.stream.synchronize()

    @property
    def rows(self) -> tuple[int, int]:
        return self.plan.r0, self.plan.r1

    def step(self, upstream_band):
        """Band forward + backward (upstream rows [r0, r1), 1 x rows x W x C on
        the device) + the shared-gradient SUM.  Returns the cache; outputs are
        in self.image, self.d_col / self.d_pos (band-local points) and
        self.shared_buf (the reduced gradients of the shared points)."""
        torch, _ = _torch()
        ctx, p = self.g.ctx, self.plan
        cache = ctx.forward_device(self.pos, self.col, 1, self.N, self.C, self.width, p.rows,
                                   self.sigma, self.cutoff, self.fallback, self.image)
        ctx.backward_device(self.pos, self.col, 1, self.N, self.C, self.width, p.rows, self.sigma,
                            self.cutoff, self.fallback, cache, upstream_band, self.d_col,
                            self.d_pos)
        with torch.cuda.stream(self.g.stream):
            self.shared_buf[:, :self.C] = self.d_col[0].index_select(0, self._li) * self._have
            self.shared_buf[:, self.C:] = self.d_pos[0].index_select(0, self._li) * self._have
        self.g.sum_(self.shared_buf)
        return cache

    def gradients(self):
        """Host full-size gradients as this rank holds them: its own points
        and every shared point (reduced); other ranks' points are zero."""
        self.g.stream.synchronize()
        return self.plan.assemble(self.d_col[0].cpu().numpy(), self.d_pos[0].cpu().numpy(),
                                  self.shared_buf.cpu().numpy(), self.N_full)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(nproc: int, argv: list[str], env: dict | None = None) -> int:
    """Runs `python argv...` as `nproc` ranks on this node (torchrun, one
    process per GPU, rendezvous on 127.0.0.1) and returns the exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", *argv]
    return subprocess.call(cmd, env={**os.environ, **(env or {})})
