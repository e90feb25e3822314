"""CPU: the multi-GPU host logic with world_size 2 over gloo (the GPU runs use
one process per GPU over NCCL; only the plumbing differs)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2012_13257_b200 import dist as gdist  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # batch sharding of B=64 images (weak/strong): disjoint cover
        s, e = gdist.shard_range(64, world, rank)
        t = torch.zeros(64)
        t[s:e] = 1.0
        dist.all_reduce(t)
        ok_cover = bool(torch.all(t == 1.0))
        # device time: max over ranks (timing rule)
        tmax = gdist.max_over_ranks(10.0 + rank)
        # huge image: bands + halo-point partial gradients summed over ranks
        rng = np.random.default_rng(0)
        H, cutoff = 64, 3.0
        pos_y = rng.uniform(-0.5, H - 0.5, 500)
        r0, r1 = gdist.band_rows(H, world, rank)
        mine = gdist.band_point_mask(pos_y, r0, r1, gdist.default_halo(cutoff))
        part = torch.tensor(mine.astype(np.float32))
        gdist.sum_over_ranks(part)
        nbands = gdist.halo_points(pos_y, H, world, gdist.default_halo(cutoff))
        ok_halo = bool(np.array_equal(part.numpy().astype(np.int32), nbands))
        out[rank] = (ok_cover, tmax, ok_halo, int((nbands > 1).sum()))
    finally:
        dist.destroy_process_group()


def _band_worker(rank, world, port, out):
    """configs[3] decomposition on CPU: every rank renders its row band from
    its halo points with the oracle (the reference restated), the shared
    points' partial gradients are SUM-reduced over gloo, and the result must
    equal the full-frame reference."""
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle.Oracle()
        rng = np.random.default_rng(5)
        W, H, N, C, sigma, cutoff = 48, 40, 900, 3, 1.0, 3.0
        pos = np.stack([rng.uniform(-0.5, W - 0.5, N), rng.uniform(-0.5, H - 0.5, N)], 1).astype(np.float32)
        col = rng.uniform(0, 1, (N, C)).astype(np.float32)
        up = rng.uniform(-1, 1, (H, W, C))
        full = orc.forward(pos, col, W, H, sigma, cutoff)
        rdc, rdp = orc.backward(pos, col, full, up, sigma, cutoff)
        plan = gdist.BandPlan(pos, H, world, rank, cutoff)
        bpos = plan.local_positions(pos)
        f = orc.forward(bpos, col[plan.idx], W, plan.rows, sigma, cutoff)
        dc, dp = orc.backward(bpos, col[plan.idx], f, up[plan.r0:plan.r1], sigma, cutoff)
        buf = torch.from_numpy(plan.shared_partials(dc, dp))
        gdist.sum_over_ranks(buf)
        g_col, g_pos = plan.assemble(dc, dp, buf.numpy(), N)
        rows_ok = bool(np.array_equal(f["image"], full["image"][plan.r0:plan.r1]))
        nofb = int(full["fallback_flag"].sum()) == 0
        mine = np.zeros(N, bool)
        mine[plan.idx[plan.owned_local]] = True
        mine[plan.shared] = True
        err_c = float(np.abs(g_col[mine] - rdc[mine]).max())
        err_p = float(np.abs(g_pos[mine] - rdp[mine]).max())
        out[rank] = (rows_ok, nofb, err_c, err_p, int(plan.shared.size))
    finally:
        dist.destroy_process_group()


def _hole_instance():
    """Density 0.25 (configs[3]'s), r = 3, with rows 10..30 empty except one
    point at y = 26: the fallback pixels of band 0's last rows have their
    nearest point in band 1's territory, 7+ rows past band 0's edge — beyond
    the default cutoff + 1 halo."""
    rng = np.random.default_rng(11)
    W, H, sigma, cutoff = 48, 40, 1.0, 3.0
    n = int(0.25 * W * H)
    pos = np.stack([rng.uniform(-0.5, W - 0.5, n), rng.uniform(-0.5, H - 0.5, n)], 1)
    pos = pos[(pos[:, 1] < 10) | (pos[:, 1] > 30)]
    pos = np.concatenate([pos, [[24.25, 26.0]]]).astype(np.float32)
    col = rng.uniform(0, 1, (pos.shape[0], 3)).astype(np.float32)
    up = rng.uniform(-1, 1, (H, W, 3))
    return pos, col, up, W, H, sigma, cutoff


def _band_fallback_worker(rank, world, port, out):
    """Band fallbacks against the full frame: the certified halo makes every
    band's nearest-point choice (and the routed gradient) the reference's."""
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle.Oracle()
        pos, col, up, W, H, sigma, cutoff = _hole_instance()
        N = pos.shape[0]
        full = orc.forward(pos, col, W, H, sigma, cutoff)
        rdc, rdp = orc.backward(pos, col, full, up, sigma, cutoff)

        def probe(plan):
            f = orc.forward(plan.local_positions(pos), col[plan.idx], W, plan.rows, sigma, cutoff)
            fb = np.nonzero(f["fallback_flag"].ravel())[0]
            return fb, f["nearest_index"].ravel()[fb]

        def reduce_max(v):
            t = torch.tensor([v], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        # the default halo alone gets band 0's fallbacks wrong
        naive = gdist.BandPlan(pos, H, world, rank, cutoff)
        nf = orc.forward(naive.local_positions(pos), col[naive.idx], W, naive.rows, sigma, cutoff)
        naive_near = np.where(nf["fallback_flag"] == 1, naive.idx[nf["nearest_index"]], -1)
        want_near = np.where(full["fallback_flag"] == 1, full["nearest_index"], -1)[naive.r0:naive.r1]
        naive_ok = bool(np.array_equal(naive_near, want_near))

        plan = gdist.resolve_band_plan(pos, W, H, world, rank, cutoff, probe, reduce_max)
        bpos = plan.local_positions(pos)
        f = orc.forward(bpos, col[plan.idx], W, plan.rows, sigma, cutoff)
        dc, dp = orc.backward(bpos, col[plan.idx], f, up[plan.r0:plan.r1], sigma, cutoff)
        near = np.where(f["fallback_flag"] == 1, plan.idx[f["nearest_index"]], -1)
        near_ok = bool(np.array_equal(near, want_near))
        rows_ok = bool(np.array_equal(f["image"], full["image"][plan.r0:plan.r1]))
        buf = torch.from_numpy(plan.shared_partials(dc, dp))
        gdist.sum_over_ranks(buf)
        g_col, g_pos = plan.assemble(dc, dp, buf.numpy(), N)
        mine = np.zeros(N, bool)
        mine[plan.idx[plan.owned_local]] = True
        mine[plan.shared] = True
        err_c = float(np.abs(g_col[mine] - rdc[mine]).max())
        err_p = float(np.abs(g_pos[mine] - rdp[mine]).max())
        nfb = int(f["fallback_flag"].sum())
        out[rank] = (naive_ok, near_ok, rows_ok, err_c, err_p, plan.halo, nfb)
    finally:
        dist.destroy_process_group()


def test_two_rank_band_fallbacks_match_full_frame():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_band_fallback_worker, args=(world, port, out), nprocs=world, join=True)
    assert not out[0][0], "instance does not exercise a far fallback across the band edge"
    halos = {out[r][5] for r in range(world)}
    assert len(halos) == 1 and halos.pop() > gdist.default_halo(3.0)
    for r in range(world):
        naive_ok, near_ok, rows_ok, err_c, err_p, halo, nfb = out[r]
        assert nfb > 0
        assert near_ok, "band nearest indices differ from the full frame"
        assert rows_ok, "band image rows differ from the full-frame reference"
        assert err_c < 1e-9 and err_p < 1e-9, (err_c, err_p)


def test_two_rank_band_split_matches_full_frame():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_band_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        rows_ok, nofb, err_c, err_p, n_shared = out[r]
        assert rows_ok, "band image rows differ from the full-frame reference"
        assert nofb
        assert err_c < 1e-9 and err_p < 1e-9, (err_c, err_p)
        assert n_shared > 0


def test_two_rank_sharding_and_reductions():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        ok_cover, tmax, ok_halo, n_shared = out[r]
        assert ok_cover
        assert tmax == 11.0
        assert ok_halo
        assert n_shared > 0  # points near the band boundary are shared


def test_shard_and_band_logic():
    for total in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            spans = [gdist.shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[k][1] == spans[k + 1][0] for k in range(world - 1))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    assert gdist.bands_cover(8192, 8)
    # a point exactly cutoff above a band still reaches its first row
    assert gdist.band_point_mask(np.array([10.0 - 3.0, 10.0 - 4.1]), 10, 20,
                                 gdist.default_halo(3.0)).tolist() == [True, False]
    assert gdist.weak_scaling_units(64, 8) == 512
    assert sum(gdist.strong_scaling_batch(64, 8, r) for r in range(8)) == 64


def _group_worker(rank, world, port, out):
    """The product driver's plumbing (paper_2012_13257_b200.multi.Group) on
    gloo: rank / world from the env, max-over-ranks timing, in-place SUM of a
    shared-gradient buffer, batch shards covering the global batch."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2012_13257_b200 import multi

    g = multi.Group("gloo")
    try:
        tmax = g.max_over_ranks(1.5 + rank)
        buf = torch.full((4, 5), float(rank + 1))
        g.sum_(buf)
        shards = multi.BatchShards(g, 64, 48, 1.0, 3.0)
        s, e = shards.local_range(64)
        t = torch.zeros(64)
        t[s:e] = 1.0
        g.sum_(t)
        g.barrier()
        out[rank] = (g.rank, g.world, tmax, float(buf[0, 0]), bool(torch.all(t == 1.0)))
    finally:
        g.close()


def test_product_driver_group_on_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_group_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        rank, w, tmax, s, cover = out[r]
        assert (rank, w) == (r, world)
        assert tmax == 2.5 and s == 3.0 and cover
