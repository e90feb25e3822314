"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact: bin grid (origin, n_cols, n_rows, bin_start, point_index), fallback
set, nearest indices, per-pixel contribution counts.  Tolerance (north star):
|a-b| <= 1e-6 + 1e-5*max(|a|,|b|) for image, d_colors, d_positions.
Inputs are fp32-representable so both sides see identical values.
"""
import numpy as np
import pytest

from conftest import assert_close

pytestmark = pytest.mark.gpu


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def run_gpu(gmi, ctx, pos, col, w, h, sigma, cutoff, up=None, fallback="nearest"):
    pos = np.asarray(pos, np.float32).reshape(1, -1, 2)
    col = np.asarray(col, np.float32).reshape(1, pos.shape[1], -1)
    img, cache = gmi.forward_batch(pos, col, w, h, sigma, cutoff, fallback, ctx=ctx)
    out = dict(image=img[0], cache=cache)
    if up is not None:
        dc, dp = gmi.backward_batch(pos, col, cache, np.asarray(up, np.float32)[None], sigma,
                                    cutoff, fallback, ctx=ctx)
        out.update(dc=dc[0], dp=dp[0])
    return out


def check_instance(gmi, ctx, orc, pos, col, w, h, sigma, cutoff, fallback=0, seed=0,
                   counts=True):
    pos = f32(pos)
    col = f32(col)
    rng = np.random.default_rng(seed)
    up = f32(rng.uniform(-1, 1, (h, w, col.shape[1])))
    fb = "nearest" if fallback == 0 else "zero"
    g = run_gpu(gmi, ctx, pos, col, w, h, sigma, cutoff, up, fb)
    r = orc.forward(pos, col, w, h, sigma, cutoff, fallback)
    rdc, rdp = orc.backward(pos, col, r, up, sigma, cutoff, fallback)
    norm, flag, near = g["cache"].pixels()
    assert np.array_equal(flag[0], r["fallback_flag"]), "fallback set differs"
    assert np.array_equal(near[0], np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)
                          if fallback == 0 else np.full_like(near[0], -1)), "nearest differs"
    if counts:
        cnt = gmi.forward_counts(g["cache"])
        assert np.array_equal(cnt[0], r["counts"]), "per-pixel contribution counts differ"
    assert_close(g["image"], r["image"], what="image")
    ok = ~np.isnan(norm[0]) & (r["fallback_flag"] == 0)
    assert_close(norm[0][ok], r["normalizer"][ok], what="normalizer")
    assert_close(g["dc"], rdc, what="d_colors")
    assert_close(g["dp"], rdp, what="d_positions")
    return g, r


# ---------------------------------------------------------------- KATs ----
def test_three_point_mixture(gmi, ctx):
    # test_engine.cpp:53-70: e^-0.25/(e^-0.25 + 2e^-1.25) at q=(0.5,0.5)
    ps = gmi.PointSet([[-0.5, -0.5], [1.5, -0.5], [-0.5, 1.5]], [[1.0], [0.0], [0.0]])
    img, cache = gmi.forward(ps, 1, 1, 1.0, radius=10.0)
    assert img[0, 0, 0] == pytest.approx(0.5761168847658291, rel=1e-6)


def test_single_point_paints_everywhere(gmi, ctx):
    # test_engine.cpp:26-40
    ps = gmi.PointSet([[3.7, -2.1]], [[0.7]])
    img, cache = gmi.forward(ps, 5, 4, 1.0)
    assert np.allclose(img, 0.7, rtol=1e-6, atol=0)
    norm, flag, near = cache.pixels()
    assert cache.fallback_count == int((flag == 1).sum())


def test_equidistant_two_points(gmi, ctx):
    # test_engine.cpp:42-51
    ps = gmi.PointSet([[0, 1], [2, 1]], [[0.2], [0.8]])
    img, _ = gmi.forward(ps, 3, 3, 1.0)
    assert img[1, 1, 0] == pytest.approx(0.5, rel=1e-6)


@pytest.mark.parametrize("fallback,value", [("nearest", 0.9), ("zero", 0.0)])
def test_fallback_out_of_range(gmi, ctx, fallback, value):
    # test_engine.cpp:217-239
    ps = gmi.PointSet([[100, 100], [200, 200]], [[0.9], [0.1]])
    img, cache = gmi.forward(ps, 4, 4, 1.0, radius=2.0, fallback=fallback)
    assert cache.fallback_count == 16
    assert np.all(img == np.float32(value).astype(np.float64))


def test_total_underflow_falls_back(gmi, ctx):
    # test_engine.cpp:241-249
    ps = gmi.PointSet([[1000.0, 0.0]], [[0.6]])
    img, cache = gmi.forward(ps, 1, 1, 0.5, radius=10000.0)
    assert cache.fallback_count == 1
    assert img[0, 0, 0] == np.float64(np.float32(0.6))


def test_backward_single_point_unit_upstream(gmi, ctx):
    # test_engine.cpp:302-311
    ps = gmi.PointSet([[2, 2]], [[0.5]])
    img, cache = gmi.forward(ps, 6, 5, 1.0, radius=100.0)
    dc, dp = gmi.backward(ps, cache, np.ones((5, 6, 1)), 1.0, radius=100.0)
    assert dc[0, 0] == pytest.approx(30.0, rel=1e-6)
    assert abs(dp[0, 0]) < 1e-6 and abs(dp[0, 1]) < 1e-6


def test_fallback_gradient_routing(gmi, ctx):
    # test_engine.cpp:347-370
    ps = gmi.PointSet([[-50, 0], [-60, 0]], [[0.3], [0.7]])
    img, cache = gmi.forward(ps, 2, 2, 1.0, radius=3.0)
    assert cache.fallback_count == 4
    dc, dp = gmi.backward(ps, cache, np.ones((2, 2, 1)), 1.0, radius=3.0)
    assert dc[0, 0] == 4.0 and dc[1, 0] == 0.0
    assert np.all(dp == 0.0)
    img0, cache0 = gmi.forward(ps, 2, 2, 1.0, radius=3.0, fallback="zero")
    dc0, dp0 = gmi.backward(ps, cache0, np.ones((2, 2, 1)), 1.0, radius=3.0, fallback="zero")
    assert np.all(dc0 == 0.0) and np.all(dp0 == 0.0)


def test_cache_mismatch_and_validation(gmi, ctx):
    # test_engine.cpp:372-400, core.cpp:55-120
    ps = gmi.PointSet([[0.5, 0.5], [3.0, 1.0]], [[0.5], [0.25]])
    img, cache = gmi.forward(ps, 4, 4, 1.0)
    with pytest.raises(gmi.GmiError) as e:
        gmi.backward(ps, cache, np.ones((4, 4, 1)), 2.0, radius=6.0)
    assert e.value.name == "CacheMismatch"
    with pytest.raises(gmi.GmiError):
        gmi.backward(ps, cache, np.ones((5, 4, 1)), 1.0)
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward(ps, 0, 5, 1.0)
    assert e.value.name == "InvalidDimensions"
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward(ps, 4, 4, -1.0, radius=3.0)
    assert e.value.name == "ConfigInvalid"
    # device-side validation of raw batch arrays
    pos = np.zeros((1, 3, 2), np.float32)
    col = np.full((1, 3, 1), 0.5, np.float32)
    pos[0, 2, 0] = np.nan
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward_batch(pos, col, 4, 4, 1.0, ctx=ctx)
    assert e.value.name == "NonFiniteValue" and "index 2" in str(e.value)
    pos[0, 2, 0] = 1.0
    col[0, 1, 0] = 1.5
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward_batch(pos, col, 4, 4, 1.0, ctx=ctx)
    assert e.value.name == "ColorOutOfRange" and "index 1" in str(e.value)


# ------------------------------------------------------------- binning ----
@pytest.mark.parametrize("n,extent,cell", [(4096, 128, 3.0), (5000, 8192, 3.0), (1, 10, 1.0),
                                           (3000, 64, 0.37), (20000, 300, 4.5)])
def test_bin_grid_bit_exact(gmi, ctx, orc, n, extent, cell):
    rng = np.random.default_rng(n)
    pos = f32(rng.uniform(-0.5, extent - 0.5, (n, 2)))
    got = gmi.bin_grid(pos, cell, ctx=ctx)
    want = orc.bin_grid(pos, cell)
    assert np.array_equal(got["origin"], want["origin"])
    assert (got["n_cols"], got["n_rows"]) == (want["n_cols"], want["n_rows"])
    assert np.array_equal(got["bin_start"], want["bin_start"])
    assert np.array_equal(got["point_index"], want["point_index"])


def test_bin_grid_clustered_big_cells(gmi, ctx, orc):
    rng = np.random.default_rng(5)
    pos = f32(np.concatenate([rng.uniform(0, 400, (3000, 2)), rng.uniform(100, 103, (9000, 2)),
                              np.full((20, 2), 7.0)]))
    got = gmi.bin_grid(pos, 12.0, ctx=ctx)
    want = orc.bin_grid(pos, 12.0)
    assert np.array_equal(got["bin_start"], want["bin_start"])
    assert np.array_equal(got["point_index"], want["point_index"])


# ------------------------------------------------- forward + backward ----
@pytest.mark.parametrize("seed", [21, 22, 23, 24, 31, 77])
def test_random_instances_truncated(gmi, ctx, orc, seed):
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(1, 30)), int(rng.integers(1, 30))
    n = int(rng.integers(1, 60))
    ch = int(rng.choice([1, 3]))
    pos = np.stack([rng.uniform(-1, w, n), rng.uniform(-1, h, n)], 1)
    col = rng.uniform(0, 1, (n, ch))
    sigma = float(rng.uniform(0.5, 4.0))
    for cutoff in (3 * sigma, 1.0, 2.5):
        for fb in (0, 1):
            check_instance(gmi, ctx, orc, pos, col, w, h, sigma, cutoff, fb, seed)


def test_config1_shape(gmi, ctx, orc):
    pos, col, up = orc.synth_batch(1, 1, 4096, 3, 128, 128)
    check_instance(gmi, ctx, orc, pos[0], col[0], 128, 128, 1.0, 3.0)


def test_sparse_with_many_fallbacks(gmi, ctx, orc):
    pos, col, up = orc.synth_batch(3, 1, 2000, 3, 256, 256)
    check_instance(gmi, ctx, orc, pos[0], col[0], 256, 256, 1.0, 3.0)


@pytest.mark.parametrize("ch", [1, 2, 5, 9])
def test_channel_counts(gmi, ctx, orc, ch):
    pos, col, up = orc.synth_batch(9, 1, 3000, ch, 96, 80)
    check_instance(gmi, ctx, orc, pos[0], col[0], 96, 80, 1.5, 4.5)


def test_integer_lattice_exact_ties(gmi, ctx, orc):
    # integer positions at r=3: d^2 == r^2 exactly for many pairs (closed ball)
    xs, ys = np.meshgrid(np.arange(0, 40, 3), np.arange(0, 30, 3))
    pos = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float64)
    rng = np.random.default_rng(1)
    col = rng.uniform(0, 1, (pos.shape[0], 3))
    check_instance(gmi, ctx, orc, pos, col, 40, 30, 1.0, 3.0)
    check_instance(gmi, ctx, orc, pos + 0.5, col, 40, 30, 1.0, 3.0)


@pytest.mark.parametrize("ch,sigma", [(3, 1.3), (1, 0.7), (4, 2.1)])
def test_near_boundary_ties(gmi, ctx, orc, ch, sigma):
    # every point within ~1e-5 r^2 of the ball boundary of some pixel (fp32
    # rounding of the position keeps it in that band): the K1 ambiguity flag
    # must route each decision the fp32 test could get wrong to the f64
    # predicate, so per-pixel counts stay bit-exact
    rng = np.random.default_rng(int(sigma * 10) + ch)
    r = 3.0 * sigma
    n = 1500
    q = rng.integers(4, 60, (n, 2)).astype(np.float64)
    th = rng.uniform(0, 2 * np.pi, n)
    eps = rng.uniform(-4e-6, 4e-6, n)
    pos = q + (r * (1.0 + eps))[:, None] * np.stack([np.cos(th), np.sin(th)], 1)
    col = rng.uniform(0, 1, (n, ch))
    check_instance(gmi, ctx, orc, pos, col, 64, 64, sigma, r)


def test_duplicates_and_single_pixel(gmi, ctx, orc):
    pos = np.array([[1, 1], [1, 1], [1, 1], [0.25, 0.75]], np.float64)
    col = np.array([[0.1], [0.2], [0.3], [0.9]])
    check_instance(gmi, ctx, orc, pos, col, 3, 3, 1.0, 2.0)
    check_instance(gmi, ctx, orc, pos, col, 1, 1, 1.0, 2.0)


def test_huge_cutoff_underflow_exact_path(gmi, ctx, orc):
    # untruncated radius: fp32 weights underflow where f64 ones do not
    rng = np.random.default_rng(4)
    pos = np.stack([rng.uniform(-1, 24, 12), rng.uniform(-1, 20, 12)], 1)
    col = rng.uniform(0, 1, (12, 3))
    check_instance(gmi, ctx, orc, pos, col, 24, 20, 0.5, 60.0)


@pytest.mark.parametrize("ch,n,cluster", [(1, 1200, 0.0), (3, 1200, 0.0), (4, 1200, 0.0),
                                          (3, 6000, 0.5)])
def test_slot_order_gradients_identical(gmi, ctx, orc, monkeypatch, ch, n, cluster):
    # large images route gradients through slot order + one permutation pass
    # (GMI_SLOT_GRADS_MIN_N, default 2^20 points per image); forced on here at
    # a small size, it must give bit-identical gradients to the direct path,
    # fallback routing (nearest) included, and match the oracle; the
    # clustered case has cells above the gather's chunk capacity, whose
    # records K1 re-sorts (the inverse map follows them)
    pos, col, up = orc.synth_batch(21, 2, n, ch, 120, 100, cluster, 8)
    outs = []
    for env in ("1", None):
        if env is None:
            monkeypatch.delenv("GMI_SLOT_GRADS_MIN_N", raising=False)
        else:
            monkeypatch.setenv("GMI_SLOT_GRADS_MIN_N", env)
        img, cache = gmi.forward_batch(pos, col, 120, 100, 1.5, 4.5, ctx=ctx)
        dc, dp = gmi.backward_batch(pos, col, cache, up, 1.5, 4.5, ctx=ctx)
        outs.append((img, dc, dp))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]), "d_colors differ between slot-order and direct paths"
    assert np.array_equal(outs[0][2], outs[1][2]), "d_positions differ between slot-order and direct paths"
    monkeypatch.setenv("GMI_SLOT_GRADS_MIN_N", "1")
    check_instance(gmi, ctx, orc, pos[1], col[1], 120, 100, 1.5, 4.5)


def test_batch_equals_single_calls(gmi, ctx, orc):
    pos, col, up = orc.synth_batch(11, 3, 3000, 3, 100, 90)
    img, cache = gmi.forward_batch(pos, col, 100, 90, 1.0, 3.0, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=ctx)
    for b in range(3):
        i1, c1 = gmi.forward_batch(pos[b:b + 1], col[b:b + 1], 100, 90, 1.0, 3.0, ctx=ctx)
        d1, p1 = gmi.backward_batch(pos[b:b + 1], col[b:b + 1], c1, up[b:b + 1], 1.0, 3.0, ctx=ctx)
        assert np.array_equal(img[b], i1[0])
        assert np.array_equal(dc[b], d1[0]) and np.array_equal(dp[b], p1[0])


@pytest.mark.parametrize("C,sigma", [(3, 1.5), (64, 4.0)])
def test_deterministic_repeat(gmi, ctx, orc, C, sigma):
    pos, col, up = orc.synth_batch(12, 2, 20000, C, 256, 256, cluster_frac=0.05, cluster_px=16)
    r = 3 * sigma
    a = gmi.forward_batch(pos, col, 256, 256, sigma, r, ctx=ctx)
    b = gmi.forward_batch(pos, col, 256, 256, sigma, r, ctx=ctx)
    assert np.array_equal(a[0], b[0])
    ga = gmi.backward_batch(pos, col, a[1], up, sigma, r, ctx=ctx)
    gb = gmi.backward_batch(pos, col, b[1], up, sigma, r, ctx=ctx)
    assert np.array_equal(ga[0], gb[0]) and np.array_equal(ga[1], gb[1])


@pytest.mark.parametrize("ch", [1, 3, 6])
def test_fallback_routing_fixed_point_sums(gmi, ctx, orc, ch):
    # K5: a sparse frame routes hundreds of upstream values of wildly mixed
    # magnitude and sign into each point; the fixed-point sums must match the
    # oracle's f64 sums at the north-star tolerance, be bit-identical across
    # calls, and carry an infinite upstream through as the reference does
    rng = np.random.default_rng(8)
    n, w, h = 12, 90, 70
    pos = f32(np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], 1))
    col = f32(rng.uniform(0, 1, (n, ch)))
    up = rng.uniform(-1, 1, (h, w, ch)) * 10.0 ** rng.integers(-8, 4, (h, w, ch))
    up = f32(up)
    p32, c32 = pos.astype(np.float32)[None], col.astype(np.float32)[None]
    img, cache = gmi.forward_batch(p32, c32, w, h, 1.0, 3.0, ctx=ctx)
    dc1, dp1 = gmi.backward_batch(p32, c32, cache, up.astype(np.float32)[None], 1.0, 3.0, ctx=ctx)
    dc2, dp2 = gmi.backward_batch(p32, c32, cache, up.astype(np.float32)[None], 1.0, 3.0, ctx=ctx)
    assert np.array_equal(dc1, dc2) and np.array_equal(dp1, dp2)
    r = orc.forward(pos, col, w, h, 1.0, 3.0, 0)
    assert r["fallback_flag"].sum() > 0.8 * w * h
    rdc, rdp = orc.backward(pos, col, r, up, 1.0, 3.0, 0)
    # (d_colors only: K5 routes no position gradient, and 1e3-sized upstream
    # values cancelling in the disk sums are outside the fp32 path's envelope)
    assert_close(dc1[0], rdc, what="d_colors")
    # one infinite upstream on a fallback pixel: its point's channel is inf
    fy, fx = np.argwhere(r["fallback_flag"] == 1)[0]
    up_inf = up.copy()
    cinf = ch - 1
    up_inf[fy, fx, cinf] = np.inf
    dci, _ = gmi.backward_batch(p32, c32, cache, up_inf.astype(np.float32)[None], 1.0, 3.0, ctx=ctx)
    k = r["nearest_index"][fy, fx]
    assert np.isposinf(dci[0, k, cinf])
    rest = np.ones_like(dci[0], bool)
    rest[k, cinf] = False
    assert np.array_equal(dci[0][rest], dc1[0][rest])


def test_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


def test_band_split_matches_full_frame(gmi, ctx, orc):
    """configs[3] decomposition on the real kernels (one GPU, bands run in
    sequence, the shared-point reduction done on the host): band images and
    the reduced gradients match the full-frame reference within tolerance
    (the summation order inside a tile follows the band's own cell grid)."""
    from paper_2012_13257_b200 import dist as gdist

    W, H, world, sigma, cutoff = 160, 128, 4, 1.5, 4.5
    pos, col, up = orc.synth_batch(21, 1, 10000, 3, W, H)
    pos, col, up = f32(pos[0]), f32(col[0]), f32(up[0])
    img, cache = gmi.forward_batch(pos[None], col[None], W, H, sigma, cutoff, ctx=ctx)
    assert cache.fallback_count == 0
    r = orc.forward(pos, col, W, H, sigma, cutoff)
    rdc, rdp = orc.backward(pos, col, r, up, sigma, cutoff)
    g_col = np.zeros_like(rdc, dtype=np.float64)
    g_pos = np.zeros_like(rdp, dtype=np.float64)
    for rank in range(world):
        plan = gdist.BandPlan(pos, H, world, rank, cutoff)
        bpos = plan.local_positions(pos)
        bimg, bcache = gmi.forward_batch(bpos[None], col[plan.idx][None], W, plan.rows, sigma,
                                         cutoff, ctx=ctx)
        assert_close(bimg[0], r["image"][plan.r0:plan.r1], what=f"band {rank} image")
        dc, dp = gmi.backward_batch(bpos[None], col[plan.idx][None], bcache,
                                    up[plan.r0:plan.r1][None], sigma, cutoff, ctx=ctx)
        g_col[plan.idx] += dc[0]
        g_pos[plan.idx] += dp[0]
    assert_close(g_col, rdc, what="band d_colors")
    assert_close(g_pos, rdp, what="band d_positions")


def test_band_fallbacks_match_full_frame(gmi, ctx, orc):
    """Row bands at configs[3]'s density (0.25) and r = 3 with fallback
    pixels whose nearest point lies beyond the default halo (the instance of
    tests/test_multirank.py): the certified halo (dist.resolve_band_plan,
    max over the bands) reproduces the full frame's nearest indices bit for
    bit on the real kernels, and the routed gradients."""
    from paper_2012_13257_b200 import dist as gdist
    from test_multirank import _hole_instance

    pos, col, up, W, H, sigma, cutoff = _hole_instance()
    up = f32(up)
    world = 2
    r = orc.forward(pos, col, W, H, sigma, cutoff)
    rdc, rdp = orc.backward(pos, col, r, up, sigma, cutoff)
    want_near = np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)

    def probe(plan):
        _, c = gmi.forward_batch(plan.local_positions(pos)[None], col[plan.idx][None], W,
                                 plan.rows, sigma, cutoff, ctx=ctx)
        _, flag, near = c.pixels()
        fb = np.nonzero(flag[0].ravel())[0]
        return fb, near[0].ravel()[fb]

    halo = max(gdist.resolve_band_plan(pos, W, H, world, k, cutoff, probe).halo
               for k in range(world))
    assert halo > gdist.default_halo(cutoff)
    g_col = np.zeros_like(rdc)
    g_pos = np.zeros_like(rdp)
    for k in range(world):
        plan = gdist.BandPlan(pos, H, world, k, cutoff, halo)
        bpos = plan.local_positions(pos)
        bimg, bc = gmi.forward_batch(bpos[None], col[plan.idx][None], W, plan.rows, sigma, cutoff,
                                     ctx=ctx)
        _, flag, near = bc.pixels()
        got = np.where(flag[0] == 1, plan.idx[np.maximum(near[0], 0)], -1)
        assert np.array_equal(got, want_near[plan.r0:plan.r1]), f"band {k} nearest indices"
        assert_close(bimg[0], r["image"][plan.r0:plan.r1], what=f"band {k} image")
        dc, dp = gmi.backward_batch(bpos[None], col[plan.idx][None], bc,
                                    up[plan.r0:plan.r1][None].astype(np.float32), sigma, cutoff,
                                    ctx=ctx)
        g_col[plan.idx] += dc[0]
        g_pos[plan.idx] += dp[0]
    assert_close(g_col, rdc, what="band d_colors")
    assert_close(g_pos, rdp, what="band d_positions")


@pytest.mark.parametrize("opt", [(True, False), (False, True), (True, True)])
def test_optimize_points_matches_reference(gmi, ctx, opt):
    """optimize_points (optimize.cpp:47-98) on the device against the
    reference's own loop (oracle/_ref): loss curve and final points."""
    import oracle

    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle.Reference()
    rng = np.random.default_rng(11)
    W, H, N, steps, lr = 40, 32, 500, 6, 0.5
    pos = f32(np.stack([rng.uniform(-0.5, W - 0.5, N), rng.uniform(-0.5, H - 0.5, N)], 1))
    col = f32(rng.uniform(0, 1, (N, 3)))
    tgt = f32(rng.uniform(0, 1, (H, W, 3)))
    rp, rc, rl = ref.optimize_points(pos, col, tgt, 1.0, 3.0, steps, lr, *opt)
    out = gmi.optimize_points(gmi.PointSet(pos, col), tgt, 1.0, steps=steps, learning_rate=lr,
                              optimize_positions=opt[0], optimize_colors=opt[1], log_every=4,
                              ctx=ctx)
    assert_close(out["loss_curve"], rl, what="loss curve")
    assert_close(out["points"].positions, rp, what="positions")
    assert_close(out["points"].colors, rc, what="colors")
    steps_logged = sorted({e[0] for e in out["trajectory"]})
    assert steps_logged == [0, 4, 6]


def test_async_host_api_matches_sync(gmi, ctx, orc):
    # GMI_CTX_ASYNC_ERRORS: the host-buffer calls return with their copies
    # queued; after gmi_ctx_synchronize the outputs equal the synchronous ones
    pos, col, up = orc.synth_batch(21, 4, 3000, 3, 100, 90)
    img, cache = gmi.forward_batch(pos, col, 100, 90, 1.0, 3.0, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=ctx)
    actx = gmi.Context(0)
    actx.set_flags(1)
    for _ in range(2):
        img2, cache2 = gmi.forward_batch(pos, col, 100, 90, 1.0, 3.0, ctx=actx)
        dc2, dp2 = gmi.backward_batch(pos, col, cache2, up, 1.0, 3.0, ctx=actx)
        del cache2
        actx.synchronize()
        assert np.array_equal(img, img2)
        assert np.array_equal(dc, dc2) and np.array_equal(dp, dp2)


@pytest.mark.parametrize("factor,ch", [(2, 3), (3, 1), (4, 3), (8, 3)])
def test_gmm_benchmark_matches_reference(gmi, ctx, orc, factor, ch):
    # the GMM row of run_benchmark on the device vs the restatement (pinned
    # to the reference in test_oracle.py) and, when built, the reference
    import oracle
    rng = np.random.default_rng(factor)
    yy, xx = np.mgrid[0:67, 0:75]
    base = 0.5 + 0.4 * np.sin(xx / 7.0)[:, :, None] * np.cos(yy / 5.0)[:, :, None]
    img = np.clip(base + 0.05 * rng.standard_normal((67, 75, ch)), 0, 1).astype(np.float32)
    row = gmi.gmm_benchmark(img, factor, ctx=ctx)
    l1, best = oracle.gmm_benchmark(orc, img.astype(np.float64), factor)
    assert row["sigmas"][best] == row["sigma_used"]
    np.testing.assert_allclose(row["l1_per_sigma"], l1, rtol=1e-5, atol=1e-7)
    if oracle.reference_available():
        rl1, rsig, _ = oracle.Reference().run_benchmark_gmm(img.astype(np.float64), factor)
        assert rsig == row["sigma_used"]
        assert abs(rl1 - row["l1"]) <= 1e-7 + 1e-5 * rl1
    # a caller-supplied low-resolution raster and a fixed sigma
    low = oracle.block_mean_downsample(img.astype(np.float64), factor).astype(np.float32)
    row2 = gmi.gmm_benchmark(img, factor, sigma=0.45 * factor, lowres=low, ctx=ctx)
    l1b, _ = oracle.gmm_benchmark(orc, img.astype(np.float64), factor, sigmas=[0.45 * factor],
                                  lowres=low.astype(np.float64))
    np.testing.assert_allclose(row2["l1"], l1b[0], rtol=1e-5, atol=1e-7)


def test_gmm_benchmark_invalid_factor(gmi, ctx):
    with pytest.raises(gmi.GmiError) as e:
        gmi.gmm_benchmark(np.zeros((8, 8, 1), np.float32), 0, ctx=ctx)
    assert e.value.code == 9


def test_async_host_api_defers_validation_errors(gmi, orc):
    # GMI_CTX_ASYNC_ERRORS: a host-buffer forward returns at once and the
    # reference's NonFiniteValue surfaces at gmi_ctx_synchronize
    pos, col, _ = orc.synth_batch(23, 2, 500, 3, 40, 30)
    pos[1, 77, 0] = np.nan
    actx = gmi.Context(0)
    actx.set_flags(1)
    _, cache = gmi.forward_batch(pos, col, 40, 30, 1.0, 3.0, ctx=actx)
    with pytest.raises(gmi.GmiError) as e:
        actx.synchronize()
    assert e.value.code == 1 and "77" in str(e.value)
    del cache
