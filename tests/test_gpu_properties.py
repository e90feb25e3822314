"""Property tests of the device path, restating the reference's engine
invariants (proj/tests/test_engine.cpp) and adding size-independent checks at
the BASELINE frame size, where the oracle would take minutes.

Reference pins restated (the reference asserts them in f64 at 1e-12; the
device computes in fp32, so the north-star tolerance |a-b| <= 1e-6 + 1e-5
max(|a|,|b|) applies unless the arithmetic is exact):
  - shared weights across channels          test_engine.cpp:72-88
  - convex-combination bound                test_engine.cpp:122-139
  - constant colours reconstruct            test_engine.cpp:141-156
  - translation equivariance (bit-exact)    test_engine.cpp:158-187
  - sigma-scaling consistency               test_engine.cpp:189-215
  - constant colours -> d_pos = 0           test_engine.cpp:313-330
At the BASELINE sizes (configs[2] through the host API; configs[3], one
8192^2 image with 16.7M points, and one configs[4] image, C = 64 with a 5%
cluster, through the zero-copy device path):
  - partition of unity of the backward: sum_i d_col[i] = sum_p upstream[p]
    (every pixel's ratios sum to 1; fallback pixels route to their nearest
    point under NearestPoint, engine.cpp:200-211), per image and channel;
  - the image is a convex combination of colours in [0, 1].
"""
import numpy as np
import pytest

from conftest import ABS_TOL, REL_TOL, assert_close

pytestmark = pytest.mark.gpu


def random_points(rng, n, c, extent):
    """gmi_test::random_points (test_support.hpp): positions U[-1, extent)."""
    pos = rng.uniform(-1.0, extent, size=(1, n, 2)).astype(np.float32)
    col = rng.uniform(0.0, 1.0, size=(1, n, c)).astype(np.float32)
    return pos, col


def test_shared_weights_flat_channel(gmi, ctx):
    rng = np.random.default_rng(5)
    pos, col = random_points(rng, 12, 3, 8.0)
    col[..., 1] = 0.25
    img, _ = gmi.forward_batch(pos, col, 8, 8, 1.5, ctx=ctx)
    assert_close(img[..., 1], np.full_like(img[..., 1], 0.25), what="flat channel")


def test_convex_bound(gmi, ctx):
    rng = np.random.default_rng(7)
    pos, col = random_points(rng, 30, 1, 10.0)
    img, cache = gmi.forward_batch(pos, col, 10, 10, 0.8, ctx=ctx)
    _, flag, _ = cache.pixels()
    ok = flag[0] == 0
    lo, hi = float(col.min()), float(col.max())
    v = img[0, ..., 0][ok].astype(np.float64)
    assert (v >= lo - ABS_TOL - REL_TOL * lo).all() and (v <= hi + ABS_TOL + REL_TOL * hi).all()


@pytest.mark.parametrize("sigma", [0.5, 1.0, 3.0])
def test_constant_colours_reconstruct(gmi, ctx, sigma):
    rng = np.random.default_rng(8)
    pos, col = random_points(rng, 20, 1, 10.0)
    col[:] = 0.37
    img, _ = gmi.forward_batch(pos, col, 10, 10, sigma, ctx=ctx)
    assert_close(img, np.full_like(img, np.float32(0.37)), what=f"constant sigma={sigma}")


@pytest.mark.parametrize("cutoff", [100.0, 3.0])
def test_translation_equivariance_dyadic(gmi, ctx, cutoff):
    """Dyadic positions + integer shifts are exact in fp32 too, so every
    weight is bit-identical.  With the reference's 100-sigma cutoff (the
    precise path, ascending-index sums) the shifted render is bit-identical;
    with 3 sigma the tiles of the fast gather move against the points, so
    the summation order may change: tolerance."""
    rng = np.random.default_rng(9)
    pos = (rng.integers(0, 97, size=(1, 15, 2)) / 8.0).astype(np.float32)
    col = rng.uniform(0.0, 1.0, size=(1, 15, 1)).astype(np.float32)
    dx, dy = 3, 2
    moved = pos + np.array([dx, dy], np.float32)
    base, _ = gmi.forward_batch(pos, col, 12, 12, 1.0, cutoff, ctx=ctx)
    shifted, _ = gmi.forward_batch(moved, col, 12 + dx, 12 + dy, 1.0, cutoff, ctx=ctx)
    win = shifted[0, dy:dy + 12, dx:dx + 12]
    if cutoff == 100.0:
        assert np.array_equal(base[0], win)
    else:
        assert_close(win, base[0], what="shifted window")


def test_sigma_scaling(gmi, ctx):
    rng = np.random.default_rng(10)
    pos = rng.integers(0, 6, size=(1, 10, 2)).astype(np.float32)
    col = rng.uniform(0.0, 1.0, size=(1, 10, 1)).astype(np.float32)
    s = 2.0
    base, _ = gmi.forward_batch(pos, col, 6, 6, 0.9, 1000.0, ctx=ctx)
    big, _ = gmi.forward_batch(pos * s, col, 11, 11, 0.9 * s, 1000.0, ctx=ctx)
    # nk = -log2(e) / (2 sigma^2) rounds differently for the two sigmas: the
    # exponents (|e| <= ~100) agree to a few fp32 ulps, weights to ~1e-5 rel
    assert_close(big[0, ::2, ::2], base[0], rel=5e-5, abs_=1e-6, what="sigma scaling")


def test_constant_colours_zero_position_gradient(gmi, ctx):
    rng = np.random.default_rng(11)
    pos, col = random_points(rng, 40, 3, 16.0)
    col[:] = np.array([0.2, 0.5, 0.9], np.float32)
    sigma = 1.2
    r = 3 * sigma
    img, cache = gmi.forward_batch(pos, col, 16, 16, sigma, ctx=ctx)
    up = np.ones_like(img)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, ctx=ctx)
    # exact zero in f64; in fp32 out_p = c (1 + O(1e-7)), so
    # |d_pos_i| <= r / sigma^2 * sum_c c_c d_col_ic * O(1e-7)
    scale = (r / sigma ** 2) * (dc[0] * col[0]).sum(axis=1, keepdims=True)
    assert (np.abs(dp[0]) <= ABS_TOL + REL_TOL * scale).all(), np.abs(dp[0]).max()


def test_backward_partition_of_unity_at_scale(gmi, ctx):
    """configs[2] frame and density (2 images): sum_i d_col = sum_p upstream."""
    rng = np.random.default_rng(2026)
    B, N, C, W, H, sigma = 2, 262144, 3, 1024, 1024, 1.5
    pos = np.empty((B, N, 2), np.float32)
    pos[..., 0] = rng.uniform(-0.5, W - 0.5, size=(B, N))
    pos[..., 1] = rng.uniform(-0.5, H - 0.5, size=(B, N))
    col = rng.uniform(0.0, 1.0, size=(B, N, C)).astype(np.float32)
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, ctx=ctx)
    up = rng.uniform(-1.0, 1.0, size=img.shape).astype(np.float32)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, ctx=ctx)
    assert np.isfinite(dc).all() and np.isfinite(dp).all()
    got = dc.astype(np.float64).sum(axis=1)                     # [B, C]
    want = up.astype(np.float64).sum(axis=(1, 2))               # [B, C]
    # each d_col entry carries ~1e-6 relative fp32 error
    bound = ABS_TOL + REL_TOL * np.abs(dc.astype(np.float64)).sum(axis=1)
    assert (np.abs(got - want) <= bound).all(), (got, want, bound)
    # and the image is a convex combination wherever W > 0
    _, flag, _ = cache.pixels()
    v = img[flag == 0]
    assert v.min() >= -ABS_TOL and v.max() <= 1.0 + ABS_TOL + REL_TOL


def _device_scale_case(gmi, ctx, B, N, C, W, H, sigma, cluster, seed):
    """Forward + backward at a full BASELINE size through the zero-copy
    device path (inputs generated on the device with torch, as bench.py
    does), checked by partition of unity and the convex bound."""
    torch = pytest.importorskip("torch")
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pos = torch.empty(B, N, 2, device="cuda")
    pos[..., 0].uniform_(-0.5, W - 0.5, generator=g)
    pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
    nc = int(cluster * N)
    if nc:
        corner = torch.rand(B, 1, 2, device="cuda", generator=g) * torch.tensor([W - 32.0, H - 32.0],
                                                                                device="cuda")
        pos[:, :nc] = corner + torch.rand(B, nc, 2, device="cuda", generator=g) * 32.0
    col = torch.rand(B, N, C, device="cuda", generator=g)
    img = torch.empty(B, H, W, C, device="cuda")
    torch.cuda.synchronize()
    _, cache = gmi.forward_cuda(pos, col, W, H, sigma, image=img, ctx=ctx)
    torch.cuda.synchronize()
    up = torch.empty_like(img).uniform_(-1.0, 1.0, generator=g)
    dc = torch.empty(B, N, C, device="cuda")
    dp = torch.empty(B, N, 2, device="cuda")
    torch.cuda.synchronize()
    gmi.backward_cuda(pos, col, cache, up, sigma, d_colors=dc, d_positions=dp, ctx=ctx)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(img).all()) and bool(torch.isfinite(dc).all())
    assert bool(torch.isfinite(dp).all())
    got = dc.double().sum(dim=1)
    want = up.double().sum(dim=(1, 2))
    bound = ABS_TOL + REL_TOL * dc.double().abs().sum(dim=1)
    assert bool(((got - want).abs() <= bound).all()), (got - want).abs().max().item()
    assert float(img.min()) >= -ABS_TOL and float(img.max()) <= 1.0 + ABS_TOL + REL_TOL


def test_partition_of_unity_configs3_single_huge_image(gmi, ctx):
    """configs[3]: one 8192^2 image, N = 16,777,216, sigma = 1 (one GPU)."""
    _device_scale_case(gmi, ctx, 1, 16777216, 3, 8192, 8192, 1.0, 0.0, 33)


def test_partition_of_unity_configs4_wide_clustered(gmi, ctx):
    """configs[4] per image: 2048^2, N = 1,048,576 with 5% in one 32^2
    square, C = 64 (wide kernels), sigma = 4."""
    _device_scale_case(gmi, ctx, 1, 1048576, 64, 2048, 2048, 4.0, 0.05, 44)


def test_backward_linear_in_upstream_configs2_full_batch(gmi, ctx):
    """configs[2] at its full size (B = 64 x 1024^2, N = 262,144, sigma =
    1.5): the backward is linear in the upstream image, so
    bwd(2 u1 + u2) = 2 bwd(u1) + bwd(u2) to fp32 rounding, and a zero
    upstream gives exactly zero gradients."""
    torch = pytest.importorskip("torch")
    B, N, C, W, H, sigma = 64, 262144, 3, 1024, 1024, 1.5
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    pos = torch.empty(B, N, 2, device="cuda")
    pos[..., 0].uniform_(-0.5, W - 0.5, generator=g)
    pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
    col = torch.rand(B, N, C, device="cuda", generator=g)
    img = torch.empty(B, H, W, C, device="cuda")
    torch.cuda.synchronize()
    _, cache = gmi.forward_cuda(pos, col, W, H, sigma, image=img, ctx=ctx)
    torch.cuda.synchronize()
    u1 = torch.empty_like(img).uniform_(-1.0, 1.0, generator=g)
    u2 = torch.empty_like(img).uniform_(-1.0, 1.0, generator=g)
    u3 = 2.0 * u1 + u2
    torch.cuda.synchronize()

    def bwd(u):
        # the library runs on its context's stream, torch on its own: every
        # hand-over between them is a device synchronisation (including the
        # f64 copies below, whose float sources go back to torch's allocator)
        dc = torch.empty(B, N, C, device="cuda")
        dp = torch.empty(B, N, 2, device="cuda")
        torch.cuda.synchronize()
        gmi.backward_cuda(pos, col, cache, u, sigma, d_colors=dc, d_positions=dp, ctx=ctx)
        torch.cuda.synchronize()
        out = dc.double(), dp.double()
        torch.cuda.synchronize()
        return out

    c1, p1 = bwd(u1)
    c2, p2 = bwd(u2)
    c3, p3 = bwd(u3)
    for got, want, mag, what in ((c3, 2 * c1 + c2, 2 * c1.abs() + c2.abs(), "d_colors"),
                                 (p3, 2 * p1 + p2, 2 * p1.abs() + p2.abs(), "d_positions")):
        # north-star form on the magnitudes of the combined results, plus a
        # floor of 1e-9 x the largest magnitude: an entry whose terms cancel
        # (d_positions under a random-sign upstream) keeps the fp32 rounding
        # of its terms, not of its small total
        bound = ABS_TOL + REL_TOL * mag + 1e-4 * REL_TOL * float(mag.max())
        bad = (got - want).abs() > bound
        assert not bool(bad.any()), f"{what}: {int(bad.sum())} entries off"
    zc, zp = bwd(torch.zeros_like(u1))
    assert bool((zc == 0).all()) and bool((zp == 0).all())
