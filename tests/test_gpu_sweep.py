"""GPU parity sweep over the shapes the fast paths branch on: radius (row-pair
bins, lanes per point), channel count (one group, channel groups), density
(single / multi chunk tiles, clustered cells), fallback mode, batch (composite
host-API caches), frames that are not multiples of the 64x16 tile and points
outside the frame.  Every case: bit-exact fallback set and nearest indices,
image / d_colors / d_positions within the north-star tolerance."""
import numpy as np
import pytest

from conftest import assert_close

pytestmark = pytest.mark.gpu

CASES = [
    # (seed, B, N, C, W, H, sigma, cutoff, fallback, cluster, outside)
    (1, 1, 3000, 3, 97, 61, 1.0, 3.0, 0, 0.0, 0.0),
    (2, 2, 5000, 1, 130, 70, 1.5, 4.5, 1, 0.0, 0.0),
    (3, 1, 4000, 2, 64, 48, 2.0, 6.0, 0, 0.0, 0.1),
    (4, 3, 2500, 4, 80, 80, 0.8, 2.4, 0, 0.0, 0.0),
    (5, 1, 6000, 3, 128, 96, 1.0, 3.0, 0, 0.2, 0.0),
    (6, 1, 3000, 6, 72, 64, 1.25, 3.75, 0, 0.0, 0.0),
    (7, 1, 2000, 8, 96, 64, 3.0, 9.0, 0, 0.05, 0.0),
    (8, 2, 8000, 3, 160, 40, 1.5, 4.0, 1, 0.0, 0.05),
    (9, 1, 20000, 3, 64, 64, 1.0, 3.0, 0, 0.5, 0.0),
    (10, 1, 1500, 5, 50, 90, 4.0, 12.0, 0, 0.0, 0.0),
    # wide-channel path (C > 4): pass widths 16 / 32 / 64, ragged C, dense
    # clusters (multi-chunk tiles), points outside the frame
    (11, 2, 3000, 64, 96, 80, 4.0, 12.0, 0, 0.05, 0.0),
    (12, 1, 4000, 33, 70, 50, 1.5, 4.5, 1, 0.3, 0.05),
    (13, 1, 2500, 16, 64, 64, 2.0, 6.0, 0, 0.0, 0.1),
    (14, 1, 6000, 20, 80, 64, 1.0, 3.0, 0, 0.6, 0.0),
    (15, 1, 1200, 130, 48, 40, 1.0, 3.0, 0, 0.0, 0.0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"s{c[0]}")
def test_sweep(gmi, ctx, orc, case):
    seed, B, N, C, W, H, sigma, cutoff, fb, cluster, outside = case
    pos, col, _ = orc.synth_batch(seed, B, N, C, W, H, cluster_frac=cluster, cluster_px=16)
    rng = np.random.default_rng(seed)
    if outside:
        # a share of the points well outside the frame (clamped / far cells)
        k = int(outside * N)
        pos[:, :k] = rng.uniform(-3 * W, 4 * W, (B, k, 2)).astype(np.float32)
    up = rng.uniform(-1, 1, (B, H, W, C)).astype(np.float32)
    fbs = "nearest" if fb == 0 else "zero"
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, fbs, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, fbs, ctx=ctx)
    _, flag, near = cache.pixels()
    for b in range(B):
        p64, c64, u64 = pos[b].astype(np.float64), col[b].astype(np.float64), up[b].astype(np.float64)
        r = orc.forward(p64, c64, W, H, sigma, cutoff, fb)
        rdc, rdp = orc.backward(p64, c64, r, u64, sigma, cutoff, fb)
        assert np.array_equal(flag[b], r["fallback_flag"]), f"image {b}: fallback set differs"
        if fb == 0:
            want = np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)
            assert np.array_equal(near[b], want), f"image {b}: nearest differs"
        assert_close(img[b], r["image"], what=f"image {b}")
        assert_close(dc[b], rdc, what=f"d_colors {b}")
        assert_close(dp[b], rdp, what=f"d_positions {b}")


def test_single_cell_above_chunk_capacity(gmi, ctx, orc):
    # thousands of points inside one reference cell: the gather splits that
    # cell across TMA chunks (K1 index-orders it), results stay exact and
    # bit-deterministic
    pos, col, _ = orc.synth_batch(31, 1, 6000, 3, 48, 40, cluster_frac=0.7, cluster_px=2)
    rng = np.random.default_rng(31)
    up = rng.uniform(-1, 1, (1, 40, 48, 3)).astype(np.float32)
    img, cache = gmi.forward_batch(pos, col, 48, 40, 1.0, 3.0, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=ctx)
    img2, _ = gmi.forward_batch(pos, col, 48, 40, 1.0, 3.0, ctx=ctx)
    assert np.array_equal(img, img2)
    p64, c64, u64 = pos[0].astype(np.float64), col[0].astype(np.float64), up[0].astype(np.float64)
    r = orc.forward(p64, c64, 48, 40, 1.0, 3.0)
    rdc, rdp = orc.backward(p64, c64, r, u64, 1.0, 3.0)
    assert_close(img[0], r["image"], what="image")
    assert_close(dc[0], rdc, what="d_colors")
    assert_close(dp[0], rdp, what="d_positions")
