"""Element-wise parity at the BASELINE.json configs' own sizes (not shapes
shrunk to fit the oracle): the device path against the CPU oracle at the
north-star tolerance |a-b| <= 1e-6 + 1e-5 max(|a|,|b|), and bit-exact
binning / fallback sets / nearest indices / contribution counts.

  configs[1]  B=16 x 512^2, N=65,536, sigma 1: image 0 and 15 of one batched
              call, full frame.
  configs[2]  B=64 x 1024^2, N=262,144, sigma 1.5 (the headline): images 0
              and 63 of ONE B=64 call, full frame.
  configs[3]  1 x 8192^2, N=16.8M, sigma 1: the full-frame device call,
              checked on windows (interior, a row-band edge of the 8-GPU
              split, both frame corners — one of them the reference grid's
              2048-cap corner) against the windowed oracle: points in the
              window +- margin shifted by an integer offset, which SURVEY
              §0.7 / A.5 showed reproduces the full-frame reference bit for
              bit (translation equivariance, test_engine.cpp:158-187).
  configs[4]  1 x 2048^2, N=1M with 5% in a 32 px cluster, C = 64, sigma 4:
              a window around the cluster against the reference itself over
              channel groups (C in {1,3} only, core.cpp:60-64).
Plus the reference's bin grid (bin_grid.cpp:38-82, 2048 cap) on the full
configs[2] and configs[3] point sets, including configs[3]'s capped corner
cell of ~1M points.
"""
import os

import numpy as np
import pytest

from conftest import assert_close

pytestmark = pytest.mark.gpu


def _check_full(gmi, orc, pos, col, up, img, dc, dp, flag, near, W, H, sigma, cutoff, what):
    p64, c64, u64 = (a.astype(np.float64) for a in (pos, col, up))
    r = orc.forward(p64, c64, W, H, sigma, cutoff)
    rdc, rdp = orc.backward(p64, c64, r, u64, sigma, cutoff)
    assert np.array_equal(flag, r["fallback_flag"]), f"{what}: fallback set"
    assert np.array_equal(near, np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)), \
        f"{what}: nearest indices"
    assert_close(img, r["image"], what=f"{what} image")
    assert_close(dc, rdc, what=f"{what} d_colors")
    assert_close(dp, rdp, what=f"{what} d_positions")
    return r


@pytest.mark.parametrize("cfg", [
    dict(name="configs[1]", B=16, N=65536, W=512, H=512, sigma=1.0, seed=201, check=(0, 15)),
    dict(name="configs[2]", B=64, N=262144, W=1024, H=1024, sigma=1.5, seed=301, check=(0, 63)),
], ids=["configs1", "configs2"])
def test_batched_config_full_frame(gmi, ctx, orc, cfg):
    B, N, W, H, sigma = cfg["B"], cfg["N"], cfg["W"], cfg["H"], cfg["sigma"]
    cutoff = 3.0 * sigma
    pos, col, up = orc.synth_batch(cfg["seed"], B, N, 3, W, H)
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, ctx=ctx)
    _, flag, near = cache.pixels()
    for b in cfg["check"]:
        r = _check_full(gmi, orc, pos[b], col[b], up[b], img[b], dc[b], dp[b], flag[b], near[b],
                        W, H, sigma, cutoff, f"{cfg['name']} image {b}")
        if b == cfg["check"][0]:
            # per-pixel contribution counts (pixel_start deltas) of the same
            # image through the counting instantiation of the gather
            _, c1 = gmi.forward_batch(pos[b:b + 1], col[b:b + 1], W, H, sigma, cutoff, ctx=ctx)
            assert np.array_equal(gmi.forward_counts(c1)[0], r["counts"]), "contribution counts"


def _window(pos, x0, y0, w, h, margin):
    """Points within the window grown by `margin`, ascending original index,
    shifted by the integer offset (exact in fp32)."""
    keep = ((pos[:, 0] >= x0 - margin) & (pos[:, 0] <= x0 + w - 1 + margin) &
            (pos[:, 1] >= y0 - margin) & (pos[:, 1] <= y0 + h - 1 + margin))
    idx = np.nonzero(keep)[0]
    p = pos[idx].copy()
    p[:, 0] -= np.float32(x0)
    p[:, 1] -= np.float32(y0)
    return idx, p


def _windowed_checks(orc, pos, col, up, img, dc, dp, flag, near, windows, sigma, cutoff, margin,
                     fallback_routed, ref_any_c=None):
    """Image / fallback / nearest of each window bit-for-bit against the
    windowed oracle (tolerance for the image), gradients of the points whose
    disks lie inside the window and that receive no fallback upstream from
    outside it."""
    H_full, W_full = flag.shape
    for (x0, y0, w, h) in windows:
        idx, wp = _window(pos, x0, y0, w, h, margin)
        wc = col[idx].astype(np.float64)
        wu = up[y0:y0 + h, x0:x0 + w].astype(np.float64)
        if ref_any_c is not None:
            r, rdc, rdp = ref_any_c(wp.astype(np.float64), wc, w, h, sigma, cutoff, wu)
        else:
            r = orc.forward(wp.astype(np.float64), wc, w, h, sigma, cutoff)
            rdc, rdp = orc.backward(wp.astype(np.float64), wc, r, wu, sigma, cutoff)
        what = f"window ({x0},{y0}) {w}x{h}"
        # the windowed reference is the full-frame one only if every fallback
        # pixel's nearest point is closer than the margin
        fb = np.nonzero(r["fallback_flag"].ravel())[0]
        if fb.size:
            q = np.stack([fb % w, fb // w], 1).astype(np.float64)
            d = np.sqrt(((q - wp[r["nearest_index"].ravel()[fb]].astype(np.float64)) ** 2).sum(1))
            assert d.max() < margin - 1, f"{what}: margin does not certify the fallbacks"
        assert np.array_equal(flag[y0:y0 + h, x0:x0 + w], r["fallback_flag"]), f"{what}: fallback set"
        wnear = np.where(r["fallback_flag"] == 1, idx[np.maximum(r["nearest_index"], 0)], -1)
        assert np.array_equal(near[y0:y0 + h, x0:x0 + w], wnear), f"{what}: nearest indices"
        assert_close(img[y0:y0 + h, x0:x0 + w], r["image"], what=f"{what} image")
        # points whose closed disks are inside the window: complete gradients
        inside = ((wp[:, 0] - cutoff >= 0) & (wp[:, 0] + cutoff <= w - 1) &
                  (wp[:, 1] - cutoff >= 0) & (wp[:, 1] + cutoff <= h - 1))
        inside &= ~fallback_routed[idx]
        assert inside.sum() > 0
        assert_close(dc[idx[inside]], rdc[inside], what=f"{what} d_colors")
        assert_close(dp[idx[inside]], rdp[inside], what=f"{what} d_positions")


def _routed_from(flag, near, windows, n):
    """Points that receive fallback upstream from pixels outside any window
    (their windowed gradient is incomplete by construction)."""
    outside = flag.astype(bool).copy()
    for (x0, y0, w, h) in windows:
        outside[y0:y0 + h, x0:x0 + w] = False
    routed = np.zeros(n, bool)
    routed[near[outside & (near >= 0)]] = True
    return routed


def test_configs3_single_huge_image_windows(gmi, ctx, orc):
    W = H = 8192
    N, sigma, cutoff = 16777216, 1.0, 3.0
    pos, col, up = orc.synth_batch(401, 1, N, 3, W, H)
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, ctx=ctx)
    _, flag, near = cache.pixels()
    assert cache.fallback_count > 10000  # ~57k at density 0.25, r = 3
    windows = [(4000, 4000, 256, 192),       # interior
               (2000, 1024 - 96, 256, 192),  # across the rank-0 / rank-1 band edge (8 GPUs)
               (0, 0, 192, 160),             # top-left corner (points below -0.5 excluded)
               (W - 224, H - 176, 224, 176)]  # bottom-right: the reference grid's capped corner
    routed = _routed_from(flag[0], near[0], windows, N)
    _windowed_checks(orc, pos[0], col[0], up[0], img[0], dc[0], dp[0], flag[0], near[0], windows,
                     sigma, cutoff, margin=cutoff + 12, fallback_routed=routed)


def test_configs4_cluster_window_channel_groups(gmi, ctx, orc, ref):
    W = H = 2048
    N, C, sigma, cutoff = 1048576, 64, 4.0, 12.0
    pos, col, up = orc.synth_batch(501, 1, N, C, W, H, cluster_frac=0.05, cluster_px=32)
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, ctx=ctx)
    _, flag, near = cache.pixels()
    nc = int(0.05 * N)
    cx0, cy0 = np.floor(pos[0, :nc].min(0)).astype(int)
    # a window over the cluster's corner: clustered and plain pixels, the
    # heaviest pixels of the config (~23k contributors each)
    windows = [(max(0, cx0 - 24), max(0, cy0 - 24), 48, 40)]
    routed = _routed_from(flag[0], near[0], windows, N)
    workers = os.cpu_count() or 1

    def any_c(p, c, w, h, s, r, u):
        meta, rdc, rdp = ref.forward_backward_any_c(p, c, w, h, s, r, u, 0, workers)
        return meta, rdc, rdp

    _windowed_checks(orc, pos[0], col[0], up[0], img[0], dc[0], dp[0], flag[0], near[0], windows,
                     sigma, cutoff, margin=cutoff + 8, fallback_routed=routed, ref_any_c=any_c)


@pytest.mark.parametrize("which", ["configs2", "configs3"])
def test_bin_grid_full_size(gmi, ctx, orc, which):
    # build_bin_grid (bin_grid.cpp:38-82) with the 2048-cells cap on the full
    # point sets; configs[3]'s grid is capped (2048 x 2048, clamped edge cells)
    if which == "configs2":
        pos, _, _ = orc.synth_batch(302, 1, 262144, 1, 1024, 1024, upstream=False)
        cell = 4.5
    else:
        pos, _, _ = orc.synth_batch(402, 1, 16777216, 1, 8192, 8192, upstream=False)
        cell = 3.0
    got = gmi.bin_grid(pos[0], cell, ctx=ctx)
    want = orc.bin_grid(pos[0].astype(np.float64), cell)
    assert np.array_equal(got["origin"], want["origin"])
    assert (got["n_cols"], got["n_rows"]) == (want["n_cols"], want["n_rows"])
    if which == "configs3":
        assert want["n_cols"] == 2048 and want["n_rows"] == 2048
        assert int(np.diff(want["bin_start"]).max()) > 1_000_000  # the capped corner cell
    assert np.array_equal(got["bin_start"], want["bin_start"])
    assert np.array_equal(got["point_index"], want["point_index"])
