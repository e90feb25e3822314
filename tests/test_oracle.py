"""CPU: pins the oracle (oracle/gmi_oracle.c, a restatement of the reference)
against the reference's own known-answer tests and against fixtures produced
by the reference itself (tests/golden/reference_fixtures.npz, made by
tests/golden/gen_golden.py), plus a live comparison with the compiled
reference (oracle/_ref) when it is available in this container."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "reference_fixtures.npz")


@pytest.fixture(scope="module")
def fx():
    return np.load(FIX)


def cases(fx):
    return [str(n) for n in fx["names"]]


# ------------------------------------------------------------------- KATs --
def test_gaussian_weight_kats(orc):
    # test_core.cpp:11-17
    assert orc.gaussian_weight(0, 0, 0, 0, 1.0) == 1.0
    assert orc.gaussian_weight(1, 0, 0, 0, 1.0) == pytest.approx(0.6065306597126334, rel=1e-14)
    assert orc.gaussian_weight(0.5, 0.5, 2, 0, 1.0) == pytest.approx(0.2865047968601901, rel=1e-14)


def test_gaussian_weight_symmetry_translation(orc):
    # test_core.cpp:20-61: exact symmetry and exact translation invariance on
    # dyadic coordinates with integer shifts
    rng = np.random.default_rng(11)
    for _ in range(100):
        q, mu = rng.uniform(-50, 50, 2), rng.uniform(-50, 50, 2)
        s = rng.uniform(0.1, 5.0)
        w = orc.gaussian_weight(q[0], q[1], mu[0], mu[1], s)
        assert w == orc.gaussian_weight(mu[0], mu[1], q[0], q[1], s)
        assert 0.0 <= w <= 1.0
        dq = rng.integers(-2048, 2049, 2) / 16.0
        dm = rng.integers(-2048, 2049, 2) / 16.0
        t = rng.integers(-1000, 1001, 2).astype(float)
        assert orc.gaussian_weight(*dq, *dm, s) == orc.gaussian_weight(*(dq + t), *(dm + t), s)


def test_three_point_mixture(orc):
    # test_engine.cpp:53-70 / test_oracle.cpp:22-30
    f = orc.forward([[-0.5, -0.5], [1.5, -0.5], [-0.5, 1.5]], [[1.0], [0.0], [0.0]], 1, 1, 1.0, 10.0)
    assert f["image"][0, 0, 0] == pytest.approx(0.5761168847658291, rel=1e-12)


def test_single_point_and_equidistant(orc):
    # test_engine.cpp:26-51
    f = orc.forward([[3.7, -2.1]], [[0.7]], 5, 4, 1.0, 3.0)
    assert np.all(f["image"] == 0.7)
    f = orc.forward([[0, 1], [2, 1]], [[0.2], [0.8]], 3, 3, 1.0, 3.0)
    assert f["image"][1, 1, 0] == pytest.approx(0.5, rel=1e-14)


def test_fallback_policies_and_routing(orc):
    # test_engine.cpp:217-249, 347-370
    pos, col = [[100, 100], [200, 200]], [[0.9], [0.1]]
    f = orc.forward(pos, col, 4, 4, 1.0, 2.0, 0)
    assert f["fallback_count"] == 16 and np.all(f["image"] == 0.9)
    f = orc.forward(pos, col, 4, 4, 1.0, 2.0, 1)
    assert f["fallback_count"] == 16 and np.all(f["image"] == 0.0)
    f = orc.forward([[1000.0, 0.0]], [[0.6]], 1, 1, 0.5, 10000.0)
    assert f["fallback_count"] == 1 and f["image"][0, 0, 0] == 0.6
    pos, col = [[-50, 0], [-60, 0]], [[0.3], [0.7]]
    f = orc.forward(pos, col, 2, 2, 1.0, 3.0)
    dc, dp = orc.backward(pos, col, f, np.ones((2, 2, 1)), 1.0, 3.0)
    assert dc[0, 0] == 4.0 and dc[1, 0] == 0.0 and np.all(dp == 0.0)


def test_backward_single_point_and_constant_colours(orc):
    # test_engine.cpp:302-330
    f = orc.forward([[2, 2]], [[0.5]], 6, 5, 1.0, 100.0)
    dc, dp = orc.backward([[2, 2]], [[0.5]], f, np.ones((5, 6, 1)), 1.0, 100.0)
    assert dc[0, 0] == pytest.approx(30.0, rel=1e-12) and np.all(dp == 0.0)
    rng = np.random.default_rng(32)
    pos = rng.uniform(-1, 8, (15, 2))
    col = np.full((15, 3), 0.42)
    f = orc.forward(pos, col, 8, 8, 1.2, 3.6)
    dc, dp = orc.backward(pos, col, f, rng.uniform(-1, 1, (8, 8, 3)), 1.2, 3.6)
    # the reference asserts exact zeros on its instance; in general f64 num/W
    # reproduces the constant to within an ulp, so the sum is ~1e-16
    assert np.all(np.abs(dp) < 1e-14)


def test_validation_codes(orc):
    # core.cpp:55-96: first violated invariant by point index
    assert orc.validate(np.zeros((0, 2)), np.zeros((0, 1)))[0] == 3  # EmptyPointSet
    rc, idx = orc.validate([[0, 0], [np.nan, 0]], [[0.5], [0.5]])
    assert (rc, idx) == (1, 1)  # NonFiniteValue
    rc, idx = orc.validate([[0, 0], [1, 1]], [[0.5], [1.5]])
    assert (rc, idx) == (2, 1)  # ColorOutOfRange


def test_rng_matches_reference_stream(orc, fx):
    # rng.hpp:12-59 (pinned for reproducible inputs)
    assert np.array_equal(orc.rng_u64(42, 16), fx["rng/seed42"])


def test_kat_fixture_values(orc, fx):
    g = fx["kat/gaussian_weight"]
    assert orc.gaussian_weight(1, 0, 0, 0, 1.0) == g[0]
    assert orc.gaussian_weight(0.5, 0.5, 2, 0, 1.0) == g[1]


# ---------------------------------------------- restatement vs reference --
def test_oracle_matches_reference_fixtures(orc, fx):
    """Bit-exact: bins, neighbour counts, fallback set / nearest indices;
    f64 outputs to 1e-12 (the restatement follows the reference statement by
    statement; only glibc exp could differ across machines)."""
    for name in cases(fx):
        w, h, sigma, cutoff, fb = fx[f"{name}/params"]
        w, h, fb = int(w), int(h), int(fb)
        pos, col, up = fx[f"{name}/pos"], fx[f"{name}/col"], fx[f"{name}/upstream"]
        f = orc.forward(pos, col, w, h, sigma, cutoff, fb)
        dc, dp = orc.backward(pos, col, f, up, sigma, cutoff, fb)
        for k in ("fallback_flag", "nearest_index", "counts"):
            assert np.array_equal(f[k], fx[f"{name}/{k}"]), f"{name}: {k}"
        np.testing.assert_allclose(f["image"], fx[f"{name}/image"], rtol=1e-12, atol=0, err_msg=name)
        np.testing.assert_allclose(f["normalizer"], fx[f"{name}/normalizer"], rtol=1e-12, atol=0)
        np.testing.assert_allclose(dc, fx[f"{name}/d_colors"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(dp, fx[f"{name}/d_positions"], rtol=1e-9, atol=1e-15)
        g = orc.bin_grid(pos, cutoff)
        assert np.array_equal(g["origin"], fx[f"{name}/grid_origin"])
        assert [g["n_cols"], g["n_rows"]] == list(fx[f"{name}/grid_dims"])
        assert np.array_equal(g["bin_start"], fx[f"{name}/grid_bin_start"])
        assert np.array_equal(g["point_index"], fx[f"{name}/grid_point_index"])


def test_oracle_capped_grid_fixture(orc, fx):
    # bin_grid.cpp:14 — 8192-wide positions with cell 3 hit the 2048 cap
    g = orc.bin_grid(fx["grid_capped/pos"], float(fx["grid_capped/cell"][0]))
    assert [g["n_cols"], g["n_rows"]] == [2048, 2048]
    assert np.array_equal(g["origin"], fx["grid_capped/origin"])
    assert np.array_equal(g["bin_start"], fx["grid_capped/bin_start"])
    assert np.array_equal(g["point_index"], fx["grid_capped/point_index"])


def test_oracle_any_channel_count_decomposes(orc):
    # channels are independent: a C=5 call equals per-channel C=1 calls for the
    # image and d_colors, and d_positions is their sum
    rng = np.random.default_rng(3)
    pos = rng.uniform(-1, 20, (40, 2)).astype(np.float32).astype(np.float64)
    col = rng.uniform(0, 1, (40, 5))
    up = rng.uniform(-1, 1, (16, 20, 5))
    f = orc.forward(pos, col, 20, 16, 1.3, 3.9)
    dc, dp = orc.backward(pos, col, f, up, 1.3, 3.9)
    dp_sum = np.zeros_like(dp)
    for c in range(5):
        fc = orc.forward(pos, col[:, c:c + 1], 20, 16, 1.3, 3.9)
        dcc, dpc = orc.backward(pos, col[:, c:c + 1], fc, up[..., c:c + 1], 1.3, 3.9)
        assert np.array_equal(fc["image"][..., 0], f["image"][..., c])
        assert np.array_equal(dcc[:, 0], dc[:, c])
        dp_sum += dpc
    np.testing.assert_allclose(dp_sum, dp, rtol=1e-10, atol=1e-14)


def test_oracle_vs_live_reference(orc, ref):
    """When oracle/_ref (the reference compiled from its sources) is present:
    bit-exact equality on fresh random instances, both fallback policies."""
    for seed in (101, 202, 303, 404, 505):
        inst = ref.random_instance(seed, 16, 50)
        p, c, w, h, s = inst["pos"], inst["col"], inst["width"], inst["height"], inst["sigma"]
        for cutoff in (3 * s, 1.0):
            for fb in (0, 1):
                up = np.random.default_rng(seed).uniform(-1, 1, (h, w, c.shape[1]))
                fr = ref.forward(p, c, w, h, s, cutoff, fb)
                dcr, dpr = ref.backward(p, c, fr, up, s, cutoff, fb)
                ref.free_cache(fr)
                fo = orc.forward(p, c, w, h, s, cutoff, fb)
                dco, dpo = orc.backward(p, c, fo, up, s, cutoff, fb)
                for k in ("image", "normalizer", "fallback_flag", "nearest_index", "counts"):
                    assert np.array_equal(fr[k], fo[k]), (seed, cutoff, fb, k)
                assert np.array_equal(dcr, dco) and np.array_equal(dpr, dpo)


def test_reference_oracle_untruncated(ref):
    # test_engine.cpp:251-260: forward == oracle_forward when nothing is truncated
    for seed in (21, 22, 23, 24):
        inst = ref.random_instance(seed, 12, 30)
        p, c = inst["pos"], inst["col"]
        w, h, s = inst["width"], inst["height"], inst["sigma"]
        big = float(np.hypot(max(w - 1, p[:, 0].max()) - min(0, p[:, 0].min()),
                             max(h - 1, p[:, 1].max()) - min(0, p[:, 1].min())) + 1.0)
        f = ref.forward(p, c, w, h, s, big)
        ref.free_cache(f)
        o = ref.oracle_forward(p, c, w, h, s)
        np.testing.assert_allclose(f["image"], o, rtol=1e-12, atol=1e-300)


def test_gmm_benchmark_restatement_matches_reference(ref):
    # run_benchmark's GMM branch (benchmark.cpp:88-107): block means, block
    # centres, the sigma sweep and l1_metric, restated on the C oracle
    import oracle
    orc = oracle.Oracle()
    rng = np.random.default_rng(5)
    img = rng.uniform(0, 1, (29, 34, 3)).astype(np.float32).astype(np.float64)
    for f in (1, 2, 3, 5):
        assert np.array_equal(oracle.block_mean_downsample(img, f), ref.block_mean_downsample(img, f))
        l1, best = oracle.gmm_benchmark(orc, img, f)
        rl1, rsig, _ = ref.run_benchmark_gmm(img, f)
        assert l1[best] == rl1 and [0.4 * f, 0.5 * f, 0.6 * f][best] == rsig
    l1, best = oracle.gmm_benchmark(orc, img[:, :, :1], 4, sigmas=[1.7])
    assert l1[0] == ref.run_benchmark_gmm(img[:, :, :1], 4, sigma=1.7)[0]
