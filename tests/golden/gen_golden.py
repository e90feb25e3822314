"""Generates tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (needs /root/reference to compile oracle/_ref):

    python tests/golden/gen_golden.py

Every fixture is produced by calling the unmodified reference C++ through
oracle/_ref/libgmi_ref.so (gmi::forward, gmi::backward, gmi::build_bin_grid,
gmi::oracle_forward, gmi::random_instance, gmi::Rng).  The fixtures travel with
the repo, so the oracle restatement (oracle/gmi_oracle.c) and the GPU path can
be checked against the reference on machines where it cannot be built.
Inputs are fp32-representable (the GPU path stores fp32).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def case(R, name, pos, col, w, h, sigma, cutoff, fallback=0, seed=0, grid_cells=None):
    pos, col = f32(pos), f32(col)
    rng = np.random.default_rng(seed)
    up = f32(rng.uniform(-1, 1, (h, w, col.shape[1])))
    f = R.forward(pos, col, w, h, sigma, cutoff, fallback, 1)
    dc, dp = R.backward(pos, col, f, up, sigma, cutoff, fallback, 1)
    R.free_cache(f)
    g = R.bin_grid(pos, cutoff if grid_cells is None else grid_cells, col)
    out = {
        f"{name}/pos": pos, f"{name}/col": col, f"{name}/upstream": up,
        f"{name}/params": np.array([w, h, sigma, cutoff, fallback], np.float64),
        f"{name}/image": f["image"], f"{name}/normalizer": f["normalizer"],
        f"{name}/fallback_flag": f["fallback_flag"], f"{name}/nearest_index": f["nearest_index"],
        f"{name}/counts": f["counts"], f"{name}/d_colors": dc, f"{name}/d_positions": dp,
        f"{name}/grid_origin": g["origin"],
        f"{name}/grid_dims": np.array([g["n_cols"], g["n_rows"]], np.int64),
        f"{name}/grid_bin_start": g["bin_start"], f"{name}/grid_point_index": g["point_index"],
    }
    return out


def main():
    oracle.build(with_reference=True)
    R = oracle.Reference()
    O = oracle.Oracle()
    fx = {}
    names = []

    def add(name, *a, **k):
        fx.update(case(R, name, *a, **k))
        names.append(name)

    # test_engine.cpp:53-70 — three points shifted by (-0.5,-0.5), cutoff 10
    add("three_point", [[-0.5, -0.5], [1.5, -0.5], [-0.5, 1.5]], [[1.0], [0.0], [0.0]],
        1, 1, 1.0, 10.0)
    # test_engine.cpp:217-239 fallback policies on an out-of-range point set
    add("out_of_range_nearest", [[100, 100], [200, 200]], [[0.9], [0.1]], 4, 4, 1.0, 2.0, 0)
    add("out_of_range_zero", [[100, 100], [200, 200]], [[0.9], [0.1]], 4, 4, 1.0, 2.0, 1)
    # test_engine.cpp:241-249 total weight underflow
    add("underflow", [[1000.0, 0.0]], [[0.6]], 1, 1, 0.5, 10000.0)
    # test_engine.cpp:347-370 fallback routing
    add("fallback_routing", [[-50, 0], [-60, 0]], [[0.3], [0.7]], 2, 2, 1.0, 3.0)
    # validate.cpp:12-35 random instances (test_engine.cpp:251-260 seeds)
    for seed in (21, 22, 23, 24):
        inst = R.random_instance(seed, 12, 30)
        s = inst["sigma"]
        add(f"random_{seed}_3sigma", inst["pos"], inst["col"], inst["width"], inst["height"],
            s, 3.0 * s, 0, seed)
        add(f"random_{seed}_r1", inst["pos"], inst["col"], inst["width"], inst["height"],
            s, 1.0, 0, seed)
    # BASELINE configs[0] shape: 128^2, N=4096, C=3, sigma=1
    pos, col, _ = O.synth_batch(1, 1, 4096, 3, 128, 128, upstream=False)
    add("config1", pos[0], col[0], 128, 128, 1.0, 3.0, 0, 1)
    # sparse: many fallback pixels
    pos, col, _ = O.synth_batch(3, 1, 600, 3, 96, 80, upstream=False)
    add("sparse_fallbacks", pos[0], col[0], 96, 80, 1.0, 3.0, 0, 3)
    # clustered, sigma 4 (BASELINE configs[4] stand-in, C=3)
    pos, col, _ = O.synth_batch(5, 1, 3000, 3, 128, 128, 0.05, 16, upstream=False)
    add("clustered_sigma4", pos[0], col[0], 128, 128, 4.0, 12.0, 0, 5)
    # integer lattice: exact d^2 == r^2 ties (closed ball)
    xs, ys = np.meshgrid(np.arange(0, 30, 3), np.arange(0, 24, 3))
    lat = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float64)
    add("lattice_ties", lat, np.random.default_rng(8).uniform(0, 1, (lat.shape[0], 3)),
        30, 24, 1.0, 3.0, 0, 8)

    # bin grids only: capped axis (bin_grid.cpp:14) and test_bin_grid.cpp:65-86
    rng = np.random.default_rng(1)
    capped = f32(rng.uniform(0, 8192, (5000, 2)))
    g = R.bin_grid(capped, 3.0)
    fx.update({"grid_capped/pos": capped, "grid_capped/cell": np.array([3.0]),
               "grid_capped/origin": g["origin"],
               "grid_capped/dims": np.array([g["n_cols"], g["n_rows"]], np.int64),
               "grid_capped/bin_start": g["bin_start"], "grid_capped/point_index": g["point_index"]})

    # gmi::Rng (rng.hpp:12-59) first outputs for seed 42
    fx["rng/seed42"] = R.rng_u64(42, 16)
    # core.cpp:49-53 known values (test_core.cpp:11-17)
    fx["kat/gaussian_weight"] = np.array([R.gaussian_weight(1, 0, 0, 0, 1.0),
                                          R.gaussian_weight(0.5, 0.5, 2, 0, 1.0)])
    fx["names"] = np.array(names)
    out = os.path.join(HERE, "reference_fixtures.npz")
    np.savez_compressed(out, **fx)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB, {len(names)} cases)")


if __name__ == "__main__":
    main()
