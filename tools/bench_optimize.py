"""optimize_points (the paper's section 3.3 experiment: render -> L1 loss ->
backward -> descent, rebinning every step) on one B200 against the reference
loop on the host cores.  Prints one JSON line (steps per second both ways).

    python tools/bench_optimize.py [--size 256 --points 16384 --steps 50]
"""
import argparse, json, os, sys, time
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--points", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--ref-steps", type=int, default=5)
    a = ap.parse_args()
    import paper_2012_13257_b200 as gmi
    import oracle
    W = H = a.size
    rng = np.random.default_rng(3)
    pos = np.stack([rng.uniform(-0.5, W - 0.5, a.points), rng.uniform(-0.5, H - 0.5, a.points)], 1)
    pos = pos.astype(np.float32)
    col = rng.uniform(0, 1, (a.points, 3)).astype(np.float32)
    tgt = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    ps = gmi.PointSet(pos, col)
    gmi.optimize_points(ps, tgt, 1.0, steps=2, log_every=100, log_trajectory=False)  # warm-up
    t0 = time.perf_counter()
    out = gmi.optimize_points(ps, tgt, 1.0, steps=a.steps, log_every=a.steps, log_trajectory=False)
    t_gpu = time.perf_counter() - t0
    line = {"metric": "optimize_points steps/s (render + L1 + backward + descent, rebinning)",
            "config": {"frame": [H, W], "points": a.points, "channels": 3, "sigma": 1.0,
                       "steps": a.steps},
            "gpu_steps_per_s": round(a.steps / t_gpu, 2),
            "loss_first_last": [float(out["loss_curve"][0]), float(out["loss_curve"][-1])]}
    if oracle.reference_available() and a.ref_steps > 0:
        ref = oracle.Reference()
        t0 = time.perf_counter()
        _, _, rl = ref.optimize_points(pos.astype(np.float64), col.astype(np.float64),
                                       tgt.astype(np.float64), 1.0, 3.0, a.ref_steps, 0.5)
        t_ref = time.perf_counter() - t0
        line["reference_steps_per_s"] = round(a.ref_steps / t_ref, 3)
        line["reference"] = "oracle/_ref gmi::optimize_points, num_workers=1 (the reference's binding default)"
    print(json.dumps(line))


if __name__ == "__main__":
    main()
