"""run_benchmark's GMM branch (the paper's section 3.2 reconstruction sweep:
block-mean downsample -> one forward per sigma in {0.4, 0.5, 0.6} x factor ->
L1 against the original) on one B200 against the reference's run_benchmark
on the host cores.  Prints one JSON line per factor.

    python tools/bench_gmm.py [--size 1024 --factors 2 4 8 16 --repeat 5]
"""
import argparse, json, os, sys, time
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--channels", type=int, default=3)
    ap.add_argument("--factors", type=int, nargs="+", default=[2, 4, 8, 16])
    ap.add_argument("--repeat", type=int, default=5)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    import paper_2012_13257_b200 as gmi
    import oracle
    H = W = a.size
    yy, xx = np.mgrid[0:H, 0:W]
    rng = np.random.default_rng(7)
    img = 0.5 + 0.35 * np.sin(xx / 23.0)[:, :, None] * np.cos(yy / 17.0)[:, :, None]
    img = np.clip(img + 0.03 * rng.standard_normal((H, W, a.channels)), 0, 1).astype(np.float32)
    ctx = gmi.Context(0)
    ref = oracle.Reference() if (oracle.reference_available() and not a.no_ref) else None
    for f in a.factors:
        gmi.gmm_benchmark(img, f, ctx=ctx)  # warm-up
        t0 = time.perf_counter()
        for _ in range(a.repeat):
            row = gmi.gmm_benchmark(img, f, ctx=ctx)
        t_call = (time.perf_counter() - t0) / a.repeat
        line = {"metric": "GMM reconstruction sweep (run_benchmark gmm row: 3 forwards + L1)",
                "config": {"frame": [H, W], "channels": a.channels, "factor": f,
                           "points": ((H + f - 1) // f) * ((W + f - 1) // f)},
                "sigma_used": row["sigma_used"], "l1": row["l1"],
                "gpu_forward_ms": round(row["wall_time_ms"], 4),
                "gpu_call_ms": round(1e3 * t_call, 3)}
        if ref is not None:
            t0 = time.perf_counter()
            rl1, rsig, rms = ref.run_benchmark_gmm(img.astype(np.float64), f)
            line["reference_call_ms"] = round(1e3 * (time.perf_counter() - t0), 1)
            line["reference_forward_ms"] = round(rms, 1)
            line["reference_sigma_used"] = rsig
            line["reference_l1"] = rl1
            line["reference"] = "oracle/_ref gmi::run_benchmark (gmm), num_workers=1 (BenchmarkOptions default)"
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
