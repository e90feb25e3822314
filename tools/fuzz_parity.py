"""Randomised parity sweep of the CUDA path against the C oracle (the
restatement pinned to the reference): random frames, batch sizes, point
counts, channel counts, sigma / cutoff, clusters, points outside the frame,
integer lattices, fallback modes, synchronous and asynchronous contexts.

Pass rule: the north-star tolerance exactly, |a-b| <= 1e-6 + 1e-5 max(|a|,|b|)
for image, d_colors and d_positions (no widened floors, no excess allowance),
bit-exact fallback sets and nearest indices.  Every failing image is saved as
a replayable case under --out (tests/test_gpu_fuzz_cases.py replays the ones
committed under tests/golden/fuzz_cases/); the run exits non-zero if any case
failed.

Domains:
  baseline  the BASELINE configs' regimes: sigma 1 / 1.5 / 4 at cutoff
            3 sigma, 0.2-0.3 points/px, C in {1, 3}, configs[4]'s C = 64 with
            its cluster at sigma 4; random frames, far-out points, lattices.
  contract  inputs the reference accepts (C in {1,3}; configs[4]'s C = 64
            at its sigma through the C restatement, which is the reference
            per channel group), sigma in the reference's random_instance
            range [0.5, 4] plus the BASELINE sigmas, cutoff 1..5 sigma,
            densities 0.02..3 points/px, the configs[4] cluster (5% in 32 px)
            and a 6x denser one (30% in 16 px), far-out points, integer /
            half-integer lattices (inclusion ties), both fallbacks.
  stress    beyond every BASELINE config: C in {2,4,5,8,16,33} at any sigma,
            sigma down to 0.3, 30-80% of the points piled into 1-16 px.

    python tools/fuzz_parity.py [--seconds 300] [--seed 0] [--domain contract]
"""
import argparse, os, sys, time
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def excess(a, b):
    """max over entries of |a-b| / (1e-6 + 1e-5 max(|a|,|b|)): <= 1 is inside
    the north-star tolerance; also the flat index of the worst entry."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0, -1
    e = np.abs(a - b) / (1e-6 + 1e-5 * np.maximum(np.abs(a), np.abs(b)))
    k = int(np.argmax(e))
    return float(e.flat[k]), k


def draw_case(rng, domain, large):
    W = int(rng.integers(1, 640 if large else 200))
    H = int(rng.integers(1, 640 if large else 160))
    B = int(rng.integers(1, 4))
    if domain == "baseline":
        # the BASELINE configs' regimes (configs[0..4]): sigma 1 / 1.5 / 4 at
        # cutoff 3 sigma, densities around their 0.25 points/px, C = 3 (and
        # 1), configs[4]'s C = 64 with its 5% / 32 px cluster at sigma 4
        C = int(rng.choice([1, 3, 3, 3, 64] if not large else [1, 3, 3]))
        sigma = 4.0 if C == 64 else float(rng.choice([1.0, 1.5, 4.0]))
        cluster, cluster_px = (0.05, 32) if C == 64 else (0.0, 32)
        dens = float(rng.choice([0.2, 0.25, 0.3]))
        N = max(1, int(dens * W * H))
        N = min(N, 250000 if large else 60000)
        if C == 64:
            N = min(N, 8000)
            B = 1
        return dict(W=W, H=H, B=B, C=C, sigma=sigma, cutoff=3.0 * sigma, N=N, cluster=cluster,
                    cluster_px=cluster_px, mode=int(rng.choice([0, 0, 1, 2])),
                    fb="nearest" if rng.random() < 0.8 else "zero", seed=int(rng.integers(1 << 30)))
    if domain == "contract":
        C = int(rng.choice([1, 3, 3, 3, 64] if not large else [1, 3, 3]))
        sigma = float(rng.choice([0.5, 1.0, 1.5, 2.0, 4.0, rng.uniform(0.5, 4.0)]))
        if C == 64:  # configs[4]'s wide-channel case: sigma 4 (and 2)
            sigma = float(rng.choice([2.0, 4.0]))
        # configs[4]'s cluster (5% in 32 px) and a 6x denser one
        cluster, cluster_px = [(0.0, 32), (0.0, 32), (0.0, 32), (0.05, 32), (0.3, 16)][
            int(rng.integers(0, 5))]
    else:
        C = int(rng.choice([1, 2, 3, 4, 5, 8, 16, 33]))
        sigma = float(rng.choice([0.5, 0.8, 1.0, 1.5, 2.0, 3.0, rng.uniform(0.3, 4.0)]))
        cluster = float(rng.choice([0.0, 0.0, 0.3, 0.8]))
        cluster_px = int(rng.choice([1, 3, 16]))
    k = float(rng.choice([3.0, 3.0, 2.0, 2.5, 4.0, rng.uniform(1.0, 5.0)]))
    dens = float(rng.choice([0.02, 0.1, 0.25, 0.3, 1.0, 3.0]))
    N = max(1, int(dens * W * H))
    N = min(N, 250000 if large else 60000)
    if C == 64:
        N = min(N, 8000)
        B = 1
    return dict(W=W, H=H, B=B, C=C, sigma=sigma, cutoff=k * sigma, N=N, cluster=cluster,
                cluster_px=cluster_px, mode=int(rng.integers(0, 4)),
                fb="nearest" if rng.random() < 0.8 else "zero", seed=int(rng.integers(1 << 30)))


def make_inputs(orc, rng, c):
    pos, col, up = orc.synth_batch(c["seed"], c["B"], c["N"], c["C"], c["W"], c["H"],
                                   cluster_frac=c["cluster"], cluster_px=c["cluster_px"])
    W, H, N, B = c["W"], c["H"], c["N"], c["B"]
    if c["mode"] == 1:  # some points far outside the frame
        m = max(1, N // 10)
        pos[:, :m] = rng.uniform(-3 * max(W, H), 4 * max(W, H), (B, m, 2)).astype(np.float32)
    elif c["mode"] == 2:  # integer / half-integer lattice (boundary ties)
        step = float(rng.choice([1.0, 2.0, 3.0]))
        xs, ys = np.meshgrid(np.arange(0, W, step), np.arange(0, H, step))
        lat = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float32)
        lat += np.float32(rng.choice([0.0, 0.5]))
        n2 = min(N, lat.shape[0])
        pos[:, :n2] = lat[:n2]
    return pos, col, up


def check_image(orc, pos, col, up, img, dc, dp, flag, near, W, H, sigma, cutoff, fb):
    """-> (ok_exact, {name: (excess, flat index)}, reference dict)."""
    fbi = 0 if fb == "nearest" else 1
    p64, c64, u64 = (x.astype(np.float64) for x in (pos, col, up))
    r = orc.forward(p64, c64, W, H, sigma, cutoff, fbi)
    rdc, rdp = orc.backward(p64, c64, r, u64, sigma, cutoff, fbi)
    ok = np.array_equal(flag, r["fallback_flag"])
    if fb == "nearest":
        ok &= np.array_equal(near, np.where(r["fallback_flag"] == 1, r["nearest_index"], -1))
    ex = {"image": excess(img, r["image"]), "d_colors": excess(dc, rdc),
          "d_positions": excess(dp, rdp)}
    return ok, ex, dict(image=r["image"], d_colors=rdc, d_positions=rdp,
                        counts=r["counts"], flag=r["fallback_flag"], near=r["nearest_index"])


def describe(name, k, got, want, ref, C):
    """One line about the worst entry: value, and for point outputs how many
    pixels the point reaches and whether fallback pixels route to it."""
    g, w = float(np.asarray(got).flat[k]), float(np.asarray(want).flat[k])
    s = f"{name}[{k}] got {g:.9g} want {w:.9g} |d| {abs(g - w):.3e}"
    if name != "image":
        i = k // (C if name == "d_colors" else 2)
        routed = int(np.sum((ref["flag"] == 1) & (ref["near"] == i)))
        s += f" (point {i}, routed fallback px {routed})"
    else:
        px = k // C
        s += f" (pixel {px}, contributors {int(ref['counts'].flat[px])})"
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--domain", choices=["baseline", "contract", "stress"], default="contract")
    ap.add_argument("--large", action="store_true",
                    help="fewer, larger cases (frames up to 640 px, up to 250k points)")
    ap.add_argument("--out", default="gpurun_out/fuzz_fail")
    ap.add_argument("--max-fail", type=int, default=400)
    ap.add_argument("--max-save", type=int, default=12)
    ap.add_argument("--inject-fault", action="store_true",
                    help="negative path: GMI_CTX_INJECT_FAULT corrupts d_colors[0]; the run must FAIL")
    ap.add_argument("--precise", action="store_true",
                    help="contexts with GMI_CTX_PRECISE (f64 weights, sums and image)")
    a = ap.parse_args()
    import oracle
    import paper_2012_13257_b200 as gmi
    orc = oracle.Oracle()
    rng = np.random.default_rng(a.seed)
    sync_ctx, async_ctx = gmi.Context(0), gmi.Context(0)
    extra = (gmi.CTX_PRECISE if a.precise else 0) | (gmi.CTX_INJECT_FAULT if a.inject_fault else 0)
    sync_ctx.set_flags(extra)
    async_ctx.set_flags(gmi.CTX_ASYNC_ERRORS | extra)
    t_end = time.time() + a.seconds
    n_cases, n_images, worst, fails, saved = 0, 0, 0.0, 0, 0
    hist = {"image": 0, "d_colors": 0, "d_positions": 0, "exact": 0}
    os.makedirs(a.out, exist_ok=True)
    while time.time() < t_end and fails < a.max_fail:
        c = draw_case(rng, a.domain, a.large)
        pos, col, up = make_inputs(orc, rng, c)
        W, H, sigma, cutoff, fb = c["W"], c["H"], c["sigma"], c["cutoff"], c["fb"]
        ctx = async_ctx if rng.random() < 0.5 else sync_ctx
        img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, fb, ctx=ctx)
        dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, fb, ctx=ctx)
        ctx.synchronize()
        _, flag, near = cache.pixels()
        desc = (f"case {n_cases}: B={c['B']} N={c['N']} C={c['C']} {W}x{H} sigma={sigma:.3f} "
                f"r={cutoff:.3f} cluster={c['cluster']}/{c['cluster_px']}px mode={c['mode']} fb={fb}")
        for b in range(c["B"]):
            ok, ex, ref = check_image(orc, pos[b], col[b], up[b], img[b], dc[b], dp[b], flag[b],
                                      near[b], W, H, sigma, cutoff, fb)
            n_images += 1
            e = max(v[0] for v in ex.values())
            worst = max(worst, e)
            if ok and e <= 1.0:
                continue
            fails += 1
            if not ok:
                hist["exact"] += 1
                print(f"FAIL exact (fallback set / nearest index): {desc} image {b}", flush=True)
            for name, (v, k) in ex.items():
                if v > 1.0:
                    hist[name] += 1
                    got = {"image": img[b], "d_colors": dc[b], "d_positions": dp[b]}[name]
                    print(f"FAIL {v:.2f}x {desc} image {b}: "
                          f"{describe(name, k, got, ref[name], ref, c['C'])}", flush=True)
            # replayable fixture (small cases only: the box returns <= 64 MiB)
            if saved < a.max_save and pos[b].size + up[b].size <= 400000:
                saved += 1
                np.savez_compressed(os.path.join(a.out, f"{a.domain}_s{a.seed}_c{n_cases}_b{b}.npz"),
                                    pos=pos[b], col=col[b], up=up[b], W=W, H=H, sigma=sigma,
                                    cutoff=cutoff, fb=fb, excess=e)
        n_cases += 1
        if n_cases % 100 == 0:
            print(f"{n_cases} cases, {n_images} images, {fails} failing, worst {worst:.2f}x "
                  f"({desc})", flush=True)
    verdict = "fuzz ok" if fails == 0 else "FUZZ FAILED"
    mode = a.domain + (" large" if a.large else "") + (" precise" if a.precise else "")
    print(f"{verdict} [{mode}, seed {a.seed}]: {n_cases} cases, "
          f"{n_images} images, {a.seconds:.0f} s, worst {worst:.2f}x tolerance, {fails} image(s) "
          f"over 1x (by output: {hist})")
    sys.exit(0 if fails == 0 else 1)


if __name__ == "__main__":
    main()
