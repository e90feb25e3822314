"""One small forward + backward per hot-path kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_case.py fast3

Modes: fast1 fast3 fast4 (C <= 4 TMA gather + point-major backward), wide
(C > 4 gather / backward), generic (GMI_GENERIC: the generic gather),
precise (GMI_CTX_PRECISE f64 path), cluster (multi-chunk tiles with the f64
fold), sparse (fallback pixels: K3 nearest search, K5 routing), async (the
pipelined host-buffer API with asynchronous errors), bins (the bit-exact
bin-grid export incl. a capped grid)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(mode):
    if mode == "generic":
        os.environ["GMI_GENERIC"] = "1"
    import oracle
    import paper_2012_13257_b200 as gmi

    orc = oracle.Oracle()
    ctx = gmi.Context(0)
    C = {"fast1": 1, "fast4": 4, "wide": 9}.get(mode, 3)
    W, H, N, sigma, cutoff = 70, 52, 900, 1.5, 4.5
    cluster, cpx = 0.0, 32
    if mode == "sparse":
        N = 60
    if mode == "cluster":
        N, cluster, cpx = 6000, 0.6, 6
    if mode == "precise":
        ctx.set_flags(gmi.CTX_PRECISE)
    if mode == "async":
        ctx.set_flags(gmi.CTX_ASYNC_ERRORS)
    if mode == "bins":
        pos, _, _ = orc.synth_batch(5, 1, 3000, 1, 400, 300, upstream=False)
        g = gmi.bin_grid(pos[0], 3.0, ctx=ctx)
        far = np.concatenate([pos[0], [[9000.0, -7000.0]]]).astype(np.float32)
        g2 = gmi.bin_grid(far, 1.0, ctx=ctx)   # capped 2048-cell grid
        print("bins ok", g["n_cols"], g2["n_cols"])
        return
    pos, col, up = orc.synth_batch(7, 2, N, C, W, H, cluster_frac=cluster, cluster_px=cpx)
    img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, ctx=ctx)
    ctx.synchronize()
    r = orc.forward(pos[0], col[0], W, H, sigma, cutoff)
    err = float(np.abs(img[0] - r["image"]).max())
    print(f"{mode} ok: max|d image| {err:.2e}, fallback px {cache.fallback_count}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "fast3")
