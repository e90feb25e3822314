import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle, paper_2012_13257_b200 as gmi
d = np.load("tools/_fuzz_fail.npz")
pos, col, up = d["pos"], d["col"], d["up"]
W, H, sigma, cutoff, fb = int(d["W"]), int(d["H"]), float(d["sigma"]), float(d["cutoff"]), str(d["fb"])
orc = oracle.Oracle()
ctx = gmi.Context(0)
img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, fb, ctx=ctx)
dc, dp = gmi.backward_batch(pos, col, cache, up, sigma, cutoff, fb, ctx=ctx)
_, flag, near = cache.pixels()
cnt = gmi.forward_counts(cache)
def rep(name, a, bb):
    a, bb = np.asarray(a, np.float64), np.asarray(bb, np.float64)
    bad = np.abs(a - bb) > 1e-6 + 1e-5 * np.maximum(np.abs(a), np.abs(bb))
    print(name, "bad", int(bad.sum()), "of", bad.size, "max abs diff", float(np.abs(a - bb).max()))
    if bad.any():
        for i in np.argwhere(bad)[:6]:
            print("   at", tuple(int(v) for v in i), a[tuple(i)], bb[tuple(i)])
for b in range(pos.shape[0]):
    p64, c64, u64 = (x[b].astype(np.float64) for x in (pos, col, up))
    r = orc.forward(p64, c64, W, H, sigma, cutoff, 0)
    rdc, rdp = orc.backward(p64, c64, r, u64, sigma, cutoff, 0)
    print("image", b, "flags equal", np.array_equal(flag[b], r["fallback_flag"]), "counts equal", np.array_equal(cnt[b], r["counts"]),
          "nearest equal", np.array_equal(near[b], np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)), "fallback px", int(r["fallback_flag"].sum()))
    if not np.array_equal(near[b], np.where(r["fallback_flag"] == 1, r["nearest_index"], -1)):
        bad = np.argwhere(near[b] != np.where(r["fallback_flag"] == 1, r["nearest_index"], -1))
        print("  nearest mismatches", len(bad), [(tuple(int(v) for v in i), int(near[b][tuple(i)]), int(r["nearest_index"][tuple(i)])) for i in bad[:5]])
    rep(" image", img[b], r["image"]); rep(" d_col", dc[b], rdc); rep(" d_pos", dp[b], rdp)
