"""configs[4] cluster-window image check (C oracle): host API (pageable and
pinned) vs device API.  python tools/diag_cfg4.py"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import oracle
import paper_2012_13257_b200 as gmi

orc = oracle.Oracle()
W = H = 2048
N, C, sigma, cutoff = 1048576, 64, 4.0, 12.0
pos, col, up = orc.synth_batch(501, 1, N, C, W, H, cluster_frac=0.05, cluster_px=32, upstream=False)
ctx = gmi.Context(0)
nc = int(0.05 * N)
cx0, cy0 = np.floor(pos[0, :nc].min(0)).astype(int)
x0, y0, w, h = max(0, cx0 - 24), max(0, cy0 - 24), 48, 40
m = 20
keep = ((pos[0, :, 0] >= x0 - m) & (pos[0, :, 0] <= x0 + w - 1 + m) & (pos[0, :, 1] >= y0 - m) & (pos[0, :, 1] <= y0 + h - 1 + m))
idx = np.nonzero(keep)[0]
wp = pos[0, idx].astype(np.float64) - [x0, y0]
r = orc.forward(wp, col[0, idx].astype(np.float64), w, h, sigma, cutoff)


def err(img):
    a = img[y0:y0 + h, x0:x0 + w].astype(np.float64)
    e = np.abs(a - r["image"]) / (1e-6 + 1e-5 * np.maximum(np.abs(a), np.abs(r["image"])))
    return float(e.max()), int((e > 1).sum())


img, cache = gmi.forward_batch(pos, col, W, H, sigma, cutoff, ctx=ctx)
print("host pageable", err(img[0]))
import torch
tp, tc = torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda()
out, c2 = gmi.forward_cuda(tp, tc, W, H, sigma, radius=cutoff, ctx=ctx)
ctx.synchronize()
print("device", err(out.numpy()[0]))
