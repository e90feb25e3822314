"""Precision near a dense cluster at the configs[4] scale: device image vs an
f64 brute-force evaluation of the reference formula for pixels next to the
cluster (the worst case for fp32 accumulation)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2012_13257_b200 as gmi
B, N, C, W, H, sigma, cutoff = 1, 1048576, int(sys.argv[1]) if len(sys.argv) > 1 else 64, 2048, 2048, 4.0, 12.0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
pos = torch.empty(B, N, 2, device=dev)
pos[..., 0].uniform_(-0.5, W - 0.5, generator=g); pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
nc = int(0.05 * N)
corner = torch.tensor([900.0, 700.0], device=dev)
pos[:, :nc] = corner + torch.rand(B, nc, 2, device=dev, generator=g) * 32.0
col = torch.rand(B, N, C, device=dev, generator=g)
img = torch.empty(B, H, W, C, device=dev)
ctx = gmi.Context(0)
cache = ctx.forward_device(pos, col, B, N, C, W, H, sigma, cutoff, 0, img)
torch.cuda.synchronize()
P = pos[0].double().cpu().numpy(); Cc = col[0].double().cpu().numpy(); I = img[0].cpu().numpy()
worst = 0.0
for (qy, qx) in [(700, 900), (716, 916), (731, 931), (705, 890), (690, 920), (745, 940), (710, 944), (720, 905)]:
    d2 = (qx - P[:, 0]) ** 2 + (qy - P[:, 1]) ** 2
    m = d2 <= cutoff * cutoff
    w = np.exp(-d2[m] / (2 * sigma * sigma))
    ref = (w[:, None] * Cc[m]).sum(0) / w.sum()
    err = np.abs(I[qy, qx] - ref) / (1e-6 / 1e-5 + np.abs(ref))  # |d| / (0.1 + |ref|)
    rel = np.max(np.abs(I[qy, qx] - ref) - 1e-5 * np.maximum(np.abs(I[qy, qx]), np.abs(ref)) - 1e-6)
    worst = max(worst, rel)
    print((qy, qx), "contributors", int(m.sum()), "max |d|", float(np.abs(I[qy, qx] - ref).max()),
          "tolerance excess", float(rel))
print("within tolerance" if worst <= 0 else "EXCEEDS tolerance")
