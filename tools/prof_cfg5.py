"""configs[4]-shaped fwd+bwd (B images) for ncu captures."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2012_13257_b200 as gmi
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N, C, W, H = 1048576, 64, 2048, 2048
dev = torch.device('cuda', 0)
g = torch.Generator(device=dev); g.manual_seed(1)
pos = torch.empty(B, N, 2, device=dev)
pos[..., 0].uniform_(-0.5, W - 0.5, generator=g); pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
nc = N // 20
corner = torch.rand(B, 1, 2, device=dev, generator=g) * torch.tensor([W - 32.0, H - 32.0], device=dev)
pos[:, :nc] = corner + torch.rand(B, nc, 2, device=dev, generator=g) * 32.0
col = torch.rand(B, N, C, device=dev, generator=g); up = torch.rand(B, H, W, C, device=dev, generator=g) * 2 - 1
img = torch.empty(B, H, W, C, device=dev); dc = torch.empty(B, N, C, device=dev); dp = torch.empty(B, N, 2, device=dev)
ctx = gmi.Context(0); ctx.set_flags(1)
for it in range(2):
    cache = ctx.forward_device(pos, col, B, N, C, W, H, 4.0, 12.0, 0, img)
    ctx.backward_device(pos, col, B, N, C, W, H, 4.0, 12.0, 0, cache, up, dc, dp)
    ctx.synchronize()
    del cache
print("ok")
