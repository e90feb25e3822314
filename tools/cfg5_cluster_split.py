"""configs[4] shape with and without the 5% cluster: per-phase device times
(how much of the wide kernels' time the clustered tiles / cells cost)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2012_13257_b200 as gmi

B, N, C, W, H = 8, 1048576, 64, 2048, 2048
dev = torch.device('cuda', 0)
for frac in (0.05, 0.0):
    g = torch.Generator(device=dev); g.manual_seed(1)
    pos = torch.empty(B, N, 2, device=dev)
    pos[..., 0].uniform_(-0.5, W - 0.5, generator=g); pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
    nc = int(frac * N)
    if nc:
        corner = torch.rand(B, 1, 2, device=dev, generator=g) * torch.tensor([W - 32.0, H - 32.0], device=dev)
        pos[:, :nc] = corner + torch.rand(B, nc, 2, device=dev, generator=g) * 32.0
    col = torch.rand(B, N, C, device=dev, generator=g); up = torch.rand(B, H, W, C, device=dev, generator=g) * 2 - 1
    img = torch.empty(B, H, W, C, device=dev); dc = torch.empty(B, N, C, device=dev); dp = torch.empty(B, N, 2, device=dev)
    ctx = gmi.Context(0); ctx.set_flags(1); ctx.set_profiling(True)
    for it in range(3):
        if it == 1:
            ctx.phase_times(reset=True)
        cache = ctx.forward_device(pos, col, B, N, C, W, H, 4.0, 12.0, 0, img)
        ctx.backward_device(pos, col, B, N, C, W, H, 4.0, 12.0, 0, cache, up, dc, dp)
        ctx.synchronize()
        del cache
    ms, calls = ctx.phase_times(reset=True)
    print(f"cluster={frac}:", {n: round(ms[k] / max(1, calls[k]), 3) for k, n in enumerate(gmi.Context.PHASES)})
