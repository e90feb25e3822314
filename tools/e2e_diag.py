"""Per-step diagnosis of the host-buffer (e2e) path at the bench's config 3:
host time of each gmi_forward_host / gmi_backward_host / cache free call and
the device time of each step (events on the ctx stream after a join)."""
import ctypes as Cty, json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2012_13257_b200 as gmi
B, N, C, W, H, sigma, cutoff = 64, 262144, 3, 1024, 1024, 1.5, 4.5
if len(sys.argv) > 1 and sys.argv[1] == "4":  # BASELINE configs[3]
    B, N, C, W, H, sigma, cutoff = 1, 16777216, 3, 8192, 8192, 1.0, 3.0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
pos = torch.empty(B, N, 2, device=dev)
pos[..., 0].uniform_(-0.5, W - 0.5, generator=g); pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
col = torch.rand(B, N, C, device=dev, generator=g); up = torch.rand(B, H, W, C, device=dev, generator=g) * 2 - 1
pinned = [pos.cpu().pin_memory(), col.cpu().pin_memory(), up.cpu().pin_memory(),
          torch.empty(B, H, W, C).pin_memory(), torch.empty(B, N, C).pin_memory(), torch.empty(B, N, 2).pin_memory()]
hpos, hcol, hup, himg, hdc, hdp = (t.numpy() for t in pinned)
fp = Cty.POINTER(Cty.c_float)
cfg = gmi._lib.GmiConfig(sigma, cutoff, 0, W, H)
for mode in (1, 0, 1):
    ctx = gmi.Context(0)
    ctx.set_flags(mode)
    stream = torch.cuda.ExternalStream(ctx.stream)
    rows = []
    for k in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        t0 = time.perf_counter()
        h = Cty.c_void_p()
        gmi._check(gmi.lib.gmi_forward_host(ctx.handle, hpos.ctypes.data_as(fp), hcol.ctypes.data_as(fp),
                                            B, N, C, Cty.byref(cfg), himg.ctypes.data_as(fp), Cty.byref(h)))
        t1 = time.perf_counter()
        gmi._check(gmi.lib.gmi_backward_host(ctx.handle, hpos.ctypes.data_as(fp), hcol.ctypes.data_as(fp),
                                             B, N, C, Cty.byref(cfg), h, hup.ctypes.data_as(fp),
                                             hdc.ctypes.data_as(fp), hdp.ctypes.data_as(fp)))
        t2 = time.perf_counter()
        gmi.lib.gmi_cache_free(h)
        t3 = time.perf_counter()
        ctx.join_host_copies()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t4 = time.perf_counter()
        rows.append({"fwd_call_ms": round(1e3 * (t1 - t0), 2), "bwd_call_ms": round(1e3 * (t2 - t1), 2),
                     "free_ms": round(1e3 * (t3 - t2), 2), "wall_ms": round(1e3 * (t4 - t0), 2),
                     "event_ms": round(e0.elapsed_time(e1), 2)})
    print(json.dumps({"async": mode, "steps": rows}))
    del ctx
