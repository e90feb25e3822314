"""Pinned host<->device copy rates on this box (the e2e ceiling): H2D, D2H
alone and both directions at once, 1 GiB each, CUDA events."""
import json, torch
n = 1 << 28  # floats = 1 GiB
dev = torch.device("cuda", 0)
h1 = torch.empty(n, pin_memory=True); h2 = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device=dev); d2 = torch.empty(n, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); [torch.cuda.current_stream().wait_stream(s) for s in (s1, s2)]; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
gb = 4 * n / 1e9
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_GBps": round(gb / t1 * 1e3, 1), "d2h_GBps": round(gb / t2 * 1e3, 1),
                  "duplex_GBps_each_way": round(gb / t3 * 1e3, 1), "bytes": 4 * n}))
