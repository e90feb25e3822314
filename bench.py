"""Headline benchmark: fused forward+backward Gaussian-mixture interpolation.

Workload (BASELINE.json configs[2], the one the metric is quoted on):
B=64 images per GPU, N=262,144 points, C=3, output 1024x1024, sigma=1.5,
cutoff 3*sigma = 4.5.  One "step" = gmi_forward + gmi_backward over the whole
batch.  Synthetic inputs (positions U(-0.5, W-0.5), colours U[0,1), upstream
U(-1,1)), generated on the device with torch (plumbing only).

    python bench.py [--gpus N --steps K --warmup W] [--config 1..5] [--impl reference]

--gpus N without a launcher re-runs this script as N ranks (torchrun, one
process per GPU, rendezvous on 127.0.0.1); each rank runs the product's
multi-GPU driver (paper_2012_13257_b200.multi: BatchShards, or BandSplit for
--config 4).

value    device-resident throughput (output Mpix/s, whole job), each timed
         step one replay of a CUDA graph of the library's calls
e2e      the same through the host-buffer C-ABI (gmi_forward_host /
         gmi_backward_host): H2D of positions/colours/upstream and D2H of the
         image and both gradients inside the timed region, pinned buffers;
         e2e.numpy_shim: the reference-shaped numpy shim (forward_batch /
         backward_batch) on plain pageable arrays
roofline the binding roof of the step's algorithmic counts (SURVEY §8d:
         max of FP32 pipe, MUFU, HBM), for the dominant kernel per launch
         (`frac`) and the whole step (`step_frac`); the other two beside it
Timing: CUDA events on the library's stream, warm-up first, barrier +
synchronize around the timed region, max over ranks; ms_per_step is the
total / K, ms_per_step_median the median step.  Inputs (B*...) are far
larger than L2 (126 MB), so no explicit flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(B=64, N=262144, C=3, W=1024, H=1024, sigma=1.5, cutoff=4.5)
METRIC = "output Mpixels/s fwd+bwd at 1024^2, N=262k pts, C=3 (1/2/4/8 B200) vs CPU"
WORKLOAD = "B=64 x 1024^2, N=262144, C=3, sigma=1.5, cutoff=3sigma (BASELINE configs[2])"
# BASELINE.json configs (1-based); the headline line is config 3 (the default)
CONFIGS = {
    1: dict(B=1, N=4096, C=3, W=128, H=128, sigma=1.0, cutoff=3.0, fwd_only=True,
            workload="B=1 x 128^2, N=4096, C=3, sigma=1, forward only (BASELINE configs[0])"),
    2: dict(B=16, N=65536, C=3, W=512, H=512, sigma=1.0, cutoff=3.0,
            workload="B=16 x 512^2, N=65536, C=3, sigma=1 (BASELINE configs[1])"),
    3: dict(CFG, workload=WORKLOAD),
    4: dict(B=1, N=16777216, C=3, W=8192, H=8192, sigma=1.0, cutoff=3.0,
            workload="B=1 x 8192^2, N=16M, C=3, sigma=1, single GPU (BASELINE configs[3])"),
    5: dict(B=8, N=1048576, C=64, W=2048, H=2048, sigma=4.0, cutoff=12.0, cluster=0.05,
            workload="B=8 x 2048^2, N=1M (5% in a 32^2 cluster), C=64, sigma=4 (BASELINE configs[4])"),
}


def pcie_duplex_gbps(dev, mib: int = 256) -> float:
    """Pinned host<->device copy rate with both directions in flight (GB/s
    each way, best of 3): the ceiling of the host-buffer (e2e) step."""
    import torch
    n = mib << 18
    h1, h2 = torch.empty(n, pin_memory=True), torch.empty(n, pin_memory=True)
    d1, d2 = torch.empty(n, device=dev), torch.empty(n, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s1)
        torch.cuda.current_stream(dev).wait_stream(s2)
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1))
    return 4 * n / (best * 1e-3) / 1e9


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()),
                 default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


def traffic_of(kernel: str, config: int, batch: int):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture of this workload (profiles/traffic_cfg3.json, made by
    tools/capture_traffic.sh + tools/traffic_json.py), else None."""
    if config != 3 or batch != CFG["B"]:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_cfg3.json")) as f:
            d = json.load(f)
        v = d.get(kernel, {}).get("traffic_bytes")
        return int(v) if v else None
    except Exception:
        return None


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "gmi" else "gloo"
        dist.init_process_group(backend, init_method="env://")
    return world, rank, local


def cpu_reference_sample(cfg, seconds_budget: float, max_images: int, seed: int = 7):
    """Times the UNMODIFIED reference CPU path (oracle/_ref, compiled from the
    reference sources) — gmi::forward + gmi::backward per image with
    num_workers = all host threads — on a bounded sample of the workload.
    Returns (Mpix/s, images, threads, seconds, kind)."""
    import numpy as np

    import oracle

    if oracle.reference_available():
        impl, kind = oracle.Reference(), "reference"
    else:
        if not oracle.oracle_available():
            oracle.build(with_reference=False)
        impl, kind = oracle.Oracle(), "port"
    threads = os.cpu_count() or 1
    gen = oracle.Oracle() if oracle.oracle_available() else None
    if gen is None:
        oracle.build(with_reference=False)
        gen = oracle.Oracle()
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    done, elapsed = 0, 0.0
    while done < max_images and (done == 0 or elapsed < seconds_budget):
        pos, col, up = gen.synth_batch(seed + done, 1, cfg["N"], C, W, H)
        p64, c64, u64 = (pos[0].astype(np.float64), col[0].astype(np.float64),
                         up[0].astype(np.float64))
        t0 = time.perf_counter()
        if kind == "reference":
            impl.forward_backward(p64, c64, W, H, cfg["sigma"], cfg["cutoff"], u64, 0, threads)
        else:
            f = impl.forward(p64, c64, W, H, cfg["sigma"], cfg["cutoff"])
            impl.backward(p64, c64, f, u64, cfg["sigma"], cfg["cutoff"])
        elapsed += time.perf_counter() - t0
        done += 1
    threads_used = threads if kind == "reference" else 1
    return done * W * H / elapsed / 1e6, done, threads_used, elapsed, kind


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)
    on the box's host cores, rank 0 only; each step = one image of the
    workload (bounded sample)."""
    if rank != 0:
        return
    import numpy as np

    import oracle

    cfg = CFG
    if oracle.reference_available():
        impl, kind = oracle.Reference(), "reference"
    else:
        impl, kind = None, "port"
        if not oracle.oracle_available():
            oracle.build(with_reference=False)
    gen = oracle.Oracle()
    threads = os.cpu_count() or 1
    W, H = cfg["W"], cfg["H"]
    times = []
    for s in range(args.warmup + args.steps):
        pos, col, up = gen.synth_batch(100 + s, 1, cfg["N"], cfg["C"], W, H)
        p64, c64, u64 = (a[0].astype(np.float64) for a in (pos, col, up))
        t0 = time.perf_counter()
        if kind == "reference":
            impl.forward_backward(p64, c64, W, H, cfg["sigma"], cfg["cutoff"], u64, 0, threads)
        else:
            f = gen.forward(p64, c64, W, H, cfg["sigma"], cfg["cutoff"])
            gen.backward(p64, c64, f, u64, cfg["sigma"], cfg["cutoff"])
        t = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(t)
    total = sum(times)
    value = args.steps * W * H / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mpix/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD + " — one image per step (bounded CPU sample)",
                   "global_batch": 1, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpix/s", "cores": threads,
                         "kind": kind, "sample": f"{args.steps} images of 1024^2 after {args.warmup} warm-up"},
        "e2e": {"value": round(value, 4), "unit": "Mpix/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> bool:
    """`--gpus N` without a launcher: re-run this script as N ranks (torchrun,
    one process per GPU, rendezvous on 127.0.0.1).  True when it did."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # communicator lines on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    sys.exit(subprocess.call(cmd, env=env))


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# roofline peaks of the non-tensor pipes (B200: 148 SMs; FP32 128 lanes and
# MUFU 16 lanes per SM per clock at the max SM clock — the nominal rates, a
# harder bar than the measured FFMA 122 / EX2 15.9, profiles/ubench_pipes_b200.txt)
def pipe_peaks(sm_mhz: float):
    return 148 * 128 * sm_mhz * 1e6, 148 * 16 * sm_mhz * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gmi", choices=["gmi", "reference"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each timed step as one captured CUDA graph (auto: every "
                         "config but the multi-GPU row bands, whose step holds a collective)")
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS),
                    help="BASELINE.json config (1-based); 3 is the headline")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    self_launch(args)
    if args.impl == "reference":
        world, rank, local = dist_setup(args)
        run_reference_arm(args, world, rank)
        return

    import numpy as np
    import torch

    import paper_2012_13257_b200 as gmi
    from paper_2012_13257_b200 import multi

    assert args.warmup >= 3, "contract: at least 3 warm-up steps"
    group = multi.Group("nccl")
    world, rank, local = group.world, group.rank, group.local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["B"] = args.batch
    fwd_only = cfg.get("fwd_only", False)
    B, N, C, W, H = cfg["B"], cfg["N"], cfg["C"], cfg["W"], cfg["H"]
    sigma, cutoff = cfg["sigma"], cfg["cutoff"]

    stream = group.stream
    ctx = group.ctx
    ctx.set_flags(1)  # asynchronous validation errors; checked after the loop

    # configs[3] on N > 1 GPUs: ONE image split into row bands (strong
    # scaling); every rank generates the same point set
    band = args.config == 4 and world > 1
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + (0 if band else rank))
    with torch.cuda.stream(stream):
        pos = torch.empty(B, N, 2, device=dev)
        pos[..., 0].uniform_(-0.5, W - 0.5, generator=g)
        pos[..., 1].uniform_(-0.5, H - 0.5, generator=g)
        nc = int(cfg.get("cluster", 0.0) * N)
        if nc:
            # configs[4]: the first 5% of the points in one 32x32-pixel square
            corner = torch.rand(B, 1, 2, device=dev, generator=g) * torch.tensor([W - 32.0, H - 32.0], device=dev)
            pos[:, :nc] = corner + torch.rand(B, nc, 2, device=dev, generator=g) * 32.0
        col = torch.rand(B, N, C, device=dev, generator=g)
        up = torch.rand(B, H, W, C, device=dev, generator=g) * 2 - 1
    stream.synchronize()
    H_full = H
    if band:
        # the product's band driver: plan (halo certified for far nearest-
        # point fallbacks), band-local points on the device, NCCL SUM of the
        # shared points' partial gradients inside every step
        splitter = multi.BandSplit(group, pos[0].cpu().numpy(), col[0].cpu().numpy(), W, H,
                                   sigma, cutoff)
        r0, r1 = splitter.rows
        with torch.cuda.stream(stream):
            up = up[:, r0:r1].contiguous()
        stream.synchronize()
        N, H = splitter.N, r1 - r0

        def step():
            return splitter.step(up)
        img = splitter.image
    else:
        shards = multi.BatchShards(group, W, H, sigma, cutoff)
        with torch.cuda.stream(stream):
            img = torch.empty(B, H, W, C, device=dev)
            dcol = torch.empty(B, N, C, device=dev)
            dpos = torch.empty(B, N, 2, device=dev)
        stream.synchronize()

        def step():
            return shards.step(pos, col, up, img, dcol, dpos, forward_only=fwd_only)

    # warm-up mirrors the timed loop (two caches kept alive) so the
    # stream-ordered memory pool reaches its steady state before timing
    warm = []
    for _ in range(args.warmup):
        warm.append(step())
        if len(warm) > 2:
            warm.pop(0)
    ctx.synchronize()

    # ---- device-resident timed region ----
    # Each timed step replays ONE captured CUDA graph of the whole step
    # (binning, gather, special pixels, backward and the cache's stream-
    # ordered allocations and frees): no host launch gaps between kernels.
    # Per-phase times come from an eager profiled pass (events cannot sit in
    # the graph); if capture is unavailable the steps run eagerly.
    def capture_step():
        ctx.set_profiling(True)
        ctx.phase_times(reset=True)
        for _ in range(args.warmup):
            c = step()
            del c
        ctx.synchronize()
        pm, pc = ctx.phase_times(reset=True)
        ctx.set_profiling(False)
        torch.cuda.synchronize(dev)
        n0 = ctx.launch_count
        gr = torch.cuda.CUDAGraph()
        # thread-local capture: CUDA calls from other threads (the NCCL
        # watchdog under torchrun, the clock sampler) are not disturbed
        with torch.cuda.graph(gr, stream=stream, capture_error_mode="thread_local"):
            c = step()
            del c
        n = ctx.launch_count - n0
        with torch.cuda.stream(stream):  # replay() launches on the current stream
            for _ in range(2):
                gr.replay()
        torch.cuda.synchronize(dev)
        return gr, n, pm, pc

    use_graph = args.graph == "on" or (args.graph == "auto" and not band)
    graph, graph_note = None, None
    if use_graph:
        warm.clear()
        try:
            graph, per_step_launches, phase_ms, phase_calls = capture_step()
        except Exception as exc:
            graph = None
            graph_note = f"graph capture failed ({type(exc).__name__}): eager steps"
            ctx.set_profiling(False)
            torch.cuda.synchronize(dev)
    if graph is None:
        ctx.set_profiling(True)
        ctx.phase_times(reset=True)
    group.barrier()
    torch.cuda.synchronize(dev)
    launches0 = ctx.launch_count
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    caches = warm
    with ClockSampler(local) as clocks:
        evs[0].record(stream)
        for k in range(args.steps):
            if graph is not None:
                with torch.cuda.stream(stream):  # replay() launches on the current stream
                    graph.replay()
            else:
                caches.append(step())
                if len(caches) > 2:
                    caches.pop(0)
            evs[k + 1].record(stream)
        torch.cuda.synchronize(dev)
    ms = evs[0].elapsed_time(evs[-1])
    per_step = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps))
    group.barrier()
    launches = (per_step_launches * args.steps if graph is not None
                else ctx.launch_count - launches0)
    ctx.synchronize()  # raises on any pending validation error
    if graph is None:
        phase_ms, phase_calls = ctx.phase_times(reset=True)
        ctx.set_profiling(False)
    caches.clear()
    ms = group.max_over_ranks(ms)
    med = group.max_over_ranks(per_step[len(per_step) // 2])
    ms_step = ms / args.steps
    # band mode: the job renders one full image per step (strong scaling)
    units = W * H_full if band else world * B * W * H
    value = units / (ms_step * 1e-3) / 1e6

    # ---- pair count P (exact, counting instantiation of the same kernel) ----
    with torch.cuda.stream(stream):
        img1 = torch.empty(1, H, W, C, device=dev)
    p1 = splitter.pos if band else pos[:1]
    c1 = splitter.col if band else col[:1]
    cache = ctx.forward_device(p1, c1, 1, N, C, W, H, sigma, cutoff, 0, img1)
    P_img = int(gmi.forward_counts(cache).astype(np.int64).sum())
    del cache

    # ---- rooflines: the binding pipe (FP32 for the C <= 4 configs), MUFU
    # and HBM beside it; per launch of the dominant kernel and per step ----
    hbm_peak, sm_mhz, peak_kind = peaks()
    fp32_peak, mufu_peak = pipe_peaks(sm_mhz)
    per_call = {name: phase_ms[k] / max(1, phase_calls[k]) for k, name in enumerate(gmi.Context.PHASES)}
    dom = "gather" if fwd_only else max(("gather", "points_bwd"), key=lambda k: per_call[k])
    Bk = 1 if band else B
    pts_bytes = 4 * N * (2 + C)
    img_bytes = 4 * H * W * C
    alg_bytes = {"gather": Bk * (pts_bytes + img_bytes),            # points in, image out
                 "points_bwd": Bk * (2 * pts_bytes + img_bytes)}   # points in, grads out, upstream in
    alg_fp32 = {"gather": Bk * P_img * (6 + C), "points_bwd": Bk * P_img * (11 + 2 * C)}
    alg_mufu = {"gather": Bk * (P_img + H * W), "points_bwd": Bk * (P_img + H * W)}
    t_dom = per_call[dom] * 1e-3
    step_fp32 = Bk * P_img * ((6 + C) if fwd_only else (17 + 3 * C))
    step_mufu = Bk * ((P_img + H * W) if fwd_only else 2 * (P_img + H * W))
    step_bytes = Bk * ((pts_bytes + img_bytes + 12 * N) if fwd_only
                       else (3 * pts_bytes + 2 * img_bytes + 12 * N))
    t_roof = {"fp32": step_fp32 / fp32_peak, "mufu": step_mufu / mufu_peak,
              "hbm": step_bytes / (hbm_peak * 1e9)}
    binding = max(t_roof, key=t_roof.get)
    t_step = ms_step * 1e-3

    def roof(kind):
        if kind == "fp32":
            a, pk, unit = alg_fp32[dom] / t_dom / 1e12, fp32_peak / 1e12, "T FP32-instr/s"
            counts = "fwd 6+C, bwd 11+2C FP32 instr per (pixel, point) pair (SURVEY §8d)"
        elif kind == "mufu":
            a, pk, unit = alg_mufu[dom] / t_dom / 1e12, mufu_peak / 1e12, "T MUFU-op/s"
            counts = "1 ex2 per pair + 1 rcp per pixel per pass (SURVEY §8d)"
        else:
            a, pk, unit = alg_bytes[dom] / t_dom / 1e9, hbm_peak, "GB/s"
            counts = "4[N(2+C)+HWC] fwd, 4[2N(2+C)+HWC] bwd per image (SURVEY §8d)"
        return {"bound": {"fp32": "fp32_pipe", "mufu": "mufu_pipe", "hbm": "hbm"}[kind],
                "kernel": dom, "achieved": round(a, 3), "peak": round(pk, 2), "unit": unit,
                "frac": round(a / pk, 4), "step_frac": round(t_roof[kind] / t_step, 4),
                "step_roof_ms": round(t_roof[kind] * 1e3, 4), "counts": counts,
                "peak_kind": peak_kind if kind == "hbm" else "nominal (148 SMs x lanes x sm_max_mhz)"}

    roofline = roof(binding)
    roofline["traffic"] = traffic_of(dom, args.config, B)
    roofline["note"] = ("binding roof = max(FP32, MUFU, HBM) of the step's algorithmic counts; "
                        "frac = the dominant kernel per launch, step_frac = the whole step")
    others = {f"roofline_{k}": roof(k) for k in ("fp32", "mufu", "hbm") if k != binding}

    # forward_host uploads positions+colours and downloads the image;
    # backward_host uploads upstream and downloads both gradients
    h2d = B * N * 4 * (2 + C) + (0 if fwd_only else B * H * W * C * 4)
    d2h = B * H * W * C * 4 + (0 if fwd_only else B * N * 4 * (C + 2))
    e2e_ms = e2e_np_ms = None
    if args.e2e_steps > 0 and not band:
        pinned = [pos.cpu().pin_memory(), col.cpu().pin_memory(), up.cpu().pin_memory(),
                  torch.empty(B, H, W, C).pin_memory(), torch.empty(B, N, C).pin_memory(),
                  torch.empty(B, N, 2).pin_memory()]
        hpos, hcol, hup, himg, hdc, hdp = (t.numpy() for t in pinned)
        import ctypes as Cty
        fp = Cty.POINTER(Cty.c_float)
        cfg_c = gmi._lib.GmiConfig(sigma, cutoff, 0, W, H)

        def e2e_step():
            h = Cty.c_void_p()
            gmi._check(gmi.lib.gmi_forward_host(ctx.handle, hpos.ctypes.data_as(fp), hcol.ctypes.data_as(fp),
                                                B, N, C, Cty.byref(cfg_c), himg.ctypes.data_as(fp), Cty.byref(h)))
            if not fwd_only:
                gmi._check(gmi.lib.gmi_backward_host(ctx.handle, hpos.ctypes.data_as(fp),
                                                     hcol.ctypes.data_as(fp), B, N, C, Cty.byref(cfg_c), h,
                                                     hup.ctypes.data_as(fp), hdc.ctypes.data_as(fp),
                                                     hdp.ctypes.data_as(fp)))
            gmi.lib.gmi_cache_free(h)
            # a user's step ends when its host outputs are complete (the
            # asynchronous calls overlap the backward's upload with the
            # forward's download inside the step)
            ctx.synchronize()

        def timed(fn, n):
            for _ in range(max(2, args.warmup)):  # grows the memory pool
                fn()
            group.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            return group.max_over_ranks(e0.elapsed_time(e1) / n)

        e2e_ms = timed(e2e_step, args.e2e_steps)
        e2e_value = world * B * W * H / (e2e_ms * 1e-3) / 1e6
        pcie = pcie_duplex_gbps(dev)

        # the reference-shaped numpy shim (forward_batch / backward_batch) on
        # plain pageable numpy arrays, as a user of gmi._core would call it
        npos, ncol, nup = (np.array(t) for t in (hpos, hcol, hup))

        def e2e_numpy_step():
            im, cc = gmi.forward_batch(npos, ncol, W, H, sigma, cutoff, ctx=ctx)
            if not fwd_only:
                gmi.backward_batch(npos, ncol, cc, nup, sigma, cutoff, ctx=ctx)
            ctx.synchronize()
            cc.close()

        e2e_np_ms = timed(e2e_numpy_step, max(1, min(args.e2e_steps, 2)))

    if rank != 0:
        group.close()
        return
    line = {
        "metric": METRIC if args.config == 3 else METRIC.replace("1024^2, N=262k pts, C=3", cfg["workload"]),
        "value": round(value, 2), "unit": "Mpix/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "ms_per_step_median": round(med, 4), "ms_per_step_min": round(per_step[0], 4),
        "higher_is_better": True, "scaling": "strong" if band else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "batch_per_gpu": B, "global_batch": B if band else world * B,
                   "points": N, "channels": C, "frame": [H, W], "sigma": sigma,
                   "cutoff": cutoff, "pairs_per_image": P_img,
                   "l2": "inputs > L2 (126 MB): no flush needed",
                   "parallelism": (f"row bands x{world} (rows {H} + halo {splitter.plan.halo:g} per rank), "
                                   f"NCCL SUM of {int(splitter.plan.shared.size)} shared points' gradients per step")
                                  if band else f"batch-sharded x{world}, no collective"},
        "phases_ms_per_step": {k: round(v, 4) for k, v in per_call.items()},
        "roofline": roofline,
        **others,
        "e2e": ({"value": round(e2e_value, 2), "unit": "Mpix/s", "h2d_bytes_per_step": h2d,
                 "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
                 "api": "gmi_forward_host / gmi_backward_host, pinned host buffers",
                 # the e2e bound: both directions' bytes at the measured
                 # pinned full-duplex PCIe rate of this box
                 "roofline": {"bound": "pcie_duplex", "peak_GBps_each_way": round(pcie, 1),
                              "bound_ms": round(max(h2d, d2h) / (pcie * 1e9) * 1e3, 3),
                              "frac": round(max(h2d, d2h) / (pcie * 1e9) * 1e3 / e2e_ms, 4)},
                 "numpy_shim": {"value": round(world * B * W * H / (e2e_np_ms * 1e-3) / 1e6, 2),
                                "ms_per_step": round(e2e_np_ms, 3),
                                "api": "forward_batch / backward_batch on pageable numpy arrays"}}
                if e2e_ms else None),
        "gpu_launches": launches,
        "cuda_graph": graph is not None if graph_note is None else graph_note,
        "clocks": clocks.summary(),
    }
    if not args.no_cpu_baseline and args.config == 3:
        v, imgs, threads, secs, kind = cpu_reference_sample(cfg, args.cpu_seconds, 64)
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "Mpix/s", "cores": threads,
                                "kind": kind,
                                "sample": f"{imgs} image(s) of the workload, fwd+bwd, {secs:.1f} s"}
    print(json.dumps(line), flush=True)
    group.close()


if __name__ == "__main__":
    main()
