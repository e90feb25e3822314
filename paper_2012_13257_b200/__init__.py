"""B200-native Gaussian-mixture interpolation (arXiv 2012.13257) — Python shim.

A thin numpy/ctypes layer over ``libgmi_b200.so`` that keeps the reference's
Python surface (``gmi._core``, /root/reference/proj/python/bindings.cpp:120-184
and python/gmi/__init__.py:7-28) for the hot path:

    PointSet(positions, colors)            bindings.cpp:127-131
    ForwardCache.fallback_count/width/height  bindings.cpp:133-139
    GmiError                               bindings.cpp:123
    gaussian_weight(qx, qy, mux, muy, sigma)  bindings.cpp:141-145
    forward(points, width, height, sigma, radius=0.0, fallback="nearest",
            workers=1) -> (image HxWxC, cache)        bindings.cpp:147-160
    backward(points, cache, upstream, sigma, radius=0.0, fallback="nearest",
             workers=1) -> (d_colors NxC, d_positions Nx2)  bindings.cpp:162-184

plus the batch and device-resident entry points of the B200 path
(``forward_batch`` / ``backward_batch`` on host arrays, ``Context`` for device
pointers given as ``__cuda_array_interface__`` objects or raw addresses) and
the bit-exact ``bin_grid`` export.  No PyTorch dependency; the compute runs
only on the GPU — there is no CPU fallback.

Numerics: the device path stores fp32 (the reference is f64); arrays passed
in are converted to float32, so results match the reference bit-exactly for
binning / neighbour sets / fallback choices and within rel 1e-5 / abs 1e-6 for
image and gradients whenever the inputs are fp32-representable.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import warnings

import numpy as np

from . import _lib
from ._lib import GmiConfig, lib

__all__ = [
    "ForwardCache", "GmiError", "PointSet", "backward", "forward", "gaussian_weight",
    "forward_batch", "backward_batch", "Context", "bin_grid", "forward_counts",
    "default_context", "optimize_points", "gmm_benchmark", "ERROR_NAMES", "__version__",
    "load_point_set", "save_point_set", "load_image", "save_image",
    "DeviceArray", "forward_cuda", "backward_cuda", "CTX_ASYNC_ERRORS", "CTX_PRECISE",
    "CTX_INJECT_FAULT", "PrecisionWarning", "set_fp32_inputs",
]

__version__ = "0.2.0"

# context flags (include/gmi_b200.h)
CTX_ASYNC_ERRORS = 1   # errors reported by Context.synchronize()
CTX_PRECISE = 4        # f64 weights, sums and image (reference-grade precision)
CTX_INJECT_FAULT = 8   # test hook: the backward corrupts d_colors[0] (harness check)

# gmi::ErrorCode names (core.hpp:35-50), index = code - 1
ERROR_NAMES = ["NonFiniteValue", "ColorOutOfRange", "EmptyPointSet", "ShapeMismatch",
               "InvalidCellSize", "ConfigInvalid", "CacheMismatch", "InvalidDimensions",
               "InvalidFactor", "InvalidCount", "UnsupportedFormat", "CorruptFile", "EmptyLog",
               "IoError"]


class GmiError(RuntimeError):
    """gmi::Error (core.hpp:54-62) as raised by the reference binding."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.name = lib.gmi_error_name(code).decode()


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.gmi_last_error().decode()
        if rc in (101,):
            raise ValueError(msg)
        raise GmiError(rc, msg)


class PrecisionWarning(UserWarning):
    """Inputs rounded to the device path's fp32 (see set_fp32_inputs)."""


_fp32_policy = "allow"


def set_fp32_inputs(policy: str) -> None:
    """What PointSet does with positions / colours fp32 cannot hold exactly
    (the device computes in fp32; the reference in f64): "allow" (default:
    round, count in PointSet.inexact_inputs), "warn" (PrecisionWarning) or
    "reject" (GmiError) — the C++ API's gmi::set_fp32_inputs."""
    global _fp32_policy
    if policy not in ("allow", "warn", "reject"):
        raise ValueError("policy must be 'allow', 'warn' or 'reject'")
    _fp32_policy = policy


# ---------------------------------------------------------------------------
class PointSet:
    """N known points: positions Nx2 and colours NxC (core.hpp:64-79).

    Validates like ``require_valid`` (core.cpp:55-96, C >= 1 instead of
    C in {1,3}) at construction, exactly as the reference binding's
    constructor does (bindings.cpp:57-76)."""

    def __init__(self, positions, colors):
        positions = np.asarray(positions, dtype=np.float64)
        colors = np.asarray(colors, dtype=np.float64)
        if positions.ndim != 2 or positions.shape[1] != 2:
            raise ValueError("positions must be Nx2")
        if colors.ndim != 2 or colors.shape[0] != positions.shape[0]:
            raise ValueError("colors must be NxC with matching N")
        n, ch = colors.shape
        if n == 0:
            raise GmiError(3, "point set is empty")
        if ch < 1:
            raise GmiError(4, f"channels must be >= 1, got {ch}")
        bad_pos = ~np.isfinite(positions).all(axis=1)
        bad_nonfinite = ~np.isfinite(colors)
        bad_range = (colors < 0.0) | (colors > 1.0)
        issue = None
        for i in np.nonzero(bad_pos | bad_nonfinite.any(axis=1) | bad_range.any(axis=1))[0][:1]:
            if bad_pos[i]:
                issue = (1, f"non-finite position at index {i}")
            else:
                for c in range(ch):
                    if bad_nonfinite[i, c]:
                        issue = (1, f"non-finite color at index {i}")
                        break
                    if bad_range[i, c]:
                        issue = (2, f"color {colors[i, c]} out of [0,1] at index {i}")
                        break
        if issue:
            raise GmiError(*issue)
        self._pos32 = np.ascontiguousarray(positions, dtype=np.float32)
        self._col32 = np.ascontiguousarray(colors, dtype=np.float32)
        # values the fp32 device path rounds (the reference keeps them in f64)
        self.inexact_inputs = int(np.count_nonzero(self._pos32.astype(np.float64) != positions) +
                                  np.count_nonzero(self._col32.astype(np.float64) != colors))
        if self.inexact_inputs and _fp32_policy != "allow":
            msg = (f"{self.inexact_inputs} position / colour value(s) are not representable in "
                   f"fp32 and are rounded for the device path")
            if _fp32_policy == "reject":
                raise GmiError(101, msg)
            warnings.warn(msg, PrecisionWarning, stacklevel=2)

    @property
    def positions(self) -> np.ndarray:
        return self._pos32.astype(np.float64)

    @property
    def colors(self) -> np.ndarray:
        return self._col32.astype(np.float64)

    @property
    def channels(self) -> int:
        return int(self._col32.shape[1])

    def __len__(self) -> int:
        return int(self._pos32.shape[0])


# ---------------------------------------------------------------------------
class Context:
    """One device + one CUDA stream (gmi_ctx)."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = int(os.environ.get("GMI_DEVICE", "0"))
        h = C.c_void_p()
        _check(lib.gmi_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib.gmi_ctx_stream(self._h) or 0

    def set_stream(self, stream_ptr: int | None) -> None:
        _check(lib.gmi_ctx_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    def set_flags(self, flags: int) -> None:
        _check(lib.gmi_ctx_set_flags(self._h, flags))

    def synchronize(self) -> None:
        _check(lib.gmi_ctx_synchronize(self._h))

    def join_host_copies(self) -> None:
        """The ctx stream waits (device-side) for queued host-buffer copies."""
        _check(lib.gmi_ctx_join_host_copies(self._h))

    @property
    def launch_count(self) -> int:
        return int(lib.gmi_ctx_launch_count(self._h))

    PHASES = ("bin", "gather", "special_fwd", "points_bwd", "special_bwd")

    def set_profiling(self, on: bool) -> None:
        _check(lib.gmi_ctx_set_profiling(self._h, 1 if on else 0))

    def phase_times(self, reset: bool = True):
        """(ms[5], calls[5]) per phase accumulated from CUDA events on the ctx
        stream (see gmi_ctx_phase_times)."""
        ms = (C.c_double * 5)()
        calls = (C.c_uint64 * 5)()
        _check(lib.gmi_ctx_phase_times(self._h, ms, calls, 1 if reset else 0))
        return np.array(ms[:]), np.array(calls[:], dtype=np.int64)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.gmi_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- device-resident entry points (pointers) ----
    def forward_device(self, positions, colors, batch, num_points, channels, width, height,
                       sigma, cutoff, fallback, image) -> "ForwardCache":
        """gmi_forward on device memory.  Arguments are device addresses (int)
        or objects exposing ``__cuda_array_interface__``."""
        cfg = _config(sigma, cutoff, fallback, width, height)
        h = C.c_void_p()
        _check(lib.gmi_forward(self._h, _addr(positions), _addr(colors), batch, num_points,
                               channels, C.byref(cfg), _addr(image), C.byref(h)))
        return ForwardCache(h, self, keep=(positions, colors, image))

    def backward_device(self, positions, colors, batch, num_points, channels, width, height,
                        sigma, cutoff, fallback, cache: "ForwardCache", upstream, d_colors,
                        d_positions) -> None:
        cfg = _config(sigma, cutoff, fallback, width, height)
        _check(lib.gmi_backward(self._h, _addr(positions), _addr(colors), batch, num_points,
                                channels, C.byref(cfg), cache.handle, _addr(upstream),
                                _addr(d_colors), _addr(d_positions)))


_default_ctx = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default_ctx
    with _default_lock:
        if _default_ctx is None:
            _default_ctx = Context()
        return _default_ctx


def _addr(x) -> C.c_void_p:
    if x is None:
        return C.c_void_p(0)
    if isinstance(x, int):
        return C.c_void_p(x)
    cai = getattr(x, "__cuda_array_interface__", None)
    if cai is None:
        raise TypeError("expected a device address or an object with __cuda_array_interface__")
    return C.c_void_p(cai["data"][0])


def _fallback_code(fallback: str) -> int:
    # make_interp_config (bindings.cpp:95-108)
    if fallback == "nearest":
        return 0
    if fallback == "zero":
        return 1
    raise ValueError("fallback must be 'nearest' or 'zero'")


def _config(sigma, cutoff, fallback, width, height) -> GmiConfig:
    fb = _fallback_code(fallback) if isinstance(fallback, str) else int(fallback)
    return GmiConfig(float(sigma), float(cutoff), fb, int(width), int(height))


def _interp_config(sigma, radius, fallback, width, height) -> GmiConfig:
    # make_config: cutoff = 3 sigma unless radius > 0 (bindings.cpp:95-101)
    cutoff = float(radius) if radius > 0.0 else lib.gmi_default_cutoff(float(sigma))
    return _config(sigma, cutoff, fallback, width, height)


class ForwardCache:
    """ForwardCache handle (engine.hpp:20-41); frees the device state on GC."""

    def __init__(self, handle, ctx: Context, keep=()):
        self._h = handle
        self._ctx = ctx
        self._keep = keep  # device buffers the cache borrows (gmi_forward)
        b, n, ch, w, hgt = (C.c_int32() for _ in range(5))
        _check(lib.gmi_cache_shape(handle, C.byref(b), C.byref(n), C.byref(ch), C.byref(w),
                                   C.byref(hgt)))
        self.batch, self.num_points, self.channels = b.value, n.value, ch.value
        self.width, self.height = w.value, hgt.value

    @property
    def handle(self):
        return self._h

    @property
    def fallback_counts(self) -> np.ndarray:
        out = np.zeros(self.batch, np.int64)
        _check(lib.gmi_cache_fallback_count(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    @property
    def fallback_count(self) -> int:
        """ForwardCache::fallback_count (engine.cpp:27-33); summed over the batch."""
        return int(self.fallback_counts.sum())

    def pixels(self):
        """Host copies of (normalizer, fallback_flag, nearest_index), each BxHxW."""
        shape = (self.batch, self.height, self.width)
        norm = np.zeros(shape, np.float32)
        flag = np.zeros(shape, np.uint8)
        near = np.zeros(shape, np.int32)
        _check(lib.gmi_cache_copy_pixels(self._h, norm.ctypes.data_as(C.POINTER(C.c_float)),
                                         flag.ctypes.data_as(C.POINTER(C.c_uint8)),
                                         near.ctypes.data_as(C.POINTER(C.c_int32))))
        return norm, flag, near

    def close(self):
        if getattr(self, "_h", None):
            lib.gmi_cache_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
def gaussian_weight(qx, qy, mux, muy, sigma) -> float:
    """gaussian_weight (core.cpp:49-53)."""
    return float(lib.gmi_gaussian_weight(qx, qy, mux, muy, sigma))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def forward_batch(positions, colors, width, height, sigma, radius=0.0, fallback="nearest",
                  ctx: Context | None = None):
    """Batched forward on HOST arrays: positions BxNx2, colors BxNxC ->
    (image BxHxWxC float32, ForwardCache)."""
    ctx = ctx or default_context()
    pos = _f32(positions)
    col = _f32(colors)
    if pos.ndim != 3 or pos.shape[2] != 2:
        raise ValueError("positions must be BxNx2")
    if col.ndim != 3 or col.shape[:2] != pos.shape[:2]:
        raise ValueError("colors must be BxNxC with matching B, N")
    b, n, ch = col.shape
    cfg = _interp_config(sigma, radius, fallback, width, height)
    image = np.zeros((b, height, width, ch), np.float32)
    h = C.c_void_p()
    _check(lib.gmi_forward_host(ctx.handle, pos.ctypes.data_as(C.POINTER(C.c_float)),
                                col.ctypes.data_as(C.POINTER(C.c_float)), b, n, ch,
                                C.byref(cfg), image.ctypes.data_as(C.POINTER(C.c_float)),
                                C.byref(h)))
    return image, ForwardCache(h, ctx)


def backward_batch(positions, colors, cache: ForwardCache, upstream, sigma, radius=0.0,
                   fallback="nearest", ctx: Context | None = None):
    """Batched backward on HOST arrays -> (d_colors BxNxC, d_positions BxNx2) float32."""
    ctx = ctx or cache._ctx
    pos = _f32(positions)
    col = _f32(colors)
    up = _f32(upstream)
    b, n, ch = col.shape
    if up.shape != (b, cache.height, cache.width, ch):
        raise ValueError("upstream must be BxHxWxC matching the forward output")
    cfg = _interp_config(sigma, radius, fallback, cache.width, cache.height)
    dc = np.zeros((b, n, ch), np.float32)
    dp = np.zeros((b, n, 2), np.float32)
    fp = C.POINTER(C.c_float)
    _check(lib.gmi_backward_host(ctx.handle, pos.ctypes.data_as(fp), col.ctypes.data_as(fp), b,
                                 n, ch, C.byref(cfg), cache.handle, up.ctypes.data_as(fp),
                                 dc.ctypes.data_as(fp), dp.ctypes.data_as(fp)))
    return dc, dp


def forward(points: PointSet, width: int, height: int, sigma: float, radius: float = 0.0,
            fallback: str = "nearest", workers: int = 1):
    """gmi._core.forward (bindings.cpp:147-160) -> (image HxWxC float64, cache).
    ``workers`` is accepted for source compatibility (the reference output is
    worker-independent, engine.hpp:3-5)."""
    if not isinstance(points, PointSet):
        raise TypeError("points must be a PointSet")
    image, cache = forward_batch(points._pos32[None], points._col32[None], width, height, sigma,
                                 radius, fallback)
    return image[0].astype(np.float64), cache


def _upstream_array(upstream) -> np.ndarray:
    # image_from_array (bindings.cpp:27-48): HxW or HxWxC
    up = np.asarray(upstream, dtype=np.float64)
    if up.ndim == 2:
        up = up[:, :, None]
    if up.ndim != 3:
        raise ValueError("image array must be HxW or HxWxC")
    return up


def backward(points: PointSet, cache: ForwardCache, upstream, sigma: float, radius: float = 0.0,
             fallback: str = "nearest", workers: int = 1):
    """gmi._core.backward (bindings.cpp:162-184) -> (d_colors NxC, d_positions Nx2)."""
    if not isinstance(points, PointSet):
        raise TypeError("points must be a PointSet")
    up = _upstream_array(upstream)
    if up.shape != (cache.height, cache.width, points.channels) or cache.batch != 1:
        raise GmiError(7, "forward cache does not match the given inputs")
    dc, dp = backward_batch(points._pos32[None], points._col32[None], cache, up[None], sigma,
                            radius, fallback)
    return dc[0].astype(np.float64), dp[0].astype(np.float64)


def optimize_points(points: PointSet, target, sigma: float, radius: float = 0.0,
                    steps: int = 100, learning_rate: float = 0.5,
                    optimize_positions: bool = True, optimize_colors: bool = False,
                    log_every: int = 10, workers: int = 1, ctx: Context | None = None,
                    log_trajectory: bool = True) -> dict:
    """gmi._core.optimize_points (bindings.cpp:282-322, optimize.cpp:47-98) on
    the GPU: render -> L1 loss -> backward -> descent, `steps` times, the bin
    grid rebuilt on the device in every render.  Returns the reference's dict:
    points, loss_curve (steps + 1), trajectory [(step, i, x, y, loss)] at step
    0, every log_every and the last step, mean/max displacement."""
    if not isinstance(points, PointSet):
        raise TypeError("points must be a PointSet")
    if log_every < 1:
        raise GmiError(6, "log_every must be >= 1")
    ctx = ctx or default_context()
    tgt = _upstream_array(target).astype(np.float32)
    h, w = tgt.shape[:2]
    if tgt.shape[2] != points.channels:
        raise GmiError(4, "target channels do not match the point set")
    cfg = _interp_config(sigma, radius, "nearest", w, h)
    pos = points._pos32.copy()
    col = points._col32.copy()
    n, ch = col.shape
    flags = (1 if optimize_positions else 0) | (2 if optimize_colors else 0)
    fp = C.POINTER(C.c_float)
    loss_curve, trajectory = [], []

    def log(step, loss):
        if not log_trajectory:
            return
        for i in range(n):
            trajectory.append((step, i, float(pos[i, 0]), float(pos[i, 1]), float(loss)))

    # segments of log_every steps: the trajectory needs the positions at the
    # logged steps; each segment's first loss is the previous segment's last
    pos0 = pos.copy()
    done = 0
    while done < steps:
        seg = min(log_every - done % log_every, steps - done)
        lc = np.zeros(seg + 1, np.float64)
        _check(lib.gmi_optimize_points_host(ctx.handle, pos.ctypes.data_as(fp), col.ctypes.data_as(fp),
                                            1, n, ch, C.byref(cfg), tgt.ctypes.data_as(fp), seg,
                                            float(learning_rate), flags,
                                            lc.ctypes.data_as(C.POINTER(C.c_double))))
        if done == 0:
            loss_curve.append(lc[0])
            if log_trajectory:
                trajectory.extend((0, i, float(pos0[i, 0]), float(pos0[i, 1]), float(lc[0]))
                                  for i in range(n))
        loss_curve.extend(lc[1:].tolist())
        done += seg
        log(done, lc[-1])
    pts = PointSet(pos.astype(np.float64), col.astype(np.float64))
    d = np.hypot(*(pos.astype(np.float64) - pos0.astype(np.float64)).T)
    return {"points": pts, "loss_curve": np.asarray(loss_curve), "trajectory": trajectory,
            "mean_displacement": float(d.mean()) if n else 0.0,
            "max_displacement": float(d.max()) if n else 0.0}


def gmm_benchmark(image, factor: int, sigma: float | None = None, lowres=None,
                  ctx: Context | None = None) -> dict:
    """The "gmm" row of run_benchmark (benchmark.cpp:88-107) for one image and
    one factor, on the GPU: known points at the block centres of `lowres`
    (default: the block means of `image`, block_mean_downsample), one forward
    per sigma (default: the auto sweep {0.4, 0.5, 0.6} x factor), L1 against
    `image`.  Returns the BenchmarkRow fields (factor, method, sigma_used, l1,
    wall_time_ms = device time of that forward) plus the whole sweep and the
    chosen reconstruction."""
    ctx = ctx or default_context()
    img = np.ascontiguousarray(np.asarray(image, np.float32))
    if img.ndim == 2:
        img = img[:, :, None]
    h, w, ch = img.shape
    sig = None if sigma is None else np.array([float(sigma)], np.float64)
    n = 3 if sig is None else 1
    low = None
    if lowres is not None:
        low = np.ascontiguousarray(np.asarray(lowres, np.float32))
        if low.ndim == 2:
            low = low[:, :, None]
        if low.shape != ((h + factor - 1) // factor, (w + factor - 1) // factor, ch):
            raise GmiError(4, "lowres must be ceil(H/factor) x ceil(W/factor) x C")
    l1 = np.zeros(n)
    ms = np.zeros(n)
    best = C.c_int32()
    out = np.empty_like(img)
    fp = C.POINTER(C.c_float)
    dp = C.POINTER(C.c_double)
    _check(lib.gmi_gmm_benchmark_host(ctx.handle, img.ctypes.data_as(fp), w, h, ch, int(factor),
                                      low.ctypes.data_as(fp) if low is not None else None,
                                      sig.ctypes.data_as(dp) if sig is not None else None, n,
                                      l1.ctypes.data_as(dp), ms.ctypes.data_as(dp), C.byref(best),
                                      out.ctypes.data_as(fp)))
    sigmas = [0.4 * factor, 0.5 * factor, 0.6 * factor] if sig is None else [float(sigma)]
    b = best.value
    return {"factor": int(factor), "method": "gmm", "sigma_used": sigmas[b], "l1": float(l1[b]),
            "wall_time_ms": float(ms[b]), "sigmas": sigmas, "l1_per_sigma": l1.tolist(),
            "ms_per_sigma": ms.tolist(), "image": out}


def forward_counts(cache: ForwardCache) -> np.ndarray:
    """Per-pixel contribution counts (pixel_start deltas, engine.hpp:29-31) from
    the counting instantiation of the same gather kernel; BxHxW int32."""
    out = np.zeros((cache.batch, cache.height, cache.width), np.int32)
    _check(lib.gmi_forward_counts(cache._ctx.handle, cache.handle,
                                  out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def bin_grid(positions, cell_size: float, ctx: Context | None = None):
    """build_bin_grid (bin_grid.cpp:38-82) on the GPU, bit-exact.  positions
    Nx2 (or BxNx2) host array; returns a dict (or list of dicts) with origin,
    n_cols, n_rows, bin_start, point_index like the reference BinGrid."""
    ctx = ctx or default_context()
    pos = _f32(positions)
    single = pos.ndim == 2
    if single:
        pos = pos[None]
    b, n, _ = pos.shape
    if n == 0:
        raise GmiError(3, "point set is empty")
    fp = C.POINTER(C.c_float)
    origin = np.zeros((b, 2))
    ncol = np.zeros(b, np.int32)
    nrow = np.zeros(b, np.int32)
    ip = C.POINTER(C.c_int32)
    _check(lib.gmi_bin_grid_host(ctx.handle, pos.ctypes.data_as(fp), b, n, float(cell_size),
                                 origin.ctypes.data_as(C.POINTER(C.c_double)),
                                 ncol.ctypes.data_as(ip), nrow.ctypes.data_as(ip), None, None))
    total = int(sum(int(ncol[k]) * int(nrow[k]) + 1 for k in range(b)))
    bin_start = np.zeros(total, np.int32)
    point_index = np.zeros((b, n), np.int32)
    _check(lib.gmi_bin_grid_host(ctx.handle, pos.ctypes.data_as(fp), b, n, float(cell_size),
                                 origin.ctypes.data_as(C.POINTER(C.c_double)),
                                 ncol.ctypes.data_as(ip), nrow.ctypes.data_as(ip),
                                 bin_start.ctypes.data_as(ip), point_index.ctypes.data_as(ip)))
    out, off = [], 0
    for k in range(b):
        nb = int(ncol[k]) * int(nrow[k]) + 1
        out.append(dict(origin=origin[k], n_cols=int(ncol[k]), n_rows=int(nrow[k]),
                        bin_start=bin_start[off:off + nb], point_index=point_index[k]))
        off += nb
    return out[0] if single else out


from .formats import load_image, load_point_set, save_image, save_point_set  # noqa: E402
from .device import DeviceArray, backward_cuda, forward_cuda  # noqa: E402
