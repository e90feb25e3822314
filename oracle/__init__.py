"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the hot path.

Nothing in ``paper_2012_13257_b200/`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may load it, and only as the checker or the timed CPU
baseline — never as the thing measured or shipped.

Two CPU implementations sit behind one numpy API:

* ``Reference`` — the UNMODIFIED reference C++ (``/root/reference/proj``)
  compiled from its own sources into ``oracle/_ref/libgmi_ref.so`` by
  ``oracle/Makefile`` and called through ``oracle/ref_capi.cpp``.  Forwards to
  ``gmi::forward`` (engine.cpp:107-176), ``gmi::backward`` (engine.cpp:238-309),
  ``gmi::build_bin_grid`` (bin_grid.cpp:38-82) and friends.  Channels are
  restricted to {1,3} exactly as the reference restricts them
  (core.cpp:60-64); ``Reference.forward_any_c`` decomposes wider inputs into
  C=3/C=1 channel groups.
* ``Oracle`` — ``oracle/gmi_oracle.c``, a plain-C restatement that follows the
  reference statement by statement (bit-identical for C in {1,3}, pinned by
  tests/test_oracle.py against ``Reference`` and ``tests/golden/``) and accepts
  any C >= 1.

Error codes: 0 ok, else 1 + ``gmi::ErrorCode`` (core.hpp:35-50).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgmi_ref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_fp = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)

ERROR_NAMES = [
    "NonFiniteValue", "ColorOutOfRange", "EmptyPointSet", "ShapeMismatch",
    "InvalidCellSize", "ConfigInvalid", "CacheMismatch", "InvalidDimensions",
    "InvalidFactor", "InvalidCount", "UnsupportedFormat", "CorruptFile",
    "EmptyLog", "IoError",
]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        name = ERROR_NAMES[code - 1] if 0 < code <= len(ERROR_NAMES) else str(code)
        self.name = name
        super().__init__(f"{name}: {msg}")


def build(with_reference: bool | None = None) -> None:
    """Compile the checkers (gcc/g++ only).  The reference is compiled only
    when its sources are present (this container, not the GPU box)."""
    if with_reference is None:
        with_reference = os.path.isdir("/root/reference/proj/src")
    targets = ["liboracle.so"] + (["ref", "dropin"] if with_reference else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def oracle_available() -> bool:
    return os.path.exists(ORC_SO)


class Reference:
    """ctypes facade over oracle/_ref/libgmi_ref.so (the reference itself)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gaussian_weight.restype = C.c_double
        L.ref_gaussian_weight.argtypes = [C.c_double] * 5
        L.ref_bin_grid_new.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_bin_grid_info.argtypes = [C.c_void_p, _dp, _ip, _ip]
        L.ref_bin_grid_copy.argtypes = [C.c_void_p, _ip, _ip]
        L.ref_bin_grid_free.argtypes = [C.c_void_p]
        L.ref_query_radius.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, _ip, _ip]
        L.ref_nearest_point.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, _dp, C.c_int, _ip]
        L.ref_forward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp, C.POINTER(C.c_void_p)]
        L.ref_cache_info.argtypes = [C.c_void_p, _i64p, _ip]
        L.ref_cache_copy.argtypes = [C.c_void_p, _i64p, _ip, _dp, _dp, _u8p, _ip]
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_backward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_void_p, _dp, C.c_double, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_oracle_forward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        L.ref_oracle_gradients_fd.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.c_double, _dp, _dp]
        L.ref_random_instance.argtypes = [C.c_uint64, C.c_int, C.c_int, _ip, _ip, _ip, _ip, _dp, _dp, _dp]
        L.ref_rng_u64.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.ref_optimize_points.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                          C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                          C.c_int, C.c_int, _dp, _dp, _dp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def run_benchmark_gmm(self, image, factor, sigma=None, box=True):
        """gmi::run_benchmark (benchmark.cpp:53-120), method "gmm", one image,
        one factor -> (l1, sigma_used, wall_time_ms)."""
        img = np.ascontiguousarray(image, np.float64)
        h, w, ch = img.shape
        L = self.lib
        L.ref_run_benchmark_gmm.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_int, _dp, _dp, _dp]
        l1, su, ms = C.c_double(), C.c_double(), C.c_double()
        self._check(L.ref_run_benchmark_gmm(_ptr(img, _dp), w, h, ch, factor,
                                            0.0 if sigma is None else float(sigma), int(box),
                                            C.byref(l1), C.byref(su), C.byref(ms)))
        return l1.value, su.value, ms.value

    # ---- files (imaging.cpp:235-304, 433-494) ----
    def save_point_set(self, pos, col, path):
        pos, col = _d(pos), _d(col)
        L = self.lib
        L.ref_save_point_set.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_char_p]
        self._check(L.ref_save_point_set(_ptr(pos, _dp), _ptr(col, _dp), col.shape[0], col.shape[1],
                                         path.encode()))

    def load_point_set(self, path, cap=1 << 20):
        L = self.lib
        L.ref_load_point_set.argtypes = [C.c_char_p, C.c_int, _ip, _ip, _dp, _dp]
        n, ch = C.c_int(), C.c_int()
        pos = np.zeros((cap, 2))
        col = np.zeros(cap * 3)
        self._check(L.ref_load_point_set(path.encode(), cap, C.byref(n), C.byref(ch), _ptr(pos, _dp),
                                         _ptr(col, _dp)))
        return pos[:n.value].copy(), col[:n.value * ch.value].reshape(n.value, ch.value).copy()

    def save_image(self, img, path):
        img = _d(img)
        if img.ndim == 2:
            img = img[:, :, None]
        L = self.lib
        L.ref_save_image.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_char_p]
        self._check(L.ref_save_image(_ptr(img, _dp), img.shape[0], img.shape[1], img.shape[2],
                                     path.encode()))

    def load_image(self, path, cap=1 << 24):
        L = self.lib
        L.ref_load_image.argtypes = [C.c_char_p, C.c_long, _ip, _ip, _ip, _dp]
        h, w, ch = C.c_int(), C.c_int(), C.c_int()
        out = np.zeros(cap)
        self._check(L.ref_load_image(path.encode(), cap, C.byref(h), C.byref(w), C.byref(ch),
                                     _ptr(out, _dp)))
        return out[:h.value * w.value * ch.value].reshape(h.value, w.value, ch.value).copy()

    def block_mean_downsample(self, image, factor):
        """gmi::block_mean_downsample (imaging.cpp:343-350)."""
        img = np.ascontiguousarray(image, np.float64)
        h, w, ch = img.shape
        lh, lw = (h + factor - 1) // factor, (w + factor - 1) // factor
        out = np.zeros((lh, lw, ch))
        L = self.lib
        L.ref_block_mean_downsample.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        self._check(L.ref_block_mean_downsample(_ptr(img, _dp), w, h, ch, factor, _ptr(out, _dp)))
        return out

    def optimize_points(self, pos, col, target, sigma, cutoff, steps, lr, opt_pos=True,
                        opt_col=False, fallback=0):
        """gmi::optimize_points (optimize.cpp:47-98) -> (positions, colors, loss_curve)."""
        pos = np.ascontiguousarray(pos, np.float64)
        col = np.ascontiguousarray(col, np.float64)
        tgt = np.ascontiguousarray(target, np.float64)
        n, ch = col.shape
        h, w = tgt.shape[:2]
        op = np.zeros_like(pos)
        oc = np.zeros_like(col)
        loss = np.zeros(steps + 1)
        self._check(self.lib.ref_optimize_points(
            _ptr(pos, _dp), _ptr(col, _dp), n, ch, _ptr(tgt, _dp), w, h, sigma, cutoff, fallback,
            steps, lr, int(opt_pos), int(opt_col), _ptr(op, _dp), _ptr(oc, _dp), _ptr(loss, _dp)))
        return op, oc, loss

    def gaussian_weight(self, qx, qy, mx, my, sigma):
        return self.lib.ref_gaussian_weight(qx, qy, mx, my, sigma)

    def bin_grid(self, pos, cell, col=None):
        pos = _d(pos).reshape(-1, 2)
        n = pos.shape[0]
        col = _d(np.full((n, 1), 0.5) if col is None else col)
        h = C.c_void_p()
        self._check(self.lib.ref_bin_grid_new(_ptr(pos, _dp), _ptr(col, _dp), n, col.shape[1], cell, C.byref(h)))
        try:
            origin = np.zeros(2)
            nc, nr = C.c_int(), C.c_int()
            self.lib.ref_bin_grid_info(h, _ptr(origin, _dp), C.byref(nc), C.byref(nr))
            bin_start = np.zeros(nc.value * nr.value + 1, np.int32)
            point_index = np.zeros(n, np.int32)
            self.lib.ref_bin_grid_copy(h, _ptr(bin_start, _ip), _ptr(point_index, _ip))
        finally:
            self.lib.ref_bin_grid_free(h)
        return dict(origin=origin, n_cols=nc.value, n_rows=nr.value,
                    bin_start=bin_start, point_index=point_index)

    def query_radius(self, pos, cell, q, radius):
        pos = _d(pos).reshape(-1, 2)
        n = pos.shape[0]
        col = np.full((n, 1), 0.5)
        out = np.zeros(n, np.int32)
        cnt = C.c_int()
        self._check(self.lib.ref_query_radius(_ptr(pos, _dp), _ptr(col, _dp), n, 1, cell, q[0], q[1], radius, _ptr(out, _ip), C.byref(cnt)))
        return out[: cnt.value].copy()

    def nearest_point(self, pos, cell, queries):
        pos = _d(pos).reshape(-1, 2)
        q = _d(queries).reshape(-1, 2)
        n = pos.shape[0]
        col = np.full((n, 1), 0.5)
        out = np.zeros(q.shape[0], np.int32)
        self._check(self.lib.ref_nearest_point(_ptr(pos, _dp), _ptr(col, _dp), n, 1, cell, _ptr(q, _dp), q.shape[0], _ptr(out, _ip)))
        return out

    def forward(self, pos, col, width, height, sigma, cutoff, fallback=0, workers=1, want_csr=False):
        """gmi::forward; returns dict(image, normalizer, fallback_flag,
        nearest_index, counts, num_pairs[, pixel_start, contrib_point,
        contrib_weight]) plus the live cache handle under 'cache' (free it
        with free_cache or pass it to backward)."""
        pos = _d(pos).reshape(-1, 2)
        col = _d(col)
        col = col.reshape(pos.shape[0], -1)
        n, ch = col.shape
        image = np.zeros((height, width, ch))
        h = C.c_void_p()
        self._check(self.lib.ref_forward(_ptr(pos, _dp), _ptr(col, _dp), n, ch, width, height, sigma, cutoff, fallback, workers, _ptr(image, _dp), C.byref(h)))
        npairs, nfb = C.c_int64(), C.c_int()
        self.lib.ref_cache_info(h, C.byref(npairs), C.byref(nfb))
        hw = width * height
        ps = np.zeros(hw + 1, np.int64)
        cp = np.zeros(max(npairs.value, 1), np.int32) if want_csr else None
        cw = np.zeros(max(npairs.value, 1)) if want_csr else None
        norm = np.zeros(hw)
        flag = np.zeros(hw, np.uint8)
        near = np.zeros(hw, np.int32)
        self.lib.ref_cache_copy(h, _ptr(ps, _i64p), _ptr(cp, _ip), _ptr(cw, _dp), _ptr(norm, _dp), _ptr(flag, _u8p), _ptr(near, _ip))
        out = dict(image=image, normalizer=norm.reshape(height, width),
                   fallback_flag=flag.reshape(height, width),
                   nearest_index=near.reshape(height, width),
                   counts=np.diff(ps).reshape(height, width),
                   num_pairs=npairs.value, fallback_count=nfb.value, cache=h)
        if want_csr:
            out.update(pixel_start=ps, contrib_point=cp[: npairs.value], contrib_weight=cw[: npairs.value])
        return out

    def free_cache(self, fwd):
        if fwd.get("cache"):
            self.lib.ref_cache_free(fwd["cache"])
            fwd["cache"] = None

    def backward(self, pos, col, fwd, upstream, sigma, cutoff, fallback=0, workers=1):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1)
        n, ch = col.shape
        up = _d(upstream)
        dc = np.zeros((n, ch))
        dp = np.zeros((n, 2))
        self._check(self.lib.ref_backward(_ptr(pos, _dp), _ptr(col, _dp), n, ch, fwd["cache"], _ptr(up, _dp), sigma, cutoff, fallback, workers, _ptr(dc, _dp), _ptr(dp, _dp)))
        return dc, dp

    def forward_backward(self, pos, col, width, height, sigma, cutoff, upstream, fallback=0, workers=1):
        f = self.forward(pos, col, width, height, sigma, cutoff, fallback, workers)
        try:
            dc, dp = self.backward(pos, col, f, upstream, sigma, cutoff, fallback, workers)
        finally:
            self.free_cache(f)
        return f, dc, dp

    def forward_backward_any_c(self, pos, col, width, height, sigma, cutoff, upstream, fallback=0, workers=1):
        """Channel-group decomposition for C not in {1,3}:
        image and d_colors per group; d_positions summed over groups."""
        col = _d(col)
        n, ch = col.shape
        groups, s = [], 0
        while s < ch:
            g = 3 if ch - s >= 3 else 1
            groups.append((s, s + g))
            s += g
        image = np.zeros((height, width, ch))
        dc = np.zeros((n, ch))
        dp = np.zeros((n, 2))
        meta = None
        for a, b in groups:
            f, gc, gp = self.forward_backward(pos, col[:, a:b], width, height, sigma, cutoff,
                                              None if upstream is None else upstream[..., a:b], fallback, workers) \
                if upstream is not None else (self.forward(pos, col[:, a:b], width, height, sigma, cutoff, fallback, workers), None, None)
            if upstream is None:
                self.free_cache(f)
            image[..., a:b] = f["image"]
            if gc is not None:
                dc[:, a:b] = gc
                dp += gp
            meta = f
        meta = dict(meta)
        meta["image"] = image
        return meta, dc, dp

    def oracle_forward(self, pos, col, width, height, sigma):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1)
        img = np.zeros((height, width, col.shape[1]))
        self._check(self.lib.ref_oracle_forward(_ptr(pos, _dp), _ptr(col, _dp), pos.shape[0], col.shape[1], width, height, sigma, _ptr(img, _dp)))
        return img

    def oracle_gradients_fd(self, pos, col, width, height, sigma, upstream, step=1e-5):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1)
        up = _d(upstream)
        dc = np.zeros(col.shape)
        dp = np.zeros(pos.shape)
        self._check(self.lib.ref_oracle_gradients_fd(_ptr(pos, _dp), _ptr(col, _dp), pos.shape[0], col.shape[1], width, height, sigma, _ptr(up, _dp), step, _ptr(dc, _dp), _ptr(dp, _dp)))
        return dc, dp

    def random_instance(self, seed, grid_max, points_max):
        n, ch, w, h = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        sg = C.c_double()
        self._check(self.lib.ref_random_instance(seed, grid_max, points_max, C.byref(n), C.byref(ch), C.byref(w), C.byref(h), C.byref(sg), None, None))
        pos = np.zeros((n.value, 2))
        col = np.zeros((n.value, ch.value))
        self._check(self.lib.ref_random_instance(seed, grid_max, points_max, C.byref(n), C.byref(ch), C.byref(w), C.byref(h), C.byref(sg), _ptr(pos, _dp), _ptr(col, _dp)))
        return dict(pos=pos, col=col, width=w.value, height=h.value, sigma=sg.value)

    def rng_u64(self, seed, k):
        out = np.zeros(k, np.uint64)
        self.lib.ref_rng_u64(seed, k, _ptr(out, _u64p))
        return out


class Oracle:
    """ctypes facade over oracle/liboracle.so (the C restatement)."""

    def __init__(self, path: str = ORC_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle liboracle.so`")
        L = self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L.orc_gaussian_weight.restype = C.c_double
        L.orc_gaussian_weight.argtypes = [C.c_double] * 5
        L.orc_validate.argtypes = [_dp, _dp, C.c_int, C.c_int, C.POINTER(C.c_long)]
        L.orc_axis_cells.argtypes = [C.c_double, C.c_double, C.c_int]
        L.orc_bin_grid_dims.argtypes = [_dp, C.c_int, C.c_double, C.c_int, _dp, _ip, _ip]
        L.orc_bin_grid_fill.argtypes = [_dp, C.c_int, C.c_double, C.c_int, _ip, _ip]
        L.orc_query_radius.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, _ip]
        L.orc_nearest_point.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_double]
        L.orc_forward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp, _u8p, _ip, _i64p]
        L.orc_backward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp, _u8p, _ip, _dp, _dp, _dp]
        L.orc_rng_u64.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.orc_synth_batch.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _fp, _fp, _fp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, "oracle")

    def gaussian_weight(self, qx, qy, mx, my, sigma):
        return self.lib.orc_gaussian_weight(qx, qy, mx, my, sigma)

    def validate(self, pos, col):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1) if pos.shape[0] else _d(col)
        idx = C.c_long()
        ch = col.shape[1] if col.ndim == 2 else 1
        rc = self.lib.orc_validate(_ptr(pos, _dp), _ptr(col, _dp), pos.shape[0], ch, C.byref(idx))
        return rc, idx.value

    def bin_grid(self, pos, cell, cap=2048):
        pos = _d(pos).reshape(-1, 2)
        n = pos.shape[0]
        origin = np.zeros(2)
        nc, nr = C.c_int(), C.c_int()
        self._check(self.lib.orc_bin_grid_dims(_ptr(pos, _dp), n, cell, cap, _ptr(origin, _dp), C.byref(nc), C.byref(nr)))
        bin_start = np.zeros(nc.value * nr.value + 1, np.int32)
        point_index = np.zeros(n, np.int32)
        self._check(self.lib.orc_bin_grid_fill(_ptr(pos, _dp), n, cell, cap, _ptr(bin_start, _ip), _ptr(point_index, _ip)))
        return dict(origin=origin, n_cols=nc.value, n_rows=nr.value,
                    bin_start=bin_start, point_index=point_index)

    def query_radius(self, pos, cell, q, radius):
        pos = _d(pos).reshape(-1, 2)
        out = np.zeros(pos.shape[0], np.int32)
        cnt = self.lib.orc_query_radius(_ptr(pos, _dp), pos.shape[0], cell, q[0], q[1], radius, _ptr(out, _ip))
        return out[:cnt].copy()

    def nearest_point(self, pos, cell, queries):
        pos = _d(pos).reshape(-1, 2)
        q = _d(queries).reshape(-1, 2)
        return np.array([self.lib.orc_nearest_point(_ptr(pos, _dp), pos.shape[0], cell, a, b) for a, b in q], np.int32)

    def forward(self, pos, col, width, height, sigma, cutoff, fallback=0):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1)
        n, ch = col.shape
        hw = width * height
        image = np.zeros((height, width, ch))
        norm = np.zeros(hw)
        flag = np.zeros(hw, np.uint8)
        near = np.zeros(hw, np.int32)
        counts = np.zeros(hw, np.int64)
        self._check(self.lib.orc_forward(_ptr(pos, _dp), _ptr(col, _dp), n, ch, width, height, sigma, cutoff, fallback,
                                         _ptr(image, _dp), _ptr(norm, _dp), _ptr(flag, _u8p), _ptr(near, _ip), _ptr(counts, _i64p)))
        return dict(image=image, normalizer=norm.reshape(height, width),
                    fallback_flag=flag.reshape(height, width),
                    nearest_index=near.reshape(height, width),
                    counts=counts.reshape(height, width),
                    num_pairs=int(counts.sum()), fallback_count=int(flag.sum()))

    def backward(self, pos, col, fwd, upstream, sigma, cutoff, fallback=0):
        pos = _d(pos).reshape(-1, 2)
        col = _d(col).reshape(pos.shape[0], -1)
        n, ch = col.shape
        height, width = fwd["normalizer"].shape
        dc = np.zeros((n, ch))
        dp = np.zeros((n, 2))
        img = _d(fwd["image"])
        norm = _d(fwd["normalizer"])
        flag = np.ascontiguousarray(fwd["fallback_flag"], np.uint8)
        near = np.ascontiguousarray(fwd["nearest_index"], np.int32)
        up = _d(upstream)
        self._check(self.lib.orc_backward(_ptr(pos, _dp), _ptr(col, _dp), n, ch, width, height, sigma, cutoff, fallback,
                                          _ptr(img, _dp), _ptr(norm, _dp), _ptr(flag, _u8p), _ptr(near, _ip), _ptr(up, _dp),
                                          _ptr(dc, _dp), _ptr(dp, _dp)))
        return dc, dp

    def rng_u64(self, seed, k):
        out = np.zeros(k, np.uint64)
        self.lib.orc_rng_u64(seed, k, _ptr(out, _u64p))
        return out

    def synth_batch(self, seed, batch, n, channels, width, height, cluster_frac=0.0, cluster_px=32, upstream=True):
        pos = np.zeros((batch, n, 2), np.float32)
        col = np.zeros((batch, n, channels), np.float32)
        up = np.zeros((batch, height, width, channels), np.float32) if upstream else None
        self.lib.orc_synth_batch(seed, batch, n, channels, width, height, cluster_frac, cluster_px,
                                 _ptr(pos, _fp), _ptr(col, _fp), _ptr(up, _fp))
        return pos, col, up


# ---------------------------------------------------------------------------
# run_benchmark's GMM branch (benchmark.cpp:88-107), restated on top of the
# C oracle's forward.


def block_mean_downsample(image, factor):
    """grid_subsample colours (imaging.cpp:306-341): per block, the f64 sum in
    row-major order times 1/area; block_mean_downsample (343-350) lays them
    out as an lh x lw x C raster."""
    img = np.asarray(image, np.float64)
    h, w, ch = img.shape
    lh, lw = (h + factor - 1) // factor, (w + factor - 1) // factor
    pad = np.zeros((lh * factor, lw * factor, ch))
    pad[:h, :w] = img
    blocks = pad.reshape(lh, factor, lw, factor, ch)
    total = np.zeros((lh, lw, ch))
    for r in range(factor):           # the reference's loop order, sequential
        for c in range(factor):       # per block (padding adds exact zeros)
            total = total + blocks[:, r, :, c, :]
    rows = np.minimum(h, (np.arange(lh) + 1) * factor) - np.arange(lh) * factor
    cols = np.minimum(w, (np.arange(lw) + 1) * factor) - np.arange(lw) * factor
    inv_area = 1.0 / (rows[:, None] * cols[None, :]).astype(np.float64)
    return total * inv_area[:, :, None]


def point_set_from_lowres(lowres, factor):
    """point_set_from_lowres (benchmark.cpp:24-39): block centres."""
    lh, lw, ch = lowres.shape
    half = (factor - 1) / 2.0
    bc, br = np.meshgrid(np.arange(lw), np.arange(lh))
    pos = np.stack([bc.ravel() * float(factor) + half, br.ravel() * float(factor) + half], 1)
    return pos, np.asarray(lowres, np.float64).reshape(-1, ch)


def l1_metric(a, b):
    """l1_metric (imaging.cpp:376-386): sequential f64 sum / size."""
    d = np.abs(np.asarray(a, np.float64).ravel() - np.asarray(b, np.float64).ravel())
    return float(np.cumsum(d)[-1] / d.size) if d.size else 0.0


def gmm_benchmark(orc, image, factor, sigmas=None, lowres=None):
    """The GMM row of run_benchmark for one image and factor with the C
    oracle's forward: (l1 per sigma, index of the first smallest)."""
    img = np.asarray(image, np.float64)
    h, w, _ = img.shape
    if lowres is None:
        lowres = block_mean_downsample(img, factor)
    pos, col = point_set_from_lowres(lowres, factor)
    if sigmas is None:
        sigmas = [0.4 * factor, 0.5 * factor, 0.6 * factor]  # benchmark.cpp:48-50
    l1 = []
    for s in sigmas:
        out = orc.forward(pos, col, w, h, s, 3.0 * s)["image"]
        l1.append(l1_metric(out, img))
    best = 0
    for k in range(1, len(l1)):
        if l1[k] < l1[best]:
            best = k
    return l1, best
