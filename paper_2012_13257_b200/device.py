"""Zero-copy device path without PyTorch (the reference binding's
forward / backward, bindings.cpp:147-184, on device memory).

Any producer of ``__cuda_array_interface__`` (v2/v3: this package's
``DeviceArray``, PyTorch, CuPy, Numba ...) is accepted as float32,
C-contiguous, batch-major arrays: positions B x N x 2 (or N x 2), colours
B x N x C, image / upstream B x H x W x C, d_colors B x N x C, d_positions
B x N x 2.  Missing outputs are allocated as ``DeviceArray`` objects, which
other frameworks can wrap without a copy (``torch.as_tensor(arr,
device="cuda")``, ``cupy.asarray(arr)``).

Streams: the work runs on the context's stream, and a ``DeviceArray``
exports that stream in its interface (v3), so a consumer orders itself
after it.  Inputs from other producers must be complete when the call is
made (synchronise their stream first).  The returned ``ForwardCache``
borrows positions, colours and the image, exactly like the C-ABI
``gmi_forward``; keep them unchanged until the backward.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib


class DeviceArray:
    """float32 device memory owned by this object (freed on GC) with
    ``__cuda_array_interface__`` (version 3)."""

    def __init__(self, shape, ctx=None):
        from . import _check, default_context

        self.ctx = ctx or default_context()
        self.shape = tuple(int(s) for s in shape)
        self.nbytes = 4 * int(np.prod(self.shape, dtype=np.int64))
        p = C.c_void_p()
        _check(lib.gmi_device_alloc(self.ctx.handle, self.nbytes, C.byref(p)))
        self.ptr = p.value or 0

    def __del__(self):
        try:
            if getattr(self, "ptr", 0):
                lib.gmi_device_free(self.ctx.handle, C.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:
            pass

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": "<f4", "data": (self.ptr, False), "strides": None,
                "version": 3, "stream": self.ctx.stream or None}

    @classmethod
    def from_numpy(cls, a, ctx=None) -> "DeviceArray":
        from . import _check

        h = np.ascontiguousarray(a, dtype=np.float32)
        out = cls(h.shape, ctx)
        _check(lib.gmi_memcpy(out.ctx.handle, C.c_void_p(out.ptr), h.ctypes.data_as(C.c_void_p),
                              out.nbytes, 0))
        return out

    def numpy(self) -> np.ndarray:
        from . import _check

        h = np.empty(self.shape, np.float32)
        _check(lib.gmi_memcpy(self.ctx.handle, h.ctypes.data_as(C.c_void_p), C.c_void_p(self.ptr),
                              self.nbytes, 1))
        return h


def _device(x, name: str, ndim_ok=(3,)):
    """(pointer, shape) of a float32 C-contiguous CUDA array interface."""
    from . import GmiError

    cai = getattr(x, "__cuda_array_interface__", None)
    if cai is None:
        raise TypeError(f"{name}: expected an object with __cuda_array_interface__")
    shape = tuple(int(s) for s in cai["shape"])
    if cai.get("typestr") != "<f4":
        raise TypeError(f"{name}: expected float32 (typestr '<f4'), got {cai.get('typestr')}")
    strides = cai.get("strides")
    if strides is not None:
        want, acc = [], 4
        for s in reversed(shape):
            want.append(acc)
            acc *= s
        if tuple(int(v) for v in strides) != tuple(reversed(want)):
            raise GmiError(4, f"{name}: must be C-contiguous")
    if len(shape) not in ndim_ok:
        raise GmiError(4, f"{name}: expected {' or '.join(map(str, ndim_ok))} dimensions, got {shape}")
    return int(cai["data"][0]), shape


def forward_cuda(positions, colors, width: int, height: int, sigma: float, radius: float = 0.0,
                 fallback: str = "nearest", image=None, ctx=None):
    """forward (bindings.cpp:147-160) on device arrays -> (image, ForwardCache);
    the image is written into ``image`` when given, else a new DeviceArray."""
    from . import ForwardCache, GmiError, _check, _interp_config, default_context

    ctx = ctx or default_context()
    pp, ps = _device(positions, "positions", (2, 3))
    cp, cs = _device(colors, "colors", (2, 3))
    if len(ps) == 2:
        ps, cs = (1,) + ps, (1,) + cs
    if ps[2] != 2 or len(cs) != 3 or cs[:2] != ps[:2]:
        raise GmiError(4, "positions must be BxNx2 and colors BxNxC with matching B, N")
    b, n, ch = cs
    if image is None:
        image = DeviceArray((b, height, width, ch), ctx)
    ip, ishape = _device(image, "image", (3, 4))
    if int(np.prod(ishape)) != b * height * width * ch:
        raise GmiError(4, "image must hold B x H x W x C floats")
    cfg = _interp_config(sigma, radius, fallback, width, height)
    h = C.c_void_p()
    _check(lib.gmi_forward(ctx.handle, C.c_void_p(pp), C.c_void_p(cp), b, n, ch, C.byref(cfg),
                           C.c_void_p(ip), C.byref(h)))
    return image, ForwardCache(h, ctx, keep=(positions, colors, image))


def backward_cuda(positions, colors, cache, upstream, sigma: float, radius: float = 0.0,
                  fallback: str = "nearest", d_colors=None, d_positions=None, ctx=None):
    """backward (bindings.cpp:162-184) on device arrays -> (d_colors,
    d_positions), written into the given arrays or new DeviceArrays."""
    from . import GmiError, _check, _interp_config

    ctx = ctx or cache._ctx
    pp, ps = _device(positions, "positions", (2, 3))
    cp, cs = _device(colors, "colors", (2, 3))
    if len(ps) == 2:
        ps, cs = (1,) + ps, (1,) + cs
    b, n, ch = cs
    up, ushape = _device(upstream, "upstream", (3, 4))
    if int(np.prod(ushape)) != b * cache.height * cache.width * ch:
        raise GmiError(4, "upstream must be BxHxWxC matching the forward output")
    if d_colors is None:
        d_colors = DeviceArray((b, n, ch), ctx)
    if d_positions is None:
        d_positions = DeviceArray((b, n, 2), ctx)
    dcp, dcs = _device(d_colors, "d_colors", (2, 3))
    dpp, dps = _device(d_positions, "d_positions", (2, 3))
    if int(np.prod(dcs)) != b * n * ch or int(np.prod(dps)) != b * n * 2:
        raise GmiError(4, "d_colors must hold B x N x C and d_positions B x N x 2 floats")
    cfg = _interp_config(sigma, radius, fallback, cache.width, cache.height)
    _check(lib.gmi_backward(ctx.handle, C.c_void_p(pp), C.c_void_p(cp), b, n, ch, C.byref(cfg),
                            cache.handle, C.c_void_p(up), C.c_void_p(dcp), C.c_void_p(dpp)))
    return d_colors, d_positions
