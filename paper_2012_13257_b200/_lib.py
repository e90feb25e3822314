"""ctypes binding of libgmi_b200.so (include/gmi_b200.h).

The library is the product: if it is missing this import fails loudly — there
is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

from ._build import LIB_SO

# GMI_LIBRARY: an alternative build of the same library (kernel variants
# measured side by side, tools/ab_variants.sh); default the in-tree build
_PATH = os.environ.get("GMI_LIBRARY") or LIB_SO
if not os.path.exists(_PATH):
    raise ImportError(
        f"{_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(paper_2012_13257_b200 has no CPU fallback)")

lib = C.CDLL(_PATH, mode=C.RTLD_GLOBAL)

_vp = C.c_void_p
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class GmiConfig(C.Structure):
    """gmi_config (include/gmi_b200.h) == InterpConfig (core.hpp:81-88)."""
    _fields_ = [("sigma", C.c_double), ("cutoff_radius", C.c_double),
                ("fallback", C.c_int32), ("width", C.c_int32), ("height", C.c_int32)]


# exported symbols of include/gmi_b200.h, name -> (restype, argtypes)
SIGNATURES = {
    "gmi_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "gmi_ctx_destroy": (C.c_int, [_vp]),
    "gmi_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "gmi_ctx_stream": (_vp, [_vp]),
    "gmi_ctx_set_flags": (C.c_int, [_vp, C.c_uint32]),
    "gmi_ctx_synchronize": (C.c_int, [_vp]),
    "gmi_ctx_join_host_copies": (C.c_int, [_vp]),
    "gmi_ctx_launch_count": (C.c_uint64, [_vp]),
    "gmi_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "gmi_ctx_phase_times": (C.c_int, [_vp, _dp, C.POINTER(C.c_uint64), C.c_int]),
    "gmi_last_error": (C.c_char_p, []),
    "gmi_error_name": (C.c_char_p, [C.c_int]),
    "gmi_version": (C.c_char_p, []),
    "gmi_default_cutoff": (C.c_double, [C.c_double]),
    "gmi_gaussian_weight": (C.c_double, [C.c_double] * 5),
    "gmi_forward": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int32,
                              C.POINTER(GmiConfig), _vp, C.POINTER(_vp)]),
    "gmi_backward": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int32,
                               C.POINTER(GmiConfig), _vp, _vp, _vp, _vp]),
    "gmi_forward_host": (C.c_int, [_vp, _fp, _fp, C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(GmiConfig), _fp, C.POINTER(_vp)]),
    "gmi_backward_host": (C.c_int, [_vp, _fp, _fp, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(GmiConfig), _vp, _fp, _fp, _fp]),
    "gmi_cache_free": (None, [_vp]),
    "gmi_cache_fallback_count": (C.c_int, [_vp, _i64p]),
    "gmi_cache_shape": (C.c_int, [_vp, _ip, _ip, _ip, _ip, _ip]),
    "gmi_cache_copy_pixels": (C.c_int, [_vp, _fp, _u8p, _ip]),
    "gmi_forward_counts": (C.c_int, [_vp, _vp, _ip]),
    "gmi_bin_grid": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_double, _dp, _ip, _ip,
                               _ip, _ip]),
    "gmi_bin_grid_host": (C.c_int, [_vp, _fp, C.c_int32, C.c_int32, C.c_double, _dp, _ip, _ip,
                                    _ip, _ip]),
    "gmi_optimize_points": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(GmiConfig), _vp, C.c_int32, C.c_double,
                                      C.c_uint32, _dp]),
    "gmi_optimize_points_host": (C.c_int, [_vp, _fp, _fp, C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(GmiConfig), _fp, C.c_int32, C.c_double,
                                           C.c_uint32, _dp]),
    "gmi_device_alloc": (C.c_int, [_vp, C.c_size_t, C.POINTER(_vp)]),
    "gmi_device_free": (C.c_int, [_vp, _vp]),
    "gmi_memcpy": (C.c_int, [_vp, _vp, _vp, C.c_size_t, C.c_int32]),
    "gmi_gmm_benchmark_host": (C.c_int, [_vp, _fp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         _fp, _dp, C.c_int32, _dp, _dp, C.POINTER(C.c_int32),
                                         _fp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
