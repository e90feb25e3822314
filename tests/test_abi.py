"""CPU: the drop-in boundary.  libgmi_b200.so loads without a GPU, exports
every entry point include/gmi_b200.h declares, fails loudly (no CPU fallback)
when no device is present, and the Python shim mirrors the reference binding's
host-side contract (gmi._core, bindings.cpp:95-184) — argument checks, error
types and codes — without any compute."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gmi_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gmi_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("gmi_forward", "gmi_backward", "gmi_forward_host", "gmi_backward_host",
                 "gmi_bin_grid", "gmi_cache_free", "gmi_ctx_create", "gmi_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(gmi):
    from paper_2012_13257_b200._build import LIB_SO

    lib = C.CDLL(LIB_SO)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gmi_[a-z0-9_]+)\b", out))
    assert set(declared_functions()) <= exported
    # every ctypes signature the shim binds is a declared symbol
    from paper_2012_13257_b200._lib import SIGNATURES
    assert set(SIGNATURES) <= set(declared_functions())


def test_library_targets_sm100a(gmi):
    from paper_2012_13257_b200._build import LIB_SO

    out = subprocess.run(["cuobjdump", "--list-elf", LIB_SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_names_follow_reference_codes(gmi):
    # core.hpp:35-50 ErrorCode order, offset by one
    names = [gmi.lib.gmi_error_name(k).decode() for k in range(1, 9)]
    assert names == ["NonFiniteValue", "ColorOutOfRange", "EmptyPointSet", "ShapeMismatch",
                     "InvalidCellSize", "ConfigInvalid", "CacheMismatch", "InvalidDimensions"]
    assert gmi.lib.gmi_default_cutoff(1.5) == 4.5  # make_config (core.hpp:90-94)


def test_host_gaussian_weight_kats(gmi):
    # test_core.cpp:11-17 through the C-ABI helper
    assert gmi.gaussian_weight(0, 0, 0, 0, 1.0) == 1.0
    assert gmi.gaussian_weight(1, 0, 0, 0, 1.0) == pytest.approx(0.6065306597126334, rel=1e-14)
    assert gmi.gaussian_weight(0.5, 0.5, 2, 0, 1.0) == pytest.approx(0.2865047968601901, rel=1e-14)


def test_no_device_fails_loudly(gmi):
    """Without a GPU the C-ABI returns a CUDA error and a message; it never
    computes on the CPU."""
    if os.environ.get("CUDA_VISIBLE_DEVICES", None) != "" and _has_gpu():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = gmi.lib.gmi_ctx_create(0, C.byref(h))
    assert rc in (100, 101)
    assert gmi.lib.gmi_last_error().decode()
    with pytest.raises((gmi.GmiError, ValueError)):
        gmi.Context(0)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_null_and_argument_checks_without_device(gmi):
    # argument validation happens before any device work (core.cpp:98-120)
    lib = gmi.lib
    cfg = gmi._lib.GmiConfig(1.0, 3.0, 0, 4, 4)
    h = C.c_void_p()
    pos = np.zeros((1, 2, 2), np.float32)
    col = np.zeros((1, 2, 1), np.float32)
    img = np.zeros((1, 4, 4, 1), np.float32)
    fp = C.POINTER(C.c_float)
    # null ctx -> InvalidArgument
    rc = lib.gmi_forward(None, pos.ctypes.data, col.ctypes.data, 1, 2, 1, C.byref(cfg),
                         img.ctypes.data, C.byref(h))
    assert rc == 101
    # config checks come from a real ctx only; exercise check order via host API
    bad = gmi._lib.GmiConfig(-1.0, 3.0, 0, 4, 4)
    rc = lib.gmi_forward_host(C.c_void_p(1), pos.ctypes.data_as(fp), col.ctypes.data_as(fp), 1, 0,
                              1, C.byref(bad), img.ctypes.data_as(fp), C.byref(h))
    assert rc == 3  # EmptyPointSet before ConfigInvalid (validate_point_set first)


def test_pointset_validation_matches_reference(gmi):
    # bindings.cpp:57-76 + core.cpp:55-96: constructor validates
    with pytest.raises(gmi.GmiError) as e:
        gmi.PointSet(np.zeros((1, 2)), np.array([[1.5]]))
    assert e.value.name == "ColorOutOfRange"
    with pytest.raises(gmi.GmiError) as e:
        gmi.PointSet(np.array([[0.0, 0.0], [np.inf, 1.0]]), np.array([[0.5], [0.5]]))
    assert e.value.name == "NonFiniteValue" and "index 1" in str(e.value)
    with pytest.raises(gmi.GmiError) as e:
        gmi.PointSet(np.zeros((0, 2)), np.zeros((0, 1)))
    assert e.value.name == "EmptyPointSet"
    with pytest.raises(ValueError):
        gmi.PointSet(np.zeros((3, 3)), np.zeros((3, 1)))
    with pytest.raises(ValueError):
        gmi.PointSet(np.zeros((3, 2)), np.zeros((2, 1)))
    ps = gmi.PointSet(np.array([[0.25, 1.5], [3.0, 2.0]]), np.array([[0.1, 0.2, 0.3], [1.0, 0.0, 0.5]]))
    assert len(ps) == 2 and ps.channels == 3
    assert ps.positions.shape == (2, 2) and ps.colors.shape == (2, 3)


def test_interp_config_semantics(gmi):
    # make_interp_config (bindings.cpp:95-108): radius <= 0 -> 3 sigma
    c = gmi._interp_config(1.5, 0.0, "nearest", 8, 6)
    assert (c.sigma, c.cutoff_radius, c.fallback, c.width, c.height) == (1.5, 4.5, 0, 8, 6)
    c = gmi._interp_config(1.0, 2.5, "zero", 8, 6)
    assert (c.cutoff_radius, c.fallback) == (2.5, 1)
    with pytest.raises(ValueError):
        gmi._interp_config(1.0, 0.0, "bilinear", 8, 6)


def test_pointset_reports_fp32_rounding():
    # weak r1 #12: f64 inputs the fp32 device path rounds are counted, and
    # can warn or be rejected instead of silently changing the bins
    import warnings

    import paper_2012_13257_b200 as gmi

    exact = gmi.PointSet([[0.5, 1.25]], [[0.25, 0.5, 0.75]])
    assert exact.inexact_inputs == 0
    rounded = gmi.PointSet([[0.1, 1.25]], [[0.3, 0.5, 0.75]])
    assert rounded.inexact_inputs == 2
    try:
        gmi.set_fp32_inputs("warn")
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            gmi.PointSet([[0.1, 1.0]], [[0.5]])
        assert any(issubclass(x.category, gmi.PrecisionWarning) for x in w)
        gmi.set_fp32_inputs("reject")
        with pytest.raises(gmi.GmiError):
            gmi.PointSet([[0.1, 1.0]], [[0.5]])
        gmi.PointSet([[0.5, 1.0]], [[0.5]])  # exact values still pass
    finally:
        gmi.set_fp32_inputs("allow")
