"""Host-API contracts that are not numerics: asynchronous error reporting,
context lifetime against caches that outlive it, and device pointers at any
element alignment.  (sticky async errors, cache-held contexts,
misaligned 64-bit loads in the backward's staging.)"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bad_colour(orc, seed, b, i):
    pos, col, up = orc.synth_batch(seed, 2, 500, 3, 40, 30)
    col[b, i, 1] = 1.5
    return pos, col, up


def test_async_error_survives_later_calls(gmi, orc):
    # the first failing call's error stays pending across a later clean call
    actx = gmi.Context(0)
    actx.set_flags(1)
    pos, col, _ = _bad_colour(orc, 5, 1, 77)
    gmi.forward_batch(pos, col, 40, 30, 1.0, 3.0, ctx=actx)
    good, gcol, _ = orc.synth_batch(6, 3, 500, 3, 40, 30)
    gmi.forward_batch(good, gcol, 40, 30, 1.0, 3.0, ctx=actx)
    with pytest.raises(gmi.GmiError) as e:
        actx.synchronize()
    assert e.value.name == "ColorOutOfRange"
    assert "index 77" in str(e.value) and "image 1" in str(e.value)
    # reported once: nothing pending afterwards (no stale slots re-reported)
    actx.synchronize()
    gmi.forward_batch(good, gcol, 40, 30, 1.0, 3.0, ctx=actx)
    actx.synchronize()


def test_async_error_is_the_first_of_several(gmi, orc):
    actx = gmi.Context(0)
    actx.set_flags(1)
    good, gcol, _ = orc.synth_batch(8, 1, 500, 3, 40, 30)
    gmi.forward_batch(good, gcol, 40, 30, 1.0, 3.0, ctx=actx)
    pos, col, _ = _bad_colour(orc, 9, 0, 311)
    gmi.forward_batch(pos, col, 40, 30, 1.0, 3.0, ctx=actx)
    pos2, col2, _ = orc.synth_batch(10, 2, 500, 3, 40, 30)
    pos2[1, 12, 0] = np.nan
    gmi.forward_batch(pos2, col2, 40, 30, 1.0, 3.0, ctx=actx)
    with pytest.raises(gmi.GmiError) as e:
        actx.synchronize()
    assert e.value.name == "ColorOutOfRange" and "index 311" in str(e.value)
    actx.synchronize()


def test_sync_context_reports_per_call_and_leaves_nothing_pending(gmi, orc):
    sctx = gmi.Context(0)
    pos, col, _ = _bad_colour(orc, 12, 0, 3)
    with pytest.raises(gmi.GmiError):
        gmi.forward_batch(pos, col, 40, 30, 1.0, 3.0, ctx=sctx)
    sctx.synchronize()  # already reported by the call itself


def test_cache_outlives_its_context(gmi, orc):
    # a cache keeps its context (stream, device) alive: querying and freeing
    # it after the caller dropped the context handle is valid
    pos, col, up = orc.synth_batch(13, 1, 2000, 3, 64, 48)
    c1 = gmi.Context(0)
    img, cache = gmi.forward_batch(pos, col, 64, 48, 1.0, 3.0, ctx=c1)
    norm0, flag0, _ = cache.pixels()
    c1.close()
    norm1, flag1, _ = cache.pixels()
    assert np.array_equal(norm0, norm1) and np.array_equal(flag0, flag1)
    assert cache.fallback_count == int(flag0.sum())
    cache.close()
    # the device is still usable by a fresh context
    c2 = gmi.Context(0)
    img2, cache2 = gmi.forward_batch(pos, col, 64, 48, 1.0, 3.0, ctx=c2)
    assert np.array_equal(img, img2)


@pytest.mark.parametrize("offset", [1, 3])
def test_device_pointers_at_odd_element_offsets(gmi, ctx, orc, offset):
    # upstream / image views at an odd float offset: results equal the
    # aligned call bit for bit (no misaligned 64-bit loads)
    torch = pytest.importorskip("torch")
    w, h = 64, 40
    pos, col, up = orc.synth_batch(14, 1, 1500, 3, w, h)
    img, cache = gmi.forward_batch(pos, col, w, h, 1.0, 3.0, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=ctx)
    n = h * w * 3
    tpos = torch.from_numpy(pos).cuda()
    tcol = torch.from_numpy(col).cuda()
    img_store = torch.zeros(n + offset, device="cuda")
    up_store = torch.zeros(n + offset, device="cuda")
    timg = img_store[offset:].view(1, h, w, 3)
    tup = up_store[offset:].view(1, h, w, 3)
    tup.copy_(torch.from_numpy(up).cuda())
    torch.cuda.synchronize()
    out, dcache = gmi.forward_cuda(tpos, tcol, w, h, 1.0, radius=3.0, image=timg, ctx=ctx)
    ctx.synchronize()
    assert np.array_equal(timg.cpu().numpy(), img)
    ddc, ddp = gmi.backward_cuda(tpos, tcol, dcache, tup, 1.0, radius=3.0, ctx=ctx)
    ctx.synchronize()
    assert np.array_equal(ddc.numpy(), dc) and np.array_equal(ddp.numpy(), dp)


def test_parity_harness_detects_an_injected_fault(gmi, orc):
    # SURVEY §5 negative path (inject_fault, validate.cpp:207-209): the
    # device perturbs d_colors[0] by 1e-3; the parity comparison must fail
    from conftest import assert_close

    fctx = gmi.Context(0)
    fctx.set_flags(gmi.CTX_INJECT_FAULT)
    pos, col, up = orc.synth_batch(15, 1, 800, 3, 48, 40)
    img, cache = gmi.forward_batch(pos, col, 48, 40, 1.0, 3.0, ctx=fctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=fctx)
    r = orc.forward(pos[0], col[0], 48, 40, 1.0, 3.0)
    rdc, _ = orc.backward(pos[0], col[0], r, up[0], 1.0, 3.0)
    with pytest.raises(AssertionError, match="1/2400 entries"):
        assert_close(dc[0], rdc, what="d_colors")
    fctx.set_flags(0)
    dc2, _ = gmi.backward_batch(pos, col, cache, up, 1.0, 3.0, ctx=fctx)
    assert_close(dc2[0], rdc, what="d_colors")


def test_fuzzer_fails_on_an_injected_fault(tmp_path):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_parity.py"), "--seconds", "8",
                        "--inject-fault", "--out", str(tmp_path), "--max-fail", "3"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 1 and "FUZZ FAILED" in r.stdout, r.stdout[-2000:]


def test_pinned_and_pageable_host_buffers_agree(gmi, orc):
    # the host API takes two routes: all-pinned buffers run the chunked
    # three-stream pipeline (composite cache), pageable ones are staged
    # through the context's pinned slots; results are bit-identical, and a
    # cache made by either route serves a backward on either route
    import ctypes as C

    torch = pytest.importorskip("torch")
    B, N, Cc, W, H = 5, 3000, 3, 96, 80
    pos, col, up = orc.synth_batch(16, B, N, Cc, W, H)
    ctx = gmi.Context(0)
    img_a, cache_a = gmi.forward_batch(pos, col, W, H, 1.5, 4.5, ctx=ctx)   # pageable
    dc_a, dp_a = gmi.backward_batch(pos, col, cache_a, up, 1.5, 4.5, ctx=ctx)

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    ppos, pcol, pup = pinned(pos), pinned(col), pinned(up)
    pimg, pdc, pdp = pinned(np.zeros_like(img_a)), pinned(np.zeros_like(dc_a)), pinned(np.zeros_like(dp_a))
    fp = C.POINTER(C.c_float)
    cfg = gmi._lib.GmiConfig(1.5, 4.5, 0, W, H)
    h = C.c_void_p()
    gmi._check(gmi.lib.gmi_forward_host(ctx.handle, ppos.ctypes.data_as(fp), pcol.ctypes.data_as(fp), B, N,
                                        Cc, C.byref(cfg), pimg.ctypes.data_as(fp), C.byref(h)))
    cache_b = gmi.ForwardCache(h, ctx)
    gmi._check(gmi.lib.gmi_backward_host(ctx.handle, ppos.ctypes.data_as(fp), pcol.ctypes.data_as(fp), B, N,
                                         Cc, C.byref(cfg), cache_b.handle, pup.ctypes.data_as(fp),
                                         pdc.ctypes.data_as(fp), pdp.ctypes.data_as(fp)))
    assert np.array_equal(img_a, pimg)
    assert np.array_equal(dc_a, pdc) and np.array_equal(dp_a, pdp)
    # the pinned route's composite cache with a pageable backward
    dc_c, dp_c = gmi.backward_batch(pos, col, cache_b, up, 1.5, 4.5, ctx=ctx)
    assert np.array_equal(dc_a, dc_c) and np.array_equal(dp_a, dp_c)
    # the pageable route's cache with a pinned backward
    pdc[:] = 0
    gmi._check(gmi.lib.gmi_backward_host(ctx.handle, ppos.ctypes.data_as(fp), pcol.ctypes.data_as(fp), B, N,
                                         Cc, C.byref(cfg), cache_a.handle, pup.ctypes.data_as(fp),
                                         pdc.ctypes.data_as(fp), pdp.ctypes.data_as(fp)))
    assert np.array_equal(dc_a, pdc)


def test_concurrent_contexts_from_host_threads(gmi, orc):
    # SURVEY §8(b) threading: one context per host thread on the same device,
    # calls in flight concurrently (ctypes drops the GIL), results identical
    # to the same calls made one after the other
    import threading

    cases = [orc.synth_batch(100 + k, 2, 2500, 3, 80, 64) for k in range(4)]
    ctxs = [gmi.Context(0) for _ in cases]
    want = []
    for (pos, col, up), ctx in zip(cases, ctxs):
        img, cache = gmi.forward_batch(pos, col, 80, 64, 1.5, 4.5, ctx=ctx)
        dc, dp = gmi.backward_batch(pos, col, cache, up, 1.5, 4.5, ctx=ctx)
        want.append((img, dc, dp))
    got = [None] * len(cases)
    errors = []

    def work(k):
        try:
            pos, col, up = cases[k]
            for _ in range(3):
                img, cache = gmi.forward_batch(pos, col, 80, 64, 1.5, 4.5, ctx=ctxs[k])
                dc, dp = gmi.backward_batch(pos, col, cache, up, 1.5, 4.5, ctx=ctxs[k])
            got[k] = (img, dc, dp)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k in range(len(cases)):
        for a, b in zip(got[k], want[k]):
            assert np.array_equal(a, b)
