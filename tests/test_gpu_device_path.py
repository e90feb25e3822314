"""Zero-copy device path: forward_cuda / backward_cuda on
__cuda_array_interface__ arrays, DeviceArray without PyTorch, and PyTorch
interop — bitwise equal to the host-buffer path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_array_round_trip(gmi, ctx):
    a = np.random.default_rng(0).standard_normal((3, 5, 7)).astype(np.float32)
    d = gmi.DeviceArray.from_numpy(a, ctx)
    assert d.__cuda_array_interface__["shape"] == (3, 5, 7)
    assert np.array_equal(d.numpy(), a)


def test_forward_backward_cuda_match_host_path(gmi, ctx, orc):
    pos, col, up = orc.synth_batch(41, 3, 4000, 3, 90, 70)
    img, cache = gmi.forward_batch(pos, col, 90, 70, 1.5, 4.5, ctx=ctx)
    dc, dp = gmi.backward_batch(pos, col, cache, up, 1.5, 4.5, ctx=ctx)
    dpos, dcol = gmi.DeviceArray.from_numpy(pos, ctx), gmi.DeviceArray.from_numpy(col, ctx)
    dimg, dcache = gmi.forward_cuda(dpos, dcol, 90, 70, 1.5, radius=4.5, ctx=ctx)
    assert np.array_equal(dimg.numpy(), img)
    ddc, ddp = gmi.backward_cuda(dpos, dcol, dcache, gmi.DeviceArray.from_numpy(up, ctx), 1.5,
                                 radius=4.5, ctx=ctx)
    assert np.array_equal(ddc.numpy(), dc) and np.array_equal(ddp.numpy(), dp)
    assert dcache.fallback_count == cache.fallback_count


def test_torch_interop_zero_copy(gmi, ctx, orc):
    torch = pytest.importorskip("torch")
    pos, col, up = orc.synth_batch(42, 1, 3000, 1, 64, 48)
    tpos = torch.from_numpy(pos[0]).cuda()          # N x 2 (single image)
    tcol = torch.from_numpy(col[0]).cuda()
    timg = torch.empty(48, 64, 1, device="cuda")
    torch.cuda.synchronize()
    out, cache = gmi.forward_cuda(tpos, tcol, 64, 48, 1.0, image=timg, ctx=ctx)
    assert out is timg
    ref_img, _ = gmi.forward_batch(pos, col, 64, 48, 1.0, ctx=ctx)
    assert np.array_equal(timg.cpu().numpy(), ref_img[0])
    # a DeviceArray output wrapped by torch without a copy
    dc, dp = gmi.backward_cuda(tpos, tcol, cache, torch.from_numpy(up[0]).cuda(), 1.0, ctx=ctx)
    t = torch.as_tensor(dc, device="cuda")
    assert t.data_ptr() == dc.ptr and tuple(t.shape) == (1, 3000, 1)


def test_device_path_validation(gmi, ctx):
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError):
        gmi.forward_cuda(np.zeros((1, 4, 2), np.float32), np.zeros((1, 4, 1), np.float32), 8, 8, 1.0)
    with pytest.raises(TypeError):
        gmi.forward_cuda(torch.zeros(1, 4, 2, dtype=torch.float64, device="cuda"),
                         torch.zeros(1, 4, 1, device="cuda"), 8, 8, 1.0, ctx=ctx)
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward_cuda(torch.zeros(1, 4, 2, device="cuda").transpose(1, 2).contiguous().transpose(1, 2),
                         torch.zeros(1, 4, 1, device="cuda"), 8, 8, 1.0, ctx=ctx)
    assert e.value.code == 4
    with pytest.raises(gmi.GmiError) as e:
        gmi.forward_cuda(torch.zeros(1, 4, 2, device="cuda"), torch.zeros(1, 5, 1, device="cuda"),
                         8, 8, 1.0, ctx=ctx)
    assert e.value.code == 4


@pytest.mark.parametrize("n", [3000, 250])  # 250: many fallback pixels (K3 / K5 in the graph)
def test_cuda_graph_capture_replays_the_step(gmi, orc, n):
    # a whole forward + backward (binning, gather, special pixels, backward,
    # the cache's stream-ordered allocations and frees) captured once as a
    # CUDA graph and replayed gives the eager results bit for bit
    torch = pytest.importorskip("torch")
    pos, col, up = orc.synth_batch(43, 2, n, 3, 80, 60)
    if n < 1000:
        assert gmi.forward_batch(pos, col, 80, 60, 1.0, 3.0)[1].fallback_count > 0
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    tpos, tcol, tup = (torch.from_numpy(a).to(dev) for a in (pos, col, up))
    img = torch.empty(2, 60, 80, 3, device=dev)
    dc = torch.empty(2, n, 3, device=dev)
    dp = torch.empty(2, n, 2, device=dev)
    gctx = gmi.Context(0)
    gctx.set_stream(s.cuda_stream)
    gctx.set_flags(1)
    torch.cuda.synchronize()

    def step():
        cache = gctx.forward_device(tpos, tcol, 2, n, 3, 80, 60, 1.0, 3.0, 0, img)
        gctx.backward_device(tpos, tcol, 2, n, 3, 80, 60, 1.0, 3.0, 0, cache, tup, dc, dp)
        del cache

    for _ in range(3):
        step()
    gctx.synchronize()
    want = (img.cpu().numpy(), dc.cpu().numpy(), dp.cpu().numpy())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for t in (img, dc, dp):
        t.zero_()
    with torch.cuda.stream(s):
        g.replay()
        g.replay()
    torch.cuda.synchronize()
    gctx.synchronize()
    assert np.array_equal(img.cpu().numpy(), want[0])
    assert np.array_equal(dc.cpu().numpy(), want[1]) and np.array_equal(dp.cpu().numpy(), want[2])
