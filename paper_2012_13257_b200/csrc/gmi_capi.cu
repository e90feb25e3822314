// The C-ABI (include/gmi_b200.h): argument checks with the reference's error
// codes, the ForwardCache lifecycle and the orchestration of K1..K5 on one
// stream.  No exception crosses the ABI; every failure becomes a status code
// plus a thread-local message.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "gmi_internal.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        const int rc = f();
        if (rc == GMI_OK) g_last_error.clear();
        return rc;
    } catch (const GmiFail& e) {
        return fail(e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(GMI_ERR_CUDA, e.what());
    }
}

// core.cpp:104-113 (require_valid(InterpConfig)) and core.cpp:115-120
int check_config(const gmi_config* cfg) {
    if (cfg == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "config is null");
    if (!std::isfinite(cfg->sigma) || cfg->sigma <= 0.0)
        return fail(GMI_ERR_CONFIG_INVALID, "sigma must be positive and finite");
    if (!std::isfinite(cfg->cutoff_radius) || cfg->cutoff_radius <= 0.0)
        return fail(GMI_ERR_CONFIG_INVALID, "cutoff_radius must be positive and finite");
    if (cfg->fallback != GMI_FALLBACK_NEAREST && cfg->fallback != GMI_FALLBACK_ZERO)
        return fail(GMI_ERR_INVALID_ARGUMENT, "fallback must be NEAREST or ZERO");
    if (cfg->width < 1 || cfg->height < 1)
        return fail(GMI_ERR_INVALID_DIMENSIONS, "frame dimensions must be at least 1x1");
    return GMI_OK;
}

// core.cpp:55-66 (shape part of validate_point_set; C relaxed to >= 1)
int check_points(const float* pos, const float* col, int B, int N, int C) {
    if (B < 1) return fail(GMI_ERR_INVALID_ARGUMENT, "batch must be >= 1");
    if (N <= 0) return fail(GMI_ERR_EMPTY_POINT_SET, "point set is empty");
    if (C < 1) return fail(GMI_ERR_SHAPE_MISMATCH, "channels must be >= 1, got " + std::to_string(C));
    if (pos == nullptr || col == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "null point arrays");
    if (reinterpret_cast<uintptr_t>(pos) % 8 != 0)
        return fail(GMI_ERR_INVALID_ARGUMENT, "positions must be 8-byte aligned");
    if (static_cast<int64_t>(B) * N > (int64_t(1) << 31) - 1)
        return fail(GMI_ERR_INVALID_ARGUMENT, "batch*num_points exceeds 2^31-1");
    return GMI_OK;
}

// Hot-path cell cap: the reference's 2048 (bin_grid.cpp:14) unless the frame
// itself needs more cells, in which case the cap grows so the output frame
// is covered without clamping (the 2048 cap puts >1M
// points in one bin at 8192^2 / r=3).  When the reference grid is not capped
// the two are identical.
//
// The device-geometry path (no host round trip) caps at the frame's own need:
// points inside the frame never reach it, so the grid is still the
// reference's; only point sets reaching far outside the frame get clamped
// edge cells (exact, see gmi_bin.cu / nearest_exact).
int frame_cells(const gmi_config* cfg) {
    const double span = std::max(cfg->width, cfg->height) + 2.0 * cfg->cutoff_radius;
    const double need = std::ceil(span / cfg->cutoff_radius) + 8.0;
    return static_cast<int>(std::min(8192.0, need));
}

void ensure_issue(gmi_ctx* ctx, int B) {
    if (ctx->d_issue_cap < B) {
        if (ctx->d_issue) cudaFree(ctx->d_issue);
        if (ctx->h_issue) cudaFreeHost(ctx->h_issue);
        GMI_CUDA(cudaMalloc(&ctx->d_issue, sizeof(unsigned long long) * B));
        GMI_CUDA(cudaMallocHost(&ctx->h_issue, sizeof(unsigned long long) * B));
        ctx->d_issue_cap = B;
    }
}

// Reads the colour-validation keys (core.cpp:80-92) after the stream drained.
int collect_issue(gmi_ctx* ctx, int B) {
    GMI_CUDA(cudaMemcpyAsync(ctx->h_issue, ctx->d_issue, sizeof(unsigned long long) * B,
                             cudaMemcpyDeviceToHost, ctx->stream));
    GMI_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < B; ++b) {
        const unsigned long long k = ctx->h_issue[b];
        if (k == gmi_dev::kNoIssue) continue;
        const long idx = static_cast<long>(k >> 8);
        const int code = static_cast<int>(k & 0xff);
        const std::string where = " at index " + std::to_string(idx) +
                                  (B > 1 ? " (image " + std::to_string(b) + ")" : "");
        if (code == GMI_ERR_COLOR_OUT_OF_RANGE)
            return fail(code, "color out of [0,1]" + where);
        if (code == GMI_ERR_OUT_OF_MEMORY)
            return fail(code, "more than " + std::to_string(idx) + " fallback pixels in one call");
        return fail(code, "non-finite value" + where);
    }
    return GMI_OK;
}

// ---- pageable host buffers ----------------------------------------------
// cudaMemcpyAsync from / to pageable memory runs through the driver's own
// bounce buffers one piece at a time (~6 GB/s here).  The host API instead
// stages pageable buffers through two 64 MB pinned slots of the context:
// host threads copy piece k+1 into one slot while the DMA of piece k runs
// from the other.
constexpr size_t kStageSlot = size_t(64) << 20;

bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

void parallel_memcpy(void* dst, const void* src, size_t n) {
    const size_t kPer = size_t(8) << 20;
    const int hw = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    const int nt = static_cast<int>(std::min<size_t>(hw, (n + kPer - 1) / kPer));
    if (nt <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    const size_t step = ((n + nt - 1) / nt + 63) & ~size_t(63);
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) {
        const size_t a = std::min(n, t * step), b = std::min(n, (t + 1) * step);
        if (b > a)
            th.emplace_back([=] {
                std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
            });
    }
    std::memcpy(dst, src, std::min(n, step));
    for (auto& t : th) t.join();
}

void ensure_staging(gmi_ctx* ctx) {
    for (int s = 0; s < 2; ++s) {
        if (ctx->stg_slot[s] == nullptr) GMI_CUDA(cudaMallocHost(&ctx->stg_slot[s], kStageSlot));
        if (ctx->stg_ev[s] == nullptr)
            GMI_CUDA(cudaEventCreateWithFlags(&ctx->stg_ev[s], cudaEventDisableTiming));
    }
}

// host (pageable) -> device, queued on `st`; returns with the last DMA queued
void h2d_staged(gmi_ctx* ctx, void* dst, const void* src, size_t n, cudaStream_t st) {
    ensure_staging(ctx);
    int s = 0;
    for (size_t off = 0; off < n; off += kStageSlot, s ^= 1) {
        const size_t m = std::min(kStageSlot, n - off);
        GMI_CUDA(cudaEventSynchronize(ctx->stg_ev[s]));  // the slot's previous DMA is done
        parallel_memcpy(ctx->stg_slot[s], static_cast<const char*>(src) + off, m);
        GMI_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->stg_slot[s], m,
                                 cudaMemcpyHostToDevice, st));
        GMI_CUDA(cudaEventRecord(ctx->stg_ev[s], st));
    }
}

// device -> host (pageable) after the work queued on `st`; returns complete
void d2h_staged(gmi_ctx* ctx, void* dst, const void* src, size_t n, cudaStream_t st) {
    ensure_staging(ctx);
    size_t prev_off = 0, prev_m = 0;
    int s = 0;
    for (size_t off = 0; off < n; off += kStageSlot, s ^= 1) {
        const size_t m = std::min(kStageSlot, n - off);
        GMI_CUDA(cudaEventSynchronize(ctx->stg_ev[s]));
        GMI_CUDA(cudaMemcpyAsync(ctx->stg_slot[s], static_cast<const char*>(src) + off, m,
                                 cudaMemcpyDeviceToHost, st));
        GMI_CUDA(cudaEventRecord(ctx->stg_ev[s], st));
        if (prev_m) {  // the other slot's piece is down: copy it out while this one comes
            GMI_CUDA(cudaEventSynchronize(ctx->stg_ev[s ^ 1]));
            parallel_memcpy(static_cast<char*>(dst) + prev_off, ctx->stg_slot[s ^ 1], prev_m);
        }
        prev_off = off;
        prev_m = m;
    }
    if (prev_m) {
        GMI_CUDA(cudaEventSynchronize(ctx->stg_ev[s ^ 1]));
        parallel_memcpy(static_cast<char*>(dst) + prev_off, ctx->stg_slot[s ^ 1], prev_m);
    }
}

// The ctx stream waits for the copy streams of the host-buffer API.
void join_copy_streams(gmi_ctx* ctx) {
    for (cudaStream_t cs : {ctx->s_in, ctx->s_out}) {
        if (cs == nullptr) continue;
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) continue;
        cudaEventRecord(ev, cs);
        cudaStreamWaitEvent(ctx->stream, ev, 0);
        cudaEventDestroy(ev);
    }
}


// GMI_CTX_ASYNC_ERRORS, after a forward: a fallback-list overflow becomes an
// issue of the call, and the call's first failing image (slots in image
// order) becomes the ctx's pending error unless an earlier call already left
// one — stream order makes "earlier" the call order, so gmi_ctx_synchronize
// reports the first error since it last ran (pending == null: the caller
// collects the call's issues itself).
// One warp: the images' issue slots 32 at a time (ballot -> first failing
// image), so the check costs one round trip per 32 images, not one per image.
__global__ void k_async_check(const int32_t* count, int cap, unsigned long long* issue, int B,
                              int b0, unsigned long long* pending) {
    const int lane = threadIdx.x;
    if (lane == 0 && *count > cap)
        atomicMin(issue, (static_cast<unsigned long long>(cap) << 8) | GMI_ERR_OUT_OF_MEMORY);
    __syncwarp();
    if (pending == nullptr || pending[0] != gmi_dev::kNoIssue) return;
    for (int b1 = 0; b1 < B; b1 += 32) {
        const int b = b1 + lane;
        const unsigned long long k = b < B ? issue[b] : gmi_dev::kNoIssue;
        const unsigned bad = __ballot_sync(0xffffffffu, k != gmi_dev::kNoIssue);
        if (bad != 0u) {
            if (lane == __ffs(bad) - 1) {
                pending[0] = k;
                pending[1] = static_cast<unsigned long long>(b0 + b);
            }
            return;
        }
    }
}

// Reads and clears the pending asynchronous error (stream drained).
int collect_pending(gmi_ctx* ctx) {
    unsigned long long h[2];
    GMI_CUDA(cudaMemcpyAsync(h, ctx->d_pending, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    GMI_CUDA(cudaMemsetAsync(ctx->d_pending, 0xFF, sizeof(h), ctx->stream));
    GMI_CUDA(cudaStreamSynchronize(ctx->stream));
    const unsigned long long k = h[0];
    if (k == gmi_dev::kNoIssue) return GMI_OK;
    const long idx = static_cast<long>(k >> 8);
    const int code = static_cast<int>(k & 0xff);
    const std::string where = " at index " + std::to_string(idx) + " (image " +
                              std::to_string(static_cast<long>(h[1])) + ")";
    if (code == GMI_ERR_COLOR_OUT_OF_RANGE) return fail(code, "color out of [0,1]" + where);
    if (code == GMI_ERR_OUT_OF_MEMORY)
        return fail(code, "more than " + std::to_string(idx) + " fallback pixels in one call");
    return fail(code, "non-finite value" + where);
}

void ctx_retain(gmi_ctx* ctx) { ctx->refs.fetch_add(1, std::memory_order_relaxed); }

void ctx_teardown(gmi_ctx* ctx) {
    cudaSetDevice(ctx->device);
    // the grow-only scratch slots go back to the pool with the context
    for (int s = 0; s < WS_COUNT; ++s)
        if (ctx->ws_ptr[s]) cudaFreeAsync(ctx->ws_ptr[s], ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->d_issue) cudaFree(ctx->d_issue);
    if (ctx->h_issue) cudaFreeHost(ctx->h_issue);
    if (ctx->d_pending) cudaFree(ctx->d_pending);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
    if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
    for (int s = 0; s < 2; ++s) {
        if (ctx->stg_slot[s]) cudaFreeHost(ctx->stg_slot[s]);
        if (ctx->stg_ev[s]) cudaEventDestroy(ctx->stg_ev[s]);
    }
    delete ctx;
}

// Drops one reference; the last one (creator or cache) tears the ctx down.
void ctx_release(gmi_ctx* ctx) {
    if (ctx->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) ctx_teardown(ctx);
}

void free_cache_buffers(gmi_cache* c) {
    if (c->d2h_done != nullptr) {
        // an asynchronous gmi_forward_host may still be downloading the image
        cudaStreamWaitEvent(c->ctx->stream, c->d2h_done, 0);
        cudaEventDestroy(c->d2h_done);
        c->d2h_done = nullptr;
    }
    for (gmi_cache* part : c->parts) {
        free_cache_buffers(part);
        delete part;
    }
    c->parts.clear();
    c->part_b0.clear();
    for (auto& b : c->owned) cudaFreeAsync(b.p, c->ctx->stream);
    c->owned.clear();
}

// Image chunks of the pipelined host API: enough chunks that the copy of
// chunk k+1 in, chunk k-1 out and the kernels of chunk k overlap, few enough
// that each chunk still fills the GPU (>= 1 image, <= 8 chunks).
int host_chunks(int B) { return std::max(1, std::min(B, 8)); }

void ensure_copy_streams(gmi_ctx* ctx) {
    if (ctx->s_in == nullptr)
        GMI_CUDA(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
    if (ctx->s_out == nullptr)
        GMI_CUDA(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
}

struct EventSet {
    std::vector<cudaEvent_t> ev;
    cudaEvent_t get() {
        cudaEvent_t e;
        GMI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev.push_back(e);
        return e;
    }
    ~EventSet() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

// GMI_CTX_INJECT_FAULT: the parity harness's negative-path hook (the
// analogue of the reference's ValidationOptions::inject_fault, validate.cpp:
// 207-209): perturbs d_colors of point 0 of the call's first image on the
// device, after the backward, so a harness that misses it is broken.
__global__ void k_inject_fault(float* d_colors) { d_colors[0] += 1e-3f; }

// the backward of one (part) cache on device buffers at image offset 0
void backward_part(gmi_ctx* ctx, const gmi_cache* c, const float* upstream, float* d_colors,
                   float* d_positions, bool first_image = true) {
    {
        PhaseScope ph(ctx, 3);
        gmi_host::launch_backward(ctx, c, upstream, d_colors, d_positions);
    }
    {
        PhaseScope ph(ctx, 4);
        gmi_host::launch_special_backward(ctx, c, upstream, d_colors, d_positions);
    }
    if ((ctx->flags & GMI_CTX_INJECT_FAULT) && first_image) {
        k_inject_fault<<<1, 1, 0, ctx->stream>>>(d_colors);
        GMI_LAUNCHED(ctx);
    }
}

int do_forward(gmi_ctx* ctx, const float* pos, const float* col, int B, int N,
               int C, const gmi_config* cfg, float* image, gmi_cache* c,
               int32_t* counts, unsigned long long* d_issue = nullptr) {
    c->ctx = ctx;
    c->B = B;
    c->N = N;
    c->C = C;
    c->W = cfg->width;
    c->H = cfg->height;
    c->sigma = cfg->sigma;
    c->cutoff = cfg->cutoff_radius;
    c->fallback = cfg->fallback;
    c->pos = pos;
    c->col = col;
    c->image = image;
    c->force_generic = std::getenv("GMI_GENERIC") != nullptr;
    const size_t BN = static_cast<size_t>(B) * N;
    const size_t BHW = static_cast<size_t>(B) * c->H * c->W;
    c->wsum = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * BHW));
    // f64 weight mode beyond 6 sigma (see gmi_forward.cu)
    if (cfg->cutoff_radius > 6.0 * cfg->sigma || (ctx->flags & GMI_CTX_PRECISE)) {
        c->wsum64 = static_cast<double*>(gmi_host::cache_alloc(c, sizeof(double) * BHW));
        c->image64 = static_cast<double*>(gmi_host::cache_alloc(c, sizeof(double) * BHW * C));
    }
    c->special_cap = static_cast<int>(std::min<size_t>(BHW, size_t(1) << 22));
    c->special = static_cast<Special*>(gmi_host::cache_alloc(c, sizeof(Special) * c->special_cap));
    c->special_count_d = static_cast<int32_t*>(gmi_host::cache_alloc(c, sizeof(int32_t)));
    if (d_issue == nullptr) {
        ensure_issue(ctx, B);
        d_issue = ctx->d_issue;
    }
    host_trace("fwd: allocs");
    {
        PhaseScope ph(ctx, 0);
        // fast gather: unordered cells and the 32-byte record layout;
        // otherwise index-ordered cells in SoA (the generic gather's order)
        const bool fast = gmi_host::gather_fast_ok(c);
        // C > 4 (wide gather): records and colours in index-ordered cells
        c->sort_cells = !fast || C > 4;
        if (fast) {
            c->rec = static_cast<float4*>(gmi_host::cache_alloc(c, sizeof(float4) * 2 * BN));
            if (C > 4)
                c->ccol = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * BN * C));
        } else {
            c->sx = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * BN));
            c->sy = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * BN));
            c->sidx = static_cast<int32_t*>(gmi_host::cache_alloc(c, sizeof(int32_t) * BN));
            c->scol = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * BN * C));
        }
        gmi_host::bin_points(ctx, c, pos, col, frame_cells(cfg), true, nullptr, d_issue);
    }
    {
        PhaseScope ph(ctx, 1);
        gmi_host::launch_forward(ctx, c, image, counts);
    }
    {
        PhaseScope ph(ctx, 2);
        gmi_host::launch_special_forward(ctx, c, image, counts);
    }
    host_trace("fwd: gather+special launched");
    if ((ctx->flags & GMI_CTX_ASYNC_ERRORS) && counts == nullptr) {
        // no host check below: a fallback list overflow becomes a pending
        // error reported by gmi_ctx_synchronize
        k_async_check<<<1, 32, 0, ctx->stream>>>(c->special_count_d, c->special_cap, d_issue, B,
                                                static_cast<int>(d_issue - ctx->d_issue),
                                                ctx->collect_now ? nullptr : ctx->d_pending);
        GMI_LAUNCHED(ctx);
    }
    if (!(ctx->flags & GMI_CTX_ASYNC_ERRORS) || counts != nullptr) {
        int32_t nspec = 0;
        GMI_CUDA(cudaMemcpyAsync(&nspec, c->special_count_d, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        const int rc = collect_issue(ctx, B);
        if (rc != GMI_OK) return rc;
        if (nspec > c->special_cap)
            return fail(GMI_ERR_OUT_OF_MEMORY,
                        "more than " + std::to_string(c->special_cap) + " fallback pixels");
        c->special_count = nspec;
    }
    return GMI_OK;
}

int backward_checks(const gmi_cache* c, int B, int N, int C, const gmi_config* cfg) {
    // engine.cpp:243-250 (exact ==, including sigma and cutoff)
    if (c == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "cache is null");
    if (c->N != N || c->C != C || c->B != B || c->W != cfg->width || c->H != cfg->height ||
        c->sigma != cfg->sigma || c->cutoff != cfg->cutoff_radius ||
        c->fallback != cfg->fallback)
        return fail(GMI_ERR_CACHE_MISMATCH, "forward cache does not match the given inputs");
    return GMI_OK;
}

int do_backward(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                float* d_colors, float* d_positions) {
    if (c->parts.empty()) {
        backward_part(ctx, c, upstream, d_colors, d_positions);
    } else {
        const size_t hwc = static_cast<size_t>(c->H) * c->W * c->C;
        for (size_t k = 0; k < c->parts.size(); ++k) {
            const size_t b0 = c->part_b0[k];
            backward_part(ctx, c->parts[k], upstream + b0 * hwc,
                          d_colors + b0 * c->N * c->C, d_positions + b0 * c->N * 2, k == 0);
        }
    }
    if (!(ctx->flags & GMI_CTX_ASYNC_ERRORS)) GMI_CUDA(cudaStreamSynchronize(ctx->stream));
    return GMI_OK;
}

// ---- optimize_points (optimize.cpp:12-98) ----
constexpr int kLossThreads = 256;

// l1_loss_and_grad (optimize.cpp:12-28) per image: upstream = sign(pred -
// target) / (H W C) (sign(0) = 0) and per-block f64 partial sums of |d|,
// reduced in block order by k_loss_finalize (deterministic).
__global__ void k_l1_loss_grad(const float* __restrict__ pred, const float* __restrict__ target,
                               float* __restrict__ up, size_t per_img, double inv,
                               double* __restrict__ partial) {
    __shared__ double red[kLossThreads / 32];
    const int b = blockIdx.y;
    const size_t base = static_cast<size_t>(b) * per_img;
    double s = 0.0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < per_img;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(pred[base + k]) - static_cast<double>(target[base + k]);
        s += fabs(d);
        up[base + k] = static_cast<float>(d > 0.0 ? inv : (d < 0.0 ? -inv : 0.0));
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kLossThreads / 32; ++w) t += red[w];
        partial[static_cast<size_t>(b) * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void k_loss_finalize(const double* __restrict__ partial, int nblk, double inv,
                                double* __restrict__ loss, int stride, int step, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double t = 0.0;
    for (int k = 0; k < nblk; ++k) t += partial[static_cast<size_t>(b) * nblk + k];
    loss[static_cast<size_t>(b) * stride + step] = t * inv;
}

// descent update (optimize.cpp:80-96), in f64 then rounded to the fp32 state
__global__ void k_descent(float* __restrict__ pos, float* __restrict__ col,
                          const float* __restrict__ d_pos, const float* __restrict__ d_col,
                          size_t n_pts, int C, double lr, uint32_t flags) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n_pts) return;
    if (flags & GMI_OPT_POSITIONS) {
        pos[2 * i] = static_cast<float>(static_cast<double>(pos[2 * i]) - lr * d_pos[2 * i]);
        pos[2 * i + 1] =
            static_cast<float>(static_cast<double>(pos[2 * i + 1]) - lr * d_pos[2 * i + 1]);
    }
    if (flags & GMI_OPT_COLORS) {
        for (int c = 0; c < C; ++c) {
            const double v = static_cast<double>(col[i * C + c]) - lr * d_col[i * C + c];
            col[i * C + c] = static_cast<float>(fmin(fmax(v, 0.0), 1.0));
        }
    }
}

int do_optimize(gmi_ctx* ctx, float* pos, float* col, int B, int N, int C,
                const gmi_config* cfg, const float* target, int steps, double lr,
                uint32_t flags, double* loss_curve) {
    const size_t hwc = static_cast<size_t>(cfg->height) * cfg->width * C;
    const size_t BN = static_cast<size_t>(B) * N;
    float* img = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * B * hwc));
    float* up = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * B * hwc));
    float* dcol = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * BN * C));
    float* dpos = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * BN * 2));
    const int nblk = static_cast<int>(std::min<size_t>((hwc + kLossThreads - 1) / kLossThreads,
                                                       std::max(1, 2 * ctx->num_sms / B + 1)));
    double* partial = static_cast<double*>(gmi_host::dalloc(ctx, sizeof(double) * B * nblk));
    double* loss = static_cast<double*>(gmi_host::dalloc(ctx, sizeof(double) * B * (steps + 1)));
    const double inv = 1.0 / static_cast<double>(hwc);
    ensure_issue(ctx, B);
    const uint32_t saved = ctx->flags;
    ctx->flags |= GMI_CTX_ASYNC_ERRORS;
    int rc = GMI_OK;
    try {
        for (int step = 0; step <= steps && rc == GMI_OK; ++step) {
            gmi_cache c;
            c.ctx = ctx;
            rc = do_forward(ctx, pos, col, B, N, C, cfg, img, &c, nullptr);
            if (rc == GMI_OK) {
                k_l1_loss_grad<<<dim3(nblk, B), kLossThreads, 0, ctx->stream>>>(img, target, up, hwc, inv,
                                                                                partial);
                GMI_LAUNCHED(ctx);
                k_loss_finalize<<<(B + 63) / 64, 64, 0, ctx->stream>>>(partial, nblk, inv, loss, steps + 1,
                                                                       step, B);
                GMI_LAUNCHED(ctx);
                if (step < steps) {
                    backward_part(ctx, &c, up, dcol, dpos);
                    k_descent<<<static_cast<unsigned>((BN + 255) / 256), 256, 0, ctx->stream>>>(
                        pos, col, dpos, dcol, BN, C, lr, flags);
                    GMI_LAUNCHED(ctx);
                }
            }
            free_cache_buffers(&c);
        }
    } catch (...) {
        ctx->flags = saved;
        throw;
    }
    ctx->flags = saved;
    if (rc == GMI_OK && loss_curve != nullptr)
        GMI_CUDA(cudaMemcpyAsync(loss_curve, loss, sizeof(double) * B * (steps + 1),
                                 cudaMemcpyDeviceToHost, ctx->stream));
    for (void* q : {static_cast<void*>(img), static_cast<void*>(up), static_cast<void*>(dcol),
                    static_cast<void*>(dpos), static_cast<void*>(partial), static_cast<void*>(loss)})
        gmi_host::dfree(ctx, q);
    if (rc == GMI_OK) rc = collect_issue(ctx, B);  // synchronises
    return rc;
}

// ---- run_benchmark's GMM branch (benchmark.cpp:88-107) ----
// grid_subsample colours (imaging.cpp:306-341): thread per (block, channel),
// the f64 sum in the reference's row-major order times 1/area.
__global__ void k_block_mean(const float* __restrict__ img, int W, int H, int C, int f, int lw,
                             int lh, float* __restrict__ low) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= lw * lh * C) return;
    const int ch = k % C, blk = k / C, bc = blk % lw, br = blk / lw;
    const int r0 = br * f, r1 = min(H, r0 + f), c0 = bc * f, c1 = min(W, c0 + f);
    const double inv_area = 1.0 / static_cast<double>((r1 - r0) * (c1 - c0));
    double sum = 0.0;
    for (int r = r0; r < r1; ++r)
        for (int c = c0; c < c1; ++c)
            sum = __dadd_rn(sum, static_cast<double>(img[(static_cast<size_t>(r) * W + c) * C + ch]));
    low[k] = static_cast<float>(__dmul_rn(sum, inv_area));
}

// point_set_from_lowres (benchmark.cpp:24-39): block centres, exact in fp32.
__global__ void k_block_centres(float* __restrict__ pos, int lw, int lh, int f) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= lw * lh) return;
    const double half = (f - 1) / 2.0;
    pos[2 * k] = static_cast<float>((k % lw) * static_cast<double>(f) + half);
    pos[2 * k + 1] = static_cast<float>((k / lw) * static_cast<double>(f) + half);
}

// l1_metric (imaging.cpp:376-386): per-block f64 partial sums of |a - b|,
// summed in block order by k_l1_finalize (deterministic).
__global__ void k_l1_partial(const float* __restrict__ a, const float* __restrict__ b, size_t n,
                             double* __restrict__ partial) {
    __shared__ double red[kLossThreads / 32];
    double s = 0.0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x)
        s += fabs(static_cast<double>(a[k]) - static_cast<double>(b[k]));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kLossThreads / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

__global__ void k_l1_finalize(const double* __restrict__ partial, int nblk, double inv,
                              double* __restrict__ out) {
    double t = 0.0;
    for (int k = 0; k < nblk; ++k) t += partial[k];
    *out = t * inv;
}

}  // namespace

void host_trace(const char* what) {
    static const bool on = std::getenv("GMI_TRACE") != nullptr;
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gmi] %-28s %9.1f us\n", what,
                 std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
}

namespace gmi_host {

void* dalloc(gmi_ctx* ctx, size_t bytes) {
    void* p = nullptr;
    GMI_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), ctx->stream));
    return p;
}

void dfree(gmi_ctx* ctx, void* p) {
    if (p) cudaFreeAsync(p, ctx->stream);
}

int32_t* upload_table(gmi_ctx* ctx, int slot, const std::vector<int32_t>& v) {
    int32_t* d = static_cast<int32_t*>(scratch(ctx, slot, sizeof(int32_t) * v.size()));
    if (ctx->ws_table_ptr[slot] != d || ctx->ws_table[slot] != v) {
        GMI_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice,
                                 ctx->stream));
        ctx->ws_table[slot] = v;
        ctx->ws_table_ptr[slot] = d;
    }
    return d;
}

void* scratch(gmi_ctx* ctx, int slot, size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    if (ctx->ws_cap[slot] < bytes) {
        if (ctx->ws_ptr[slot]) cudaFreeAsync(ctx->ws_ptr[slot], ctx->stream);
        ctx->ws_table_ptr[slot] = nullptr;  // an uploaded table must be re-sent
        const size_t cap = bytes + bytes / 4;  // headroom for slowly growing sizes
        GMI_CUDA(cudaMallocAsync(&ctx->ws_ptr[slot], cap, ctx->stream));
        ctx->ws_cap[slot] = cap;
    }
    return ctx->ws_ptr[slot];
}

void* cache_alloc(gmi_cache* c, size_t bytes) {
    void* p = dalloc(c->ctx, bytes);
    c->owned.push_back({p, bytes});
    return p;
}

}  // namespace gmi_host

extern "C" {

const char* gmi_last_error(void) { return g_last_error.c_str(); }

const char* gmi_version(void) { return "gmi_b200 0.1.0 (sm_100a)"; }

const char* gmi_error_name(int code) {
    // error_code_name (core.cpp:7-25), offset by one; B200-side codes after
    switch (code) {
        case GMI_OK: return "Ok";
        case GMI_ERR_NON_FINITE_VALUE: return "NonFiniteValue";
        case GMI_ERR_COLOR_OUT_OF_RANGE: return "ColorOutOfRange";
        case GMI_ERR_EMPTY_POINT_SET: return "EmptyPointSet";
        case GMI_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
        case GMI_ERR_INVALID_CELL_SIZE: return "InvalidCellSize";
        case GMI_ERR_CONFIG_INVALID: return "ConfigInvalid";
        case GMI_ERR_CACHE_MISMATCH: return "CacheMismatch";
        case GMI_ERR_INVALID_DIMENSIONS: return "InvalidDimensions";
        case GMI_ERR_INVALID_FACTOR: return "InvalidFactor";
        case GMI_ERR_INVALID_COUNT: return "InvalidCount";
        case GMI_ERR_UNSUPPORTED_FORMAT: return "UnsupportedFormat";
        case GMI_ERR_CORRUPT_FILE: return "CorruptFile";
        case GMI_ERR_EMPTY_LOG: return "EmptyLog";
        case GMI_ERR_IO_ERROR: return "IoError";
        case GMI_ERR_CUDA: return "CudaError";
        case GMI_ERR_INVALID_ARGUMENT: return "InvalidArgument";
        case GMI_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    }
    return "UnknownError";
}

double gmi_default_cutoff(double sigma) { return 3.0 * sigma; }

double gmi_gaussian_weight(double qx, double qy, double mux, double muy, double sigma) {
    const double dx = qx - mux;
    const double dy = qy - muy;
    return std::exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
}

int gmi_ctx_create(int device, gmi_ctx** out) {
    return guarded([&]() -> int {
        if (out == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "out is null");
        int n = 0;
        GMI_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n)
            return fail(GMI_ERR_INVALID_ARGUMENT, "no CUDA device " + std::to_string(device));
        GMI_CUDA(cudaSetDevice(device));
        auto* ctx = new gmi_ctx();
        ctx->device = device;
        GMI_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        GMI_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
        GMI_CUDA(cudaMalloc(&ctx->d_pending, 2 * sizeof(unsigned long long)));
        GMI_CUDA(cudaMemset(ctx->d_pending, 0xFF, 2 * sizeof(unsigned long long)));
        // keep freed stream-ordered memory cached between calls
        cudaMemPool_t pool;
        GMI_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thresh = UINT64_MAX;
        GMI_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
        *out = ctx;
        return GMI_OK;
    });
}

int gmi_ctx_destroy(gmi_ctx* ctx) {
    if (ctx == nullptr) return GMI_OK;
    return guarded([&]() -> int {
        // caches still alive keep the context (their stream and device) until
        // the last of them is freed
        ctx_release(ctx);
        return GMI_OK;
    });
}

int gmi_ctx_set_stream(gmi_ctx* ctx, void* stream) {
    return guarded([&]() -> int {
        if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        if (stream == nullptr) {
            if (!ctx->own_stream) {
                GMI_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
                ctx->own_stream = true;
            }
            return GMI_OK;
        }
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        ctx->stream = static_cast<cudaStream_t>(stream);
        ctx->own_stream = false;
        return GMI_OK;
    });
}

void* gmi_ctx_stream(const gmi_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int gmi_ctx_set_flags(gmi_ctx* ctx, uint32_t flags) {
    if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
    ctx->flags = flags;
    return GMI_OK;
}

int gmi_ctx_synchronize(gmi_ctx* ctx) {
    return guarded([&]() -> int {
        if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
        GMI_CUDA(cudaSetDevice(ctx->device));
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        // host-buffer downloads queued by asynchronous host-API calls
        if (ctx->s_in) GMI_CUDA(cudaStreamSynchronize(ctx->s_in));
        if (ctx->s_out) GMI_CUDA(cudaStreamSynchronize(ctx->s_out));
        return collect_pending(ctx);
    });
}

int gmi_ctx_join_host_copies(gmi_ctx* ctx) {
    return guarded([&]() -> int {
        if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
        GMI_CUDA(cudaSetDevice(ctx->device));
        join_copy_streams(ctx);
        return GMI_OK;
    });
}

uint64_t gmi_ctx_launch_count(const gmi_ctx* ctx) { return ctx ? ctx->launches : 0; }

int gmi_ctx_set_profiling(gmi_ctx* ctx, int on) {
    if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
    ctx->profiling = on != 0;
    return GMI_OK;
}

int gmi_ctx_phase_times(gmi_ctx* ctx, double* ms, uint64_t* calls, int reset) {
    return guarded([&]() -> int {
        if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
        GMI_CUDA(cudaSetDevice(ctx->device));
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        for (auto& m : ctx->marks) {
            float t = 0.f;
            GMI_CUDA(cudaEventElapsedTime(&t, m.start, m.stop));
            ctx->phase_ms[m.phase] += t;
            ctx->phase_calls[m.phase] += 1;
            cudaEventDestroy(m.start);
            cudaEventDestroy(m.stop);
        }
        ctx->marks.clear();
        for (int k = 0; k < GMI_NUM_PHASES; ++k) {
            if (ms) ms[k] = ctx->phase_ms[k];
            if (calls) calls[k] = ctx->phase_calls[k];
            if (reset) {
                ctx->phase_ms[k] = 0;
                ctx->phase_calls[k] = 0;
            }
        }
        return GMI_OK;
    });
}

int gmi_forward(gmi_ctx* ctx, const float* positions, const float* colors, int32_t batch,
                int32_t num_points, int32_t channels, const gmi_config* cfg, float* image,
                gmi_cache** cache_out) {
    return guarded([&]() -> int {
        if (ctx == nullptr || cache_out == nullptr || image == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        int rc = check_points(positions, colors, batch, num_points, channels);
        if (rc) return rc;
        rc = check_config(cfg);
        if (rc) return rc;
        GMI_CUDA(cudaSetDevice(ctx->device));
        auto* c = new gmi_cache();
        c->ctx = ctx;
        c->holds_ctx = true;
        ctx_retain(ctx);
        try {
            rc = do_forward(ctx, positions, colors, batch, num_points, channels, cfg, image, c,
                            nullptr);
        } catch (...) {
            free_cache_buffers(c);
            delete c;
            ctx_release(ctx);
            throw;
        }
        if (rc != GMI_OK) {
            free_cache_buffers(c);
            delete c;
            ctx_release(ctx);
            return rc;
        }
        *cache_out = c;
        return GMI_OK;
    });
}

int gmi_backward(gmi_ctx* ctx, const float* positions, const float* colors, int32_t batch,
                 int32_t num_points, int32_t channels, const gmi_config* cfg,
                 const gmi_cache* cache, const float* upstream, float* d_colors,
                 float* d_positions) {
    return guarded([&]() -> int {
        if (ctx == nullptr || upstream == nullptr || d_colors == nullptr || d_positions == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        int rc = check_points(positions, colors, batch, num_points, channels);
        if (rc) return rc;
        rc = check_config(cfg);
        if (rc) return rc;
        rc = backward_checks(cache, batch, num_points, channels, cfg);
        if (rc) return rc;
        GMI_CUDA(cudaSetDevice(ctx->device));
        return do_backward(ctx, cache, upstream, d_colors, d_positions);
    });
}

// gmi_forward_host on PAGEABLE host buffers: inputs staged up through the
// pinned slots, the whole batch in one device forward, the image staged
// down; complete on return.
int forward_host_pageable(gmi_ctx* ctx, const float* positions, const float* colors, int batch,
                          int num_points, int channels, const gmi_config* cfg, float* image,
                          gmi_cache** cache_out) {
    auto* c = new gmi_cache();
    c->ctx = ctx;
    c->holds_ctx = true;
    ctx_retain(ctx);
    const size_t N = num_points, C = channels;
    const size_t hwc = static_cast<size_t>(cfg->height) * cfg->width * C;
    int rc = GMI_OK;
    try {
        float* dpos = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * N * 2));
        float* dcol = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * N * C));
        float* dimg = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * hwc));
        h2d_staged(ctx, dpos, positions, sizeof(float) * batch * N * 2, ctx->stream);
        h2d_staged(ctx, dcol, colors, sizeof(float) * batch * N * C, ctx->stream);
        rc = do_forward(ctx, dpos, dcol, batch, num_points, channels, cfg, dimg, c, nullptr);
        if (rc == GMI_OK) d2h_staged(ctx, image, dimg, sizeof(float) * batch * hwc, ctx->stream);
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);
        free_cache_buffers(c);
        delete c;
        ctx_release(ctx);
        throw;
    }
    if (rc != GMI_OK) {
        free_cache_buffers(c);
        delete c;
        ctx_release(ctx);
        return rc;
    }
    *cache_out = c;
    return GMI_OK;
}

int gmi_forward_host(gmi_ctx* ctx, const float* positions, const float* colors, int32_t batch,
                     int32_t num_points, int32_t channels, const gmi_config* cfg, float* image,
                     gmi_cache** cache_out) {
    // Pipelined over image chunks: H2D of chunk k+1 (s_in), the forward of
    // chunk k (ctx stream) and the D2H of chunk k-1 (s_out) overlap.  The
    // returned cache is composite (one part cache per chunk).
    return guarded([&]() -> int {
        if (ctx == nullptr || cache_out == nullptr || image == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        int rc = check_points(positions, colors, batch, num_points, channels);
        if (rc) return rc;
        rc = check_config(cfg);
        if (rc) return rc;
        GMI_CUDA(cudaSetDevice(ctx->device));
        if (is_pageable(positions) || is_pageable(colors) || is_pageable(image))
            return forward_host_pageable(ctx, positions, colors, batch, num_points, channels, cfg,
                                         image, cache_out);
        ensure_copy_streams(ctx);
        ensure_issue(ctx, batch);
        auto* c = new gmi_cache();
        c->ctx = ctx;
        c->holds_ctx = true;
        ctx_retain(ctx);
        c->B = batch;
        c->N = num_points;
        c->C = channels;
        c->W = cfg->width;
        c->H = cfg->height;
        c->sigma = cfg->sigma;
        c->cutoff = cfg->cutoff_radius;
        c->fallback = cfg->fallback;
        const size_t N = num_points, C = channels;
        const size_t hwc = static_cast<size_t>(cfg->height) * cfg->width * C;
        const uint32_t saved = ctx->flags;
        try {
            EventSet E;
            float* dpos = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * N * 2));
            float* dcol = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * N * C));
            float* dimg = static_cast<float*>(gmi_host::cache_alloc(c, sizeof(float) * batch * hwc));
            c->pos = dpos;
            c->col = dcol;
            c->image = dimg;
            cudaEvent_t alloc = E.get();
            GMI_CUDA(cudaEventRecord(alloc, ctx->stream));
            GMI_CUDA(cudaStreamWaitEvent(ctx->s_in, alloc, 0));
            const int nk = host_chunks(batch);
            std::vector<int> b0(nk + 1);
            for (int k = 0; k <= nk; ++k) b0[k] = static_cast<int>((static_cast<int64_t>(batch) * k) / nk);
            std::vector<cudaEvent_t> in(nk);
            for (int k = 0; k < nk; ++k) {
                const size_t o = b0[k], n = b0[k + 1] - b0[k];
                GMI_CUDA(cudaMemcpyAsync(dpos + o * N * 2, positions + o * N * 2, sizeof(float) * n * N * 2,
                                         cudaMemcpyHostToDevice, ctx->s_in));
                GMI_CUDA(cudaMemcpyAsync(dcol + o * N * C, colors + o * N * C, sizeof(float) * n * N * C,
                                         cudaMemcpyHostToDevice, ctx->s_in));
                in[k] = E.get();
                GMI_CUDA(cudaEventRecord(in[k], ctx->s_in));
            }
            ctx->flags |= GMI_CTX_ASYNC_ERRORS;
            // a synchronous call collects its parts' errors itself below
            ctx->collect_now = (saved & GMI_CTX_ASYNC_ERRORS) == 0;
            for (int k = 0; k < nk; ++k) {
                const size_t o = b0[k];
                const int n = b0[k + 1] - b0[k];
                GMI_CUDA(cudaStreamWaitEvent(ctx->stream, in[k], 0));
                auto* part = new gmi_cache();
                part->ctx = ctx;
                c->parts.push_back(part);
                c->part_b0.push_back(static_cast<int>(o));
                rc = do_forward(ctx, dpos + o * N * 2, dcol + o * N * C, n, num_points, channels, cfg,
                                dimg + o * hwc, part, nullptr, ctx->d_issue + o);
                if (rc != GMI_OK) break;
                cudaEvent_t done = E.get();
                GMI_CUDA(cudaEventRecord(done, ctx->stream));
                GMI_CUDA(cudaStreamWaitEvent(ctx->s_out, done, 0));
                GMI_CUDA(cudaMemcpyAsync(image + o * hwc, dimg + o * hwc, sizeof(float) * n * hwc,
                                         cudaMemcpyDeviceToHost, ctx->s_out));
            }
            ctx->flags = saved;
            ctx->collect_now = false;
            GMI_CUDA(cudaEventCreateWithFlags(&c->d2h_done, cudaEventDisableTiming));
            GMI_CUDA(cudaEventRecord(c->d2h_done, ctx->s_out));
            // GMI_CTX_ASYNC_ERRORS: return with the image download still
            // queued on the copy stream (complete after gmi_ctx_synchronize),
            // so a following gmi_backward_host uploads its upstream while
            // this image comes down (PCIe is full duplex)
            const bool async = (saved & GMI_CTX_ASYNC_ERRORS) != 0;
            if (!async) {
                GMI_CUDA(cudaStreamSynchronize(ctx->s_out));
                GMI_CUDA(cudaStreamSynchronize(ctx->s_in));
            }
            if (rc == GMI_OK && !async) rc = collect_issue(ctx, batch);
            if (rc == GMI_OK && !async) {
                for (gmi_cache* part : c->parts) {
                    int32_t nspec = 0;
                    GMI_CUDA(cudaMemcpyAsync(&nspec, part->special_count_d, sizeof(int32_t),
                                             cudaMemcpyDeviceToHost, ctx->stream));
                    GMI_CUDA(cudaStreamSynchronize(ctx->stream));
                    if (nspec > part->special_cap) {
                        rc = fail(GMI_ERR_OUT_OF_MEMORY, "more than " + std::to_string(part->special_cap) +
                                                             " fallback pixels");
                        break;
                    }
                    part->special_count = nspec;
                }
            }
        } catch (...) {
            ctx->flags = saved;
            ctx->collect_now = false;
            cudaStreamSynchronize(ctx->s_in);
            cudaStreamSynchronize(ctx->s_out);
            free_cache_buffers(c);
            delete c;
            ctx_release(ctx);
            throw;
        }
        if (rc != GMI_OK) {
            free_cache_buffers(c);
            delete c;
            ctx_release(ctx);
            return rc;
        }
        *cache_out = c;
        return GMI_OK;
    });
}

int gmi_backward_host(gmi_ctx* ctx, const float* positions, const float* colors, int32_t batch,
                      int32_t num_points, int32_t channels, const gmi_config* cfg,
                      const gmi_cache* cache, const float* upstream, float* d_colors,
                      float* d_positions) {
    // Pipelined over the forward cache's image chunks: H2D of upstream chunk
    // k+1, the backward of chunk k and the D2H of chunk k-1's gradients overlap.
    return guarded([&]() -> int {
        if (ctx == nullptr || upstream == nullptr || d_colors == nullptr || d_positions == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        int rc = check_points(positions, colors, batch, num_points, channels);
        if (rc) return rc;
        rc = check_config(cfg);
        if (rc) return rc;
        rc = backward_checks(cache, batch, num_points, channels, cfg);
        if (rc) return rc;
        GMI_CUDA(cudaSetDevice(ctx->device));
        const size_t N = num_points, C = channels;
        const size_t hwc = static_cast<size_t>(cfg->height) * cfg->width * C;
        if (is_pageable(upstream) || is_pageable(d_colors) || is_pageable(d_positions)) {
            // pageable buffers: staged through the pinned slots (the result
            // is complete on return)
            float* dup = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * hwc));
            float* dc = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * N * C));
            float* dp = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * N * 2));
            h2d_staged(ctx, dup, upstream, sizeof(float) * batch * hwc, ctx->stream);
            do_backward(ctx, cache, dup, dc, dp);
            d2h_staged(ctx, d_colors, dc, sizeof(float) * batch * N * C, ctx->stream);
            d2h_staged(ctx, d_positions, dp, sizeof(float) * batch * N * 2, ctx->stream);
            gmi_host::dfree(ctx, dup);
            gmi_host::dfree(ctx, dc);
            gmi_host::dfree(ctx, dp);
            return GMI_OK;
        }
        ensure_copy_streams(ctx);
        std::vector<const gmi_cache*> parts;
        std::vector<int> b0;
        if (cache->parts.empty()) {
            parts.push_back(cache);
            b0.push_back(0);
        } else {
            for (size_t k = 0; k < cache->parts.size(); ++k) {
                parts.push_back(cache->parts[k]);
                b0.push_back(cache->part_b0[k]);
            }
        }
        EventSet E;
        float* dup = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * hwc));
        float* dc = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * N * C));
        float* dp = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * batch * N * 2));
        cudaEvent_t alloc = E.get();
        GMI_CUDA(cudaEventRecord(alloc, ctx->stream));
        GMI_CUDA(cudaStreamWaitEvent(ctx->s_in, alloc, 0));
        std::vector<cudaEvent_t> in(parts.size());
        for (size_t k = 0; k < parts.size(); ++k) {
            const size_t o = b0[k], n = parts[k]->B;
            GMI_CUDA(cudaMemcpyAsync(dup + o * hwc, upstream + o * hwc, sizeof(float) * n * hwc,
                                     cudaMemcpyHostToDevice, ctx->s_in));
            in[k] = E.get();
            GMI_CUDA(cudaEventRecord(in[k], ctx->s_in));
        }
        for (size_t k = 0; k < parts.size(); ++k) {
            const size_t o = b0[k], n = parts[k]->B;
            GMI_CUDA(cudaStreamWaitEvent(ctx->stream, in[k], 0));
            backward_part(ctx, parts[k], dup + o * hwc, dc + o * N * C, dp + o * N * 2, k == 0);
            cudaEvent_t done = E.get();
            GMI_CUDA(cudaEventRecord(done, ctx->stream));
            GMI_CUDA(cudaStreamWaitEvent(ctx->s_out, done, 0));
            GMI_CUDA(cudaMemcpyAsync(d_colors + o * N * C, dc + o * N * C, sizeof(float) * n * N * C,
                                     cudaMemcpyDeviceToHost, ctx->s_out));
            GMI_CUDA(cudaMemcpyAsync(d_positions + o * N * 2, dp + o * N * 2, sizeof(float) * n * N * 2,
                                     cudaMemcpyDeviceToHost, ctx->s_out));
        }
        // staging buffers return to the pool behind the downloads (stream-
        // ordered on the copy stream, which follows the last chunk's kernels),
        // so the ctx stream — and the next call's uploads — need not wait
        GMI_CUDA(cudaFreeAsync(dup, ctx->s_out));
        GMI_CUDA(cudaFreeAsync(dc, ctx->s_out));
        GMI_CUDA(cudaFreeAsync(dp, ctx->s_out));
        // GMI_CTX_ASYNC_ERRORS: gradients complete after gmi_ctx_synchronize
        if (!(ctx->flags & GMI_CTX_ASYNC_ERRORS)) {
            GMI_CUDA(cudaStreamSynchronize(ctx->s_out));
            GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        return GMI_OK;
    });
}

void gmi_cache_free(gmi_cache* c) {
    if (c == nullptr) return;
    gmi_ctx* ctx = c->ctx;
    cudaSetDevice(ctx->device);
    free_cache_buffers(c);
    const bool held = c->holds_ctx;
    delete c;
    if (held) ctx_release(ctx);
}

int gmi_cache_shape(const gmi_cache* c, int32_t* batch, int32_t* num_points, int32_t* channels,
                    int32_t* width, int32_t* height) {
    if (c == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "cache is null");
    if (batch) *batch = c->B;
    if (num_points) *num_points = c->N;
    if (channels) *channels = c->C;
    if (width) *width = c->W;
    if (height) *height = c->H;
    return GMI_OK;
}

static int read_special(const gmi_cache* c, std::vector<Special>& sp) {
    GMI_CUDA(cudaSetDevice(c->ctx->device));
    int32_t n = 0;
    GMI_CUDA(cudaMemcpyAsync(&n, c->special_count_d, sizeof(int32_t), cudaMemcpyDeviceToHost,
                             c->ctx->stream));
    GMI_CUDA(cudaStreamSynchronize(c->ctx->stream));
    n = std::min(n, c->special_cap);
    sp.resize(n);
    if (n > 0) {
        GMI_CUDA(cudaMemcpyAsync(sp.data(), c->special, sizeof(Special) * n,
                                 cudaMemcpyDeviceToHost, c->ctx->stream));
        GMI_CUDA(cudaStreamSynchronize(c->ctx->stream));
    }
    return GMI_OK;
}

int gmi_cache_fallback_count(const gmi_cache* c, int64_t* out) {
    if (c != nullptr && out != nullptr && !c->parts.empty()) {
        for (size_t k = 0; k < c->parts.size(); ++k) {
            const int rc = gmi_cache_fallback_count(c->parts[k], out + c->part_b0[k]);
            if (rc != GMI_OK) return rc;
        }
        return GMI_OK;
    }
    return guarded([&]() -> int {
        if (c == nullptr || out == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        std::vector<Special> sp;
        read_special(c, sp);
        for (int b = 0; b < c->B; ++b) out[b] = 0;
        for (const auto& s : sp)
            if (s.kind == 1) out[s.b]++;
        return GMI_OK;
    });
}

int gmi_cache_copy_pixels(const gmi_cache* c, float* normalizer, uint8_t* fallback_flag,
                          int32_t* nearest_index) {
    if (c != nullptr && !c->parts.empty()) {
        const size_t hw = static_cast<size_t>(c->H) * c->W;
        for (size_t k = 0; k < c->parts.size(); ++k) {
            const size_t o = static_cast<size_t>(c->part_b0[k]) * hw;
            const int rc = gmi_cache_copy_pixels(c->parts[k], normalizer ? normalizer + o : nullptr,
                                                 fallback_flag ? fallback_flag + o : nullptr,
                                                 nearest_index ? nearest_index + o : nullptr);
            if (rc != GMI_OK) return rc;
        }
        return GMI_OK;
    }
    return guarded([&]() -> int {
        if (c == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "cache is null");
        const size_t BHW = static_cast<size_t>(c->B) * c->H * c->W;
        std::vector<Special> sp;
        read_special(c, sp);
        if (normalizer && c->wsum64 != nullptr) {
            // f64 weight mode: the normaliser lives in f64 (may underflow fp32)
            std::vector<double> w64(BHW);
            GMI_CUDA(cudaMemcpyAsync(w64.data(), c->wsum64, sizeof(double) * BHW,
                                     cudaMemcpyDeviceToHost, c->ctx->stream));
            GMI_CUDA(cudaStreamSynchronize(c->ctx->stream));
            for (size_t k = 0; k < BHW; ++k) normalizer[k] = static_cast<float>(w64[k]);
        } else if (normalizer) {
            GMI_CUDA(cudaMemcpyAsync(normalizer, c->wsum, sizeof(float) * BHW,
                                     cudaMemcpyDeviceToHost, c->ctx->stream));
            GMI_CUDA(cudaStreamSynchronize(c->ctx->stream));
        }
        if (fallback_flag) std::memset(fallback_flag, 0, BHW);
        if (nearest_index)
            for (size_t k = 0; k < BHW; ++k) nearest_index[k] = -1;
        for (const auto& s : sp) {
            const size_t k = static_cast<size_t>(s.b) * c->H * c->W + s.pix;
            if (s.kind == 1) {
                if (fallback_flag) fallback_flag[k] = 1;
                if (nearest_index) nearest_index[k] = s.nearest;
            }
        }
        return GMI_OK;
    });
}

int gmi_forward_counts(gmi_ctx* ctx, const gmi_cache* cache, int32_t* counts) {
    return guarded([&]() -> int {
        if (ctx == nullptr || cache == nullptr || counts == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        GMI_CUDA(cudaSetDevice(ctx->device));
        // Re-run the same forward pipeline with the counting instantiation of
        // the gather kernel into scratch image/cache buffers.
        const size_t BHW = static_cast<size_t>(cache->B) * cache->H * cache->W;
        gmi_config cfg{cache->sigma, cache->cutoff, cache->fallback, cache->W, cache->H};
        gmi_cache tmp;
        tmp.ctx = ctx;
        float* img = static_cast<float*>(gmi_host::cache_alloc(&tmp, sizeof(float) * BHW * cache->C));
        int32_t* dcounts = static_cast<int32_t*>(gmi_host::cache_alloc(&tmp, sizeof(int32_t) * BHW));
        int rc = do_forward(ctx, cache->pos, cache->col, cache->B, cache->N, cache->C, &cfg, img,
                            &tmp, dcounts);
        if (rc == GMI_OK) {
            GMI_CUDA(cudaMemcpyAsync(counts, dcounts, sizeof(int32_t) * BHW, cudaMemcpyDeviceToHost,
                                     ctx->stream));
            GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        free_cache_buffers(&tmp);
        return rc;
    });
}

int gmi_bin_grid(gmi_ctx* ctx, const float* positions, int32_t batch, int32_t num_points,
                 double cell_size, double* origin, int32_t* n_cols, int32_t* n_rows,
                 int32_t* bin_start, int32_t* point_index) {
    return guarded([&]() -> int {
        if (ctx == nullptr || positions == nullptr || origin == nullptr || n_cols == nullptr ||
            n_rows == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        if (batch < 1) return fail(GMI_ERR_INVALID_ARGUMENT, "batch must be >= 1");
        if (num_points <= 0) return fail(GMI_ERR_EMPTY_POINT_SET, "point set is empty");
        // bin_grid.cpp:40-43
        if (!std::isfinite(cell_size) || cell_size <= 0.0)
            return fail(GMI_ERR_INVALID_CELL_SIZE, "cell_size must be positive and finite");
        GMI_CUDA(cudaSetDevice(ctx->device));
        gmi_cache c;
        c.ctx = ctx;
        c.B = batch;
        c.N = num_points;
        c.C = 1;
        c.cutoff = cell_size;
        ensure_issue(ctx, batch);
        const size_t BN = static_cast<size_t>(batch) * num_points;
        int32_t* d_pi = nullptr;
        int rc = GMI_OK;
        try {
            d_pi = static_cast<int32_t*>(gmi_host::cache_alloc(&c, sizeof(int32_t) * BN));
            gmi_host::bin_points(ctx, &c, positions, nullptr, 2048, false, d_pi, ctx->d_issue);
            for (int b = 0; b < batch; ++b) {
                origin[2 * b] = c.geom_h[b].ox;
                origin[2 * b + 1] = c.geom_h[b].oy;
                n_cols[b] = c.geom_h[b].n_cols;
                n_rows[b] = c.geom_h[b].n_rows;
            }
            if (bin_start != nullptr) {
                GMI_CUDA(cudaMemcpyAsync(bin_start, c.bins, sizeof(int32_t) * c.total_bins,
                                         cudaMemcpyDeviceToHost, ctx->stream));
            }
            if (point_index != nullptr) {
                GMI_CUDA(cudaMemcpyAsync(point_index, d_pi, sizeof(int32_t) * BN,
                                         cudaMemcpyDeviceToHost, ctx->stream));
            }
            GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            free_cache_buffers(&c);
            throw;
        }
        free_cache_buffers(&c);
        return rc;
    });
}

int gmi_bin_grid_host(gmi_ctx* ctx, const float* positions, int32_t batch, int32_t num_points,
                      double cell_size, double* origin, int32_t* n_cols, int32_t* n_rows,
                      int32_t* bin_start, int32_t* point_index) {
    return guarded([&]() -> int {
        if (ctx == nullptr || positions == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        if (batch < 1) return fail(GMI_ERR_INVALID_ARGUMENT, "batch must be >= 1");
        if (num_points <= 0) return fail(GMI_ERR_EMPTY_POINT_SET, "point set is empty");
        GMI_CUDA(cudaSetDevice(ctx->device));
        const size_t bytes = sizeof(float) * 2 * static_cast<size_t>(batch) * num_points;
        float* d = static_cast<float*>(gmi_host::dalloc(ctx, bytes));
        GMI_CUDA(cudaMemcpyAsync(d, positions, bytes, cudaMemcpyHostToDevice, ctx->stream));
        const int rc = gmi_bin_grid(ctx, d, batch, num_points, cell_size, origin, n_cols, n_rows,
                                    bin_start, point_index);
        gmi_host::dfree(ctx, d);
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        return rc;
    });
}

int gmi_optimize_points(gmi_ctx* ctx, float* positions, float* colors, int32_t batch,
                        int32_t num_points, int32_t channels, const gmi_config* cfg,
                        const float* target, int32_t steps, double learning_rate,
                        uint32_t flags, double* loss_curve) {
    return guarded([&]() -> int {
        if (ctx == nullptr || target == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        int rc = check_points(positions, colors, batch, num_points, channels);
        if (rc) return rc;
        rc = check_config(cfg);
        if (rc) return rc;
        // check_optim_config (optimize.cpp:32-44)
        if (steps < 1) return fail(GMI_ERR_CONFIG_INVALID, "steps must be >= 1");
        if (!std::isfinite(learning_rate) || learning_rate < 0.0)
            return fail(GMI_ERR_CONFIG_INVALID, "learning_rate must be finite and >= 0");
        GMI_CUDA(cudaSetDevice(ctx->device));
        return do_optimize(ctx, positions, colors, batch, num_points, channels, cfg, target, steps,
                           learning_rate, flags, loss_curve);
    });
}

int gmi_device_alloc(gmi_ctx* ctx, size_t bytes, void** out) {
    return guarded([&]() -> int {
        if (ctx == nullptr || out == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        GMI_CUDA(cudaSetDevice(ctx->device));
        *out = nullptr;
        GMI_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 16)));
        return GMI_OK;
    });
}

int gmi_device_free(gmi_ctx* ctx, void* ptr) {
    return guarded([&]() -> int {
        if (ctx == nullptr) return fail(GMI_ERR_INVALID_ARGUMENT, "ctx is null");
        if (ptr == nullptr) return GMI_OK;
        GMI_CUDA(cudaSetDevice(ctx->device));
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));  // queued work may still use it
        GMI_CUDA(cudaFree(ptr));
        return GMI_OK;
    });
}

int gmi_memcpy(gmi_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind) {
    return guarded([&]() -> int {
        if (ctx == nullptr || (bytes > 0 && (dst == nullptr || src == nullptr)))
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        if (kind < 0 || kind > 2) return fail(GMI_ERR_INVALID_ARGUMENT, "kind must be 0, 1 or 2");
        GMI_CUDA(cudaSetDevice(ctx->device));
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                           : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
        GMI_CUDA(cudaMemcpyAsync(dst, src, bytes, k, ctx->stream));
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        return GMI_OK;
    });
}

int gmi_gmm_benchmark_host(gmi_ctx* ctx, const float* image, int32_t width, int32_t height,
                           int32_t channels, int32_t factor, const float* lowres,
                           const double* sigmas, int32_t n_sigma, double* l1, double* ms,
                           int32_t* best, float* best_image) {
    return guarded([&]() -> int {
        if (ctx == nullptr || image == nullptr || l1 == nullptr || best == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        if (width < 1 || height < 1 || channels < 1)
            return fail(GMI_ERR_INVALID_DIMENSIONS, "image must be at least 1x1x1");
        // benchmark.cpp:62-68
        if (factor < 1) return fail(GMI_ERR_INVALID_FACTOR, "factors must be positive integers");
        std::vector<double> sig;
        if (sigmas == nullptr) {
            sig = {0.4 * factor, 0.5 * factor, 0.6 * factor};  // auto_sigma_candidates
            if (n_sigma != 3) return fail(GMI_ERR_INVALID_ARGUMENT, "auto sweep has 3 sigmas");
        } else {
            if (n_sigma < 1) return fail(GMI_ERR_INVALID_ARGUMENT, "n_sigma must be >= 1");
            sig.assign(sigmas, sigmas + n_sigma);
        }
        GMI_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        const int lw = (width + factor - 1) / factor, lh = (height + factor - 1) / factor;
        const int N = lw * lh;
        const size_t hwc = static_cast<size_t>(height) * width * channels;
        float* dimg = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * hwc));
        float* dlow = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * N * channels));
        float* dpos = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * N * 2));
        float* dout = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * hwc * sig.size()));
        const int nblk = static_cast<int>(std::min<size_t>((hwc + kLossThreads - 1) / kLossThreads,
                                                           2 * static_cast<size_t>(ctx->num_sms)));
        double* partial = static_cast<double*>(gmi_host::dalloc(ctx, sizeof(double) * nblk));
        double* dl1 = static_cast<double*>(gmi_host::dalloc(ctx, sizeof(double) * sig.size()));
        int rc = GMI_OK;
        std::vector<cudaEvent_t> ev(2 * sig.size(), nullptr);
        try {
            GMI_CUDA(cudaMemcpyAsync(dimg, image, sizeof(float) * hwc, cudaMemcpyHostToDevice, st));
            if (lowres != nullptr) {
                GMI_CUDA(cudaMemcpyAsync(dlow, lowres, sizeof(float) * N * channels,
                                         cudaMemcpyHostToDevice, st));
            } else {
                // block_mean_downsample (imaging.cpp:343-350)
                k_block_mean<<<(N * channels + 255) / 256, 256, 0, st>>>(dimg, width, height, channels,
                                                                         factor, lw, lh, dlow);
                GMI_LAUNCHED(ctx);
            }
            k_block_centres<<<(N + 255) / 256, 256, 0, st>>>(dpos, lw, lh, factor);
            GMI_LAUNCHED(ctx);
            for (auto& e : ev) GMI_CUDA(cudaEventCreate(&e));
            for (size_t k = 0; k < sig.size() && rc == GMI_OK; ++k) {
                // make_config(sigma, full) (core.hpp:90-94): cutoff 3 sigma
                const gmi_config cfg{sig[k], 3.0 * sig[k], GMI_FALLBACK_NEAREST, width, height};
                rc = check_config(&cfg);
                if (rc != GMI_OK) break;
                gmi_cache c;
                c.ctx = ctx;
                GMI_CUDA(cudaEventRecord(ev[2 * k], st));
                rc = do_forward(ctx, dpos, dlow, 1, N, channels, &cfg, dout + k * hwc, &c, nullptr);
                GMI_CUDA(cudaEventRecord(ev[2 * k + 1], st));
                free_cache_buffers(&c);
                if (rc != GMI_OK) break;
                k_l1_partial<<<nblk, kLossThreads, 0, st>>>(dout + k * hwc, dimg, hwc, partial);
                GMI_LAUNCHED(ctx);
                k_l1_finalize<<<1, 1, 0, st>>>(partial, nblk, 1.0 / static_cast<double>(hwc), dl1 + k);
                GMI_LAUNCHED(ctx);
            }
            if (rc == GMI_OK) {
                GMI_CUDA(cudaMemcpyAsync(l1, dl1, sizeof(double) * sig.size(), cudaMemcpyDeviceToHost, st));
                GMI_CUDA(cudaStreamSynchronize(st));
                // the first sigma with the smallest L1 (benchmark.cpp:101-106)
                int b = 0;
                for (size_t k = 1; k < sig.size(); ++k)
                    if (l1[k] < l1[b]) b = static_cast<int>(k);
                *best = b;
                if (ms != nullptr)
                    for (size_t k = 0; k < sig.size(); ++k) {
                        float t = 0.f;
                        GMI_CUDA(cudaEventElapsedTime(&t, ev[2 * k], ev[2 * k + 1]));
                        ms[k] = t;
                    }
                if (best_image != nullptr)
                    GMI_CUDA(cudaMemcpyAsync(best_image, dout + b * hwc, sizeof(float) * hwc,
                                             cudaMemcpyDeviceToHost, st));
            }
        } catch (...) {
            for (auto e : ev) if (e) cudaEventDestroy(e);
            throw;
        }
        for (auto e : ev) if (e) cudaEventDestroy(e);
        for (void* q : {static_cast<void*>(dimg), static_cast<void*>(dlow), static_cast<void*>(dpos),
                        static_cast<void*>(dout), static_cast<void*>(partial), static_cast<void*>(dl1)})
            gmi_host::dfree(ctx, q);
        GMI_CUDA(cudaStreamSynchronize(st));
        return rc;
    });
}

int gmi_optimize_points_host(gmi_ctx* ctx, float* positions, float* colors, int32_t batch,
                             int32_t num_points, int32_t channels, const gmi_config* cfg,
                             const float* target, int32_t steps, double learning_rate,
                             uint32_t flags, double* loss_curve) {
    return guarded([&]() -> int {
        if (ctx == nullptr || positions == nullptr || colors == nullptr || target == nullptr || cfg == nullptr)
            return fail(GMI_ERR_INVALID_ARGUMENT, "null argument");
        if (batch < 1 || num_points < 1 || channels < 1)
            return check_points(positions, colors, batch, num_points, channels);
        GMI_CUDA(cudaSetDevice(ctx->device));
        const size_t BN = static_cast<size_t>(batch) * num_points;
        const size_t img = static_cast<size_t>(batch) * cfg->height * cfg->width * channels;
        float* dp = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * BN * 2));
        float* dc = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * BN * channels));
        float* dt = static_cast<float*>(gmi_host::dalloc(ctx, sizeof(float) * img));
        GMI_CUDA(cudaMemcpyAsync(dp, positions, sizeof(float) * BN * 2, cudaMemcpyHostToDevice, ctx->stream));
        GMI_CUDA(cudaMemcpyAsync(dc, colors, sizeof(float) * BN * channels, cudaMemcpyHostToDevice,
                                 ctx->stream));
        GMI_CUDA(cudaMemcpyAsync(dt, target, sizeof(float) * img, cudaMemcpyHostToDevice, ctx->stream));
        const int rc = gmi_optimize_points(ctx, dp, dc, batch, num_points, channels, cfg, dt, steps,
                                           learning_rate, flags, loss_curve);
        if (rc == GMI_OK) {
            GMI_CUDA(cudaMemcpyAsync(positions, dp, sizeof(float) * BN * 2, cudaMemcpyDeviceToHost,
                                     ctx->stream));
            GMI_CUDA(cudaMemcpyAsync(colors, dc, sizeof(float) * BN * channels, cudaMemcpyDeviceToHost,
                                     ctx->stream));
        }
        gmi_host::dfree(ctx, dp);
        gmi_host::dfree(ctx, dc);
        gmi_host::dfree(ctx, dt);
        GMI_CUDA(cudaStreamSynchronize(ctx->stream));
        return rc;
    });
}

}  // extern "C"
