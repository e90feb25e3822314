// Host-side internals shared by the .cu translation units: the context, the
// ForwardCache analogue and the kernel launchers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "gmi_b200.h"
#include "gmi_common.cuh"

// Error carried from deep inside the launch code back to the C-ABI.
struct GmiFail {
    int code;
    std::string msg;
};

#define GMI_CUDA(call)                                                    \
    do {                                                                  \
        cudaError_t e_ = (call);                                          \
        if (e_ != cudaSuccess) {                                          \
            throw GmiFail{e_ == cudaErrorMemoryAllocation ? GMI_ERR_OUT_OF_MEMORY \
                                                          : GMI_ERR_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_)}; \
        }                                                                 \
    } while (0)

// Raises a kernel's dynamic shared-memory limit once per device (a per-call-
// site bitmask of devices; thread-safe for one host thread per GPU).
#define GMI_SMEM_ONCE(ctx, kernel, bytes)                                 \
    do {                                                                  \
        static std::atomic<uint64_t> done_{0};                            \
        const uint64_t bit_ = 1ull << ((ctx)->device & 63);              \
        if (!(done_.load(std::memory_order_acquire) & bit_)) {            \
            GMI_CUDA(cudaFuncSetAttribute(kernel,                         \
                cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));     \
            done_.fetch_or(bit_, std::memory_order_release);              \
        }                                                                 \
    } while (0)

#define GMI_LAUNCHED(ctx)                                                 \
    do {                                                                  \
        (ctx)->launches++;                                                \
        GMI_CUDA(cudaGetLastError());                                     \
    } while (0)

struct gmi_ctx {
    // one reference held by the creator (gmi_ctx_destroy drops it) and one
    // by every live cache returned to a caller: a cache may outlive the
    // handle it was made with (the C++ API's thread-local contexts)
    std::atomic<int> refs{1};
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint32_t flags = 0;
    uint64_t launches = 0;
    // host copy of the per-image validation keys (pinned)
    unsigned long long* h_issue = nullptr;
    // device scratch for validation keys (per image of the current call)
    unsigned long long* d_issue = nullptr;
    int d_issue_cap = 0;
    // first asynchronous error since the last gmi_ctx_synchronize:
    // [0] = key (index << 8 | code), [1] = image; sticky until read
    unsigned long long* d_pending = nullptr;
    // set while a synchronous host-buffer call runs its parts asynchronously
    // (their errors are collected by that call, not left pending)
    bool collect_now = false;
    // optional per-phase CUDA-event timing (gmi_ctx_set_profiling)
    bool profiling = false;
    struct PhaseMark {
        int phase;
        cudaEvent_t start, stop;
    };
    std::vector<PhaseMark> marks;
    double phase_ms[GMI_NUM_PHASES] = {0};
    uint64_t phase_calls[GMI_NUM_PHASES] = {0};
    // grow-only per-call scratch (stream-ordered reuse on the ctx stream)
    void* ws_ptr[24] = {nullptr};
    size_t ws_cap[24] = {0};
    // host copies of small tables uploaded into scratch slots (upload_table)
    std::vector<int32_t> ws_table[24];
    void* ws_table_ptr[24] = {nullptr};
    // scan tiles of the equal-segment (device geometry) binning, cached per
    // (batch, stride) so the hot path issues no host->device copy
    int eq_B = -1;
    int64_t eq_stride = -1;
    int eq_nt = 0;
    // copy streams of the pipelined host-buffer API (created on first use)
    cudaStream_t s_in = nullptr;
    cudaStream_t s_out = nullptr;
    // pinned staging of PAGEABLE host buffers (host API): two slots copied
    // by a few host threads while the other slot's DMA runs
    void* stg_slot[2] = {nullptr, nullptr};
    cudaEvent_t stg_ev[2] = {nullptr, nullptr};
};

// scratch slots
enum WsSlot {
    WS_BBOX = 0, WS_CELLID, WS_RANK, WS_TMP, WS_BIG, WS_BIGCOUNT, WS_TILES, WS_TSUM,
    WS_SEGOFF, WS_BLKOFF, WS_PART, WS_HOST_IN0, WS_HOST_IN1, WS_HOST_IN2,
    WS_TILES_EQ, WS_SEGOFF_EQ, WS_FOLD, WS_COUNT
};

// RAII phase marker: records an event pair on the ctx stream when profiling.
struct PhaseScope {
    gmi_ctx* ctx;
    int phase;
    cudaEvent_t start = nullptr;
    PhaseScope(gmi_ctx* c, int ph) : ctx(c), phase(ph) {
        if (ctx->profiling) {
            cudaEventCreate(&start);
            cudaEventRecord(start, ctx->stream);
        }
    }
    ~PhaseScope() {
        if (ctx->profiling && start) {
            cudaEvent_t stop;
            cudaEventCreate(&stop);
            cudaEventRecord(stop, ctx->stream);
            ctx->marks.push_back({phase, start, stop});
        }
    }
};

// Host-side latency trace (GMI_TRACE=1): microseconds since the previous mark.
void host_trace(const char* what);

// A stream-ordered device allocation owned by a cache.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// Per special pixel (fallback or exact-f64 pixel), produced by the forward.
struct Special {
    int32_t b;
    int32_t pix;      // r * W + c
    int32_t nearest;  // original point index (NearestPoint fallback) or -1
    int32_t kind;     // 1 = fallback
};

struct gmi_cache {
    gmi_ctx* ctx = nullptr;
    bool holds_ctx = false;   // a caller-owned cache: one reference on ctx
    int B = 0, N = 0, C = 0, W = 0, H = 0;
    double sigma = 0, cutoff = 0;
    int fallback = 0;
    // borrowed device pointers (owned when host API was used)
    const float* pos = nullptr;
    const float* col = nullptr;
    const float* image = nullptr;
    std::vector<DevBuf> owned;
    // binning
    std::vector<gmi_dev::Geom> geom_h;
    gmi_dev::Geom* geom_d = nullptr;
    int32_t* bins = nullptr;  // concatenated bin_start per image
    int64_t total_bins = 0;
    // device-geometry binning: image b's bin_start at b * grid_stride, grid
    // dims <= grid_cap (geom_h is empty; the geometry lives only in geom_d)
    int grid_cap = 0;
    int64_t grid_stride = 0;
    bool sort_cells = true;   // within-cell index order (generic and wide gathers)
    // hot layout (sorted by cell, then fine x-column, then index)
    float* sx = nullptr;      // [B][N]
    float* sy = nullptr;      // [B][N]
    int32_t* sidx = nullptr;  // [B][N] original point index
    float* scol = nullptr;    // [B][C][N] channel-planar
    // fast-path hot layout (C <= 4, fp32 weights): one 32-byte record per
    // point in bin order, (x, y, c0, c1) (c2, c3, idx|flag bits, 0); replaces
    // sx/sy/sidx/scol, which stay null
    float4* rec = nullptr;    // [B][N][2]
    float* ccol = nullptr;    // C > 4: all colours [B][N][C] in bin order
    // large images (slot_grads): slot of each original point, so the backward
    // writes gradients in slot order and one gather pass permutes them
    int32_t* inv = nullptr;   // [B][N]
    // per pixel
    float* wsum = nullptr;    // [B][H][W]; 0 => special pixel
    double* wsum64 = nullptr; // [B][H][W] f64 normaliser (precise mode only)
    double* image64 = nullptr;// [B][H][W][C] f64 image (precise mode: the backward's out)
    // special pixels
    Special* special = nullptr;
    int32_t* special_count_d = nullptr;
    int special_cap = 0;
    int special_count = -1;   // host copy (-1 = not read yet)
    bool special_overflow = false;
    bool force_generic = false;  // use the generic gather (tests / GMI_GENERIC)
    // composite cache of the pipelined host API: image chunks [part_b0[k],
    // part_b0[k] + parts[k]->B), each a complete cache of its own
    std::vector<gmi_cache*> parts;
    std::vector<int> part_b0;
    // recorded on the copy stream after the image download (host API); the
    // buffers are freed behind it
    cudaEvent_t d2h_done = nullptr;
};

namespace gmi_host {

// memory (stream-ordered)
void* dalloc(gmi_ctx* ctx, size_t bytes);
void dfree(gmi_ctx* ctx, void* p);
// ctx scratch slot of at least `bytes` (contents undefined)
void* scratch(gmi_ctx* ctx, int slot, size_t bytes);
void* cache_alloc(gmi_cache* c, size_t bytes);
// Device copy of a small host table in a ctx scratch slot, uploaded only
// when its contents (or the slot's buffer) change: repeated calls issue no
// host->device copy, so the hot path stays capturable in a CUDA graph.
int32_t* upload_table(gmi_ctx* ctx, int slot, const std::vector<int32_t>& v);

// ---- binning (gmi_bin.cu) ----
// Validates positions, computes bbox, geometry (cap) and fills c->geom_*,
// c->bins; when hot_layout, builds the sorted SoA (and validates colours),
// else (reference export) writes point_index[B][N].
void bin_points(gmi_ctx* ctx, gmi_cache* c, const float* pos, const float* col,
                int cap, bool hot_layout, int32_t* point_index_out,
                unsigned long long* d_issue);
int host_axis_cells(double span, double cell, int cap);

// ---- forward (gmi_forward.cu) ----
void launch_forward(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts);
bool launch_gather_fast(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts);
bool gather_fast_ok(const gmi_cache* c);
// Gradients through slot order (gmi_backward.cu k_permute_grads) for images
// whose per-image gradient array is far larger than L2 would want to merge
// scattered partial-sector writes in: N >= GMI_SLOT_GRADS_MIN_N (default
// 2^20) points per image, C <= 4 (the record layout's single channel group).
bool slot_grads(int N, int C);
// wide-channel path (C > 4, gmi_wide.cu); false when it does not apply
bool launch_gather_wide(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts);
bool launch_backward_wide(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                          float* d_colors, float* d_positions);
void launch_special_forward(gmi_ctx* ctx, gmi_cache* c, float* image,
                            int32_t* counts);

// ---- backward (gmi_backward.cu) ----
void launch_backward(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                     float* d_colors, float* d_positions);
void launch_special_backward(gmi_ctx* ctx, const gmi_cache* c,
                             const float* upstream, float* d_colors,
                             float* d_positions);

}  // namespace gmi_host
