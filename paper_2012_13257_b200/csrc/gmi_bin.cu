// K1 — point binning: a device counting sort reproducing the reference's
// build_bin_grid (bin_grid.cpp:38-82) bit for bit.
//
//   k_bbox_validate  bbox (exact fp32 min/max == the reference's f64 min/max
//                    of widened fp32 values) + position finiteness
//                    (core.cpp:73-79)
//   host             origin / n_cols / n_rows in f64 (bin_grid.cpp:18-24,58-60)
//   k_count          f64 cell of each point (bin_grid.cpp:28-36,66-67) and an
//                    atomic arrival rank inside its cell
//   scan             segmented exclusive scan -> bin_start (bin_grid.cpp:72-75)
//   k_scatter        point -> bin_start[cell] + rank (unordered within a cell)
//   k_cellsort_*     order each cell by original index (bin_grid.cpp:76-80),
//                    in place: this IS the reference's point_index
//   k_emit           hot layout in that order, thread per slot: the
//                    bin-ordered SoA (x, y, index|ambiguous-flag, colour
//                    planes), boundary-ambiguity flags, colour validation
//                    (core.cpp:80-92)
#include <algorithm>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

constexpr int kScanTile = 2048;   // ints per scan tile
constexpr int kScanThreads = 256;
constexpr int kSmallCell = 32;    // cells up to this size: one thread sorts
constexpr int kBigSmemKeys = 8192;

// ---------------------------------------------------------------------------
__global__ void k_bbox_validate(const float2* __restrict__ pos, int N,
                                uint32_t* __restrict__ bbox,
                                unsigned long long* __restrict__ issue) {
    const int b = blockIdx.y;
    const float2* p = pos + static_cast<size_t>(b) * N;
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    unsigned long long bad = kNoIssue;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += gridDim.x * blockDim.x) {
        const float2 v = p[i];
        if (!is_finite_f(v.x) || !is_finite_f(v.y)) {
            // NonFiniteValue (core.hpp:36) -> 1 + 0
            bad = min(bad, (static_cast<unsigned long long>(i) << 8) | 1ull);
            continue;
        }
        mnx = fminf(mnx, v.x);
        mny = fminf(mny, v.y);
        mxx = fmaxf(mxx, v.x);
        mxy = fmaxf(mxy, v.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
        bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if ((threadIdx.x & 31) == 0) {
        uint32_t* bb = bbox + 4 * b;
        atomicMin(bb + 0, f2ord(mnx));
        atomicMin(bb + 1, f2ord(mny));
        atomicMax(bb + 2, f2ord(mxx));
        atomicMax(bb + 3, f2ord(mxy));
        if (bad != kNoIssue) atomicMin(issue + b, bad);
    }
}

// The same bbox + finiteness pass with 16-byte loads (two points each) and
// 8 points per thread in flight, one block-level reduction and 4 atomics per
// CTA (N even, positions 16-byte aligned).
constexpr int kBboxPer = 4;  // float4 per thread

__global__ void __launch_bounds__(256) k_bbox_validate4(const float4* __restrict__ pos, int N,
                                                        uint32_t* __restrict__ bbox,
                                                        unsigned long long* __restrict__ issue) {
    __shared__ float red[4][8];
    __shared__ unsigned long long red_bad[8];
    const int b = blockIdx.y;
    const int n2 = N >> 1;  // float4 per image
    const float4* p = pos + static_cast<size_t>(b) * n2;
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    unsigned long long bad = kNoIssue;
    const int k0 = blockIdx.x * (blockDim.x * kBboxPer) + threadIdx.x;
    float4 v[kBboxPer];
#pragma unroll
    for (int u = 0; u < kBboxPer; ++u) {
        const int k = k0 + u * blockDim.x;
        v[u] = k < n2 ? p[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kBboxPer; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k >= n2) continue;
        const bool f0 = is_finite_f(v[u].x) && is_finite_f(v[u].y);
        const bool f1 = is_finite_f(v[u].z) && is_finite_f(v[u].w);
        if (!f0) bad = min(bad, (static_cast<unsigned long long>(2 * k) << 8) | 1ull);
        else if (!f1) bad = min(bad, (static_cast<unsigned long long>(2 * k + 1) << 8) | 1ull);
        if (f0) {
            mnx = fminf(mnx, v[u].x);
            mny = fminf(mny, v[u].y);
            mxx = fmaxf(mxx, v[u].x);
            mxy = fmaxf(mxy, v[u].y);
        }
        if (f1) {
            mnx = fminf(mnx, v[u].z);
            mny = fminf(mny, v[u].w);
            mxx = fmaxf(mxx, v[u].z);
            mxy = fmaxf(mxy, v[u].w);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
        bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = mnx;
        red[1][w] = mny;
        red[2][w] = mxx;
        red[3][w] = mxy;
        red_bad[w] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            mnx = fminf(mnx, red[0][k]);
            mny = fminf(mny, red[1][k]);
            mxx = fmaxf(mxx, red[2][k]);
            mxy = fmaxf(mxy, red[3][k]);
            bad = min(bad, red_bad[k]);
        }
        uint32_t* bb = bbox + 4 * b;
        atomicMin(bb + 0, f2ord(mnx));
        atomicMin(bb + 1, f2ord(mny));
        atomicMax(bb + 2, f2ord(mxx));
        atomicMax(bb + 3, f2ord(mxy));
        if (bad != kNoIssue) atomicMin(issue + b, bad);
    }
}

__global__ void k_bbox_init(uint32_t* bbox, unsigned long long* issue, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        bbox[4 * b + 0] = 0xFFFFFFFFu;
        bbox[4 * b + 1] = 0xFFFFFFFFu;
        bbox[4 * b + 2] = 0u;
        bbox[4 * b + 3] = 0u;
        issue[b] = kNoIssue;
    }
}

// ---------------------------------------------------------------------------
__global__ void k_scatter(int N, const Geom* __restrict__ geom,
                          const int32_t* __restrict__ bins,
                          const int32_t* __restrict__ cellid,
                          const int32_t* __restrict__ rank,
                          int32_t* __restrict__ tmp) {
    const int b = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const size_t k = static_cast<size_t>(b) * N + i;
    const int dst = bins[geom[b].bin_off + cellid[k]] + rank[k];
    tmp[static_cast<size_t>(b) * N + dst] = i;
}

// ---------------------------------------------------------------------------
// Segmented exclusive scan (one segment per image, length n_bins + 1).
struct ScanTile {
    int64_t start;
    int32_t len;
    int32_t seg;
};

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot,
                                                    int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int w = lane < nw ? warp_tot[lane] : 0;
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < nw) warp_tot[lane] = wi - w;
        if (lane == nw - 1) *total = wi;
    }
    __syncthreads();
    const int res = warp_tot[warp] + incl - v;
    __syncthreads();
    return res;
}

// Per tile: the sum of its counts.  With `big` (the fast path), cells above
// the gather's chunk capacity are listed on the way (k_sort_big_recs puts
// their records in index order) — the counts are read here anyway.
constexpr int kBigRecCellScan = 640;   // = kBigRecCell below
__global__ void k_scan_reduce(const int32_t* __restrict__ data,
                              const ScanTile* __restrict__ tiles,
                              int32_t* __restrict__ tile_sum,
                              const Geom* __restrict__ geom = nullptr,
                              int2* __restrict__ big = nullptr, int32_t* big_count = nullptr) {
    __shared__ int red[kScanThreads / 32];
    const ScanTile t = tiles[blockIdx.x];
    int s = 0;
    for (int k = threadIdx.x; k < t.len; k += blockDim.x) {
        const int v = data[t.start + k];
        s += v;
        if (big != nullptr && v > kBigRecCellScan)
            big[atomicAdd(big_count, 1)] =
                make_int2(t.seg, static_cast<int>(t.start + k - geom[t.seg].bin_off));
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) tot += red[w];
        tile_sum[blockIdx.x] = tot;
    }
}

// one block per segment; tile sums of the segment scanned in place
__global__ void k_scan_segments(int32_t* __restrict__ tile_sum,
                                const int32_t* __restrict__ seg_tile_off) {
    __shared__ int warp_tot[32];
    __shared__ int total;
    const int t0 = seg_tile_off[blockIdx.x], t1 = seg_tile_off[blockIdx.x + 1];
    int carry = 0;
    for (int base = t0; base < t1; base += blockDim.x) {
        const int k = base + threadIdx.x;
        const int v = k < t1 ? tile_sum[k] : 0;
        const int ex = block_exclusive_scan(v, warp_tot, &total);
        if (k < t1) tile_sum[k] = carry + ex;
        carry += total;
        __syncthreads();
    }
}

__global__ void k_scan_apply(int32_t* __restrict__ data,
                             const ScanTile* __restrict__ tiles,
                             const int32_t* __restrict__ tile_off, int inclusive) {
    __shared__ int buf[kScanTile];
    __shared__ int warp_tot[32];
    __shared__ int total;
    const ScanTile t = tiles[blockIdx.x];
    for (int k = threadIdx.x; k < kScanTile; k += blockDim.x)
        buf[k] = k < t.len ? data[t.start + k] : 0;
    __syncthreads();
    constexpr int kPer = kScanTile / kScanThreads;
    int v[kPer];
    int s = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        v[j] = buf[threadIdx.x * kPer + j];
        s += v[j];
    }
    int ex = block_exclusive_scan(s, warp_tot, &total) + tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        if (!inclusive) buf[threadIdx.x * kPer + j] = ex;
        ex += v[j];
        if (inclusive) buf[threadIdx.x * kPer + j] = ex;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < t.len; k += blockDim.x) data[t.start + k] = buf[k];
}

// ---------------------------------------------------------------------------
// Within-cell ordering: ascending original index (bin_grid.cpp:76-80), sorted
// in place in the index array.  This is the reference's point_index; the hot
// SoA is emitted in exactly this order (the gather re-orders by x itself).
constexpr int kRegCell = 8;

__device__ __forceinline__ void cswap(int& a, int& b) {
    const int lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

__global__ void k_cellsort_small(int N, const Geom* __restrict__ geom,
                                 const int32_t* __restrict__ bins, int32_t* __restrict__ tmp,
                                 int2* __restrict__ big, int32_t* big_count) {
    const int b = blockIdx.y;
    const Geom g = geom[b];
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= g.n_cols * g.n_rows) return;
    const int s = bins[g.bin_off + cell], e = bins[g.bin_off + cell + 1];
    const int n = e - s;
    if (n <= 1) return;
    int32_t* t = tmp + static_cast<size_t>(b) * N + s;
    if (n <= kRegCell) {
        // sorting network on registers (padding sorts to the end)
        int v[kRegCell];
#pragma unroll
        for (int k = 0; k < kRegCell; ++k) v[k] = k < n ? t[k] : INT32_MAX;
        // Batcher odd-even merge network for 8 keys (19 comparators)
        cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
        cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[6]); cswap(v[5], v[7]);
        cswap(v[1], v[2]); cswap(v[5], v[6]);
        cswap(v[0], v[4]); cswap(v[1], v[5]); cswap(v[2], v[6]); cswap(v[3], v[7]);
        cswap(v[2], v[4]); cswap(v[3], v[5]);
        cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
#pragma unroll
        for (int k = 0; k < kRegCell; ++k)
            if (k < n) t[k] = v[k];
        return;
    }
    if (n > kSmallCell) {
        const int slot = atomicAdd(big_count, 1);
        big[slot] = make_int2(b, cell);
        return;
    }
    int key[kSmallCell];
    for (int k = 0; k < n; ++k) {
        const int v = t[k];
        int j = k;
        while (j > 0 && key[j - 1] > v) {
            key[j] = key[j - 1];
            --j;
        }
        key[j] = v;
    }
    for (int k = 0; k < n; ++k) t[k] = key[k];
}

// One CTA per big cell: bitonic sort of the cell's indices in shared memory
// (n <= kBigSmemKeys) or in place in global memory (slow path).
__global__ void k_cellsort_big(int N, const Geom* __restrict__ geom,
                               const int32_t* __restrict__ bins, int32_t* __restrict__ tmp,
                               const int2* __restrict__ big, const int32_t* __restrict__ big_count) {
    extern __shared__ int skey[];
    const int nbig = *big_count;
    for (int job = blockIdx.x; job < nbig; job += gridDim.x) {
        const int b = big[job].x, cell = big[job].y;
        const Geom g = geom[b];
        const int s = bins[g.bin_off + cell], e = bins[g.bin_off + cell + 1];
        const int n = e - s;
        int32_t* t = tmp + static_cast<size_t>(b) * N + s;
        int np2 = 1;
        while (np2 < n) np2 <<= 1;
        const bool in_smem = n <= kBigSmemKeys;
        int* key = in_smem ? skey : t;
        if (in_smem) {
            for (int k = threadIdx.x; k < np2; k += blockDim.x) skey[k] = k < n ? t[k] : INT32_MAX;
            __syncthreads();
        }
        // flip formulation: all comparators ascending, so padding (+inf) never
        // moves below n and partners >= n can be skipped in place
        for (int size = 2; size <= np2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int k = threadIdx.x; k < np2; k += blockDim.x) {
                    const int partner = (stride == (size >> 1)) ? (k ^ (size - 1)) : (k ^ stride);
                    if (partner > k && (in_smem || partner < n)) {
                        const int a = key[k], c = key[partner];
                        if (a > c) {
                            key[k] = c;
                            key[partner] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        if (in_smem) {
            for (int k = threadIdx.x; k < n; k += blockDim.x) t[k] = skey[k];
            __syncthreads();
        }
    }
}

// Hot layout, thread per slot (coalesced writes): gather the point, classify
// boundary ambiguity (kUnsafeBit, gmi_common.cuh), validate colours
// (core.cpp:80-92, first violation by index via atomicMin).
struct EmitParams {
    const float2* pos;
    const float* col;
    const int32_t* tmp;
    float* sx;
    float* sy;
    int32_t* sidx;
    float* scol;
    unsigned long long* issue;
    int32_t* inv;           // large images: slot of each original point (or null)
    int N, C;
    int classify;
    float rf, r2f;
};

__device__ __forceinline__ bool point_ambiguous_f32(float mx, float my, float rf, float r2f) {
    if (!(fabsf(mx) < 1048576.f && fabsf(my) < 1048576.f)) return true;
    const float tau = kAmbRel * r2f;
    const float tx = truncf(mx), ty = truncf(my);
    const float fmu = mx - tx, fmy = my - ty;  // exact
    const int by = static_cast<int>(ty);
    const int y0 = static_cast<int>(floorf(my - rf - 0.02f));
    const int y1 = static_cast<int>(ceilf(my + rf + 0.02f));
    for (int y = y0; y <= y1; ++y) {
        // dy = y - my to ~1 ulp (|dy| <= r + 1); h2 error ~1e-7 r^2 << tau
        const float dy = static_cast<float>(y - by) - fmy;
        const float h2f = fmaf(-dy, dy, r2f);
        if (h2f < -tau) continue;
        const float s = sqrtf(fmaxf(h2f, 0.f));
        const float nl = rintf(fmu - s), nr = rintf(fmu + s);
        const float el = fmaf(nl - fmu, nl - fmu, -h2f);
        const float er = fmaf(nr - fmu, nr - fmu, -h2f);
        if (fabsf(el) <= tau || fabsf(er) <= tau) return true;
    }
    return false;
}

__global__ void k_emit(EmitParams p) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.N) return;
    const size_t bk = static_cast<size_t>(b) * p.N + k;
    const int i = p.tmp[bk];
    const float2 v = p.pos[static_cast<size_t>(b) * p.N + i];
    p.sx[bk] = v.x;
    p.sy[bk] = v.y;
    const bool amb = p.classify && point_ambiguous_f32(v.x, v.y, p.rf, p.r2f);
    p.sidx[bk] = static_cast<int32_t>(static_cast<uint32_t>(i) | (amb ? kUnsafeBit : 0u));
    const float* c = p.col + (static_cast<size_t>(b) * p.N + i) * p.C;
    unsigned code = 0;
    for (int ch = 0; ch < p.C; ++ch) {
        const float cv = c[ch];
        p.scol[(static_cast<size_t>(b) * p.C + ch) * p.N + k] = cv;
        if (code == 0) {
            if (!is_finite_f(cv)) code = 1;             // NonFiniteValue
            else if (cv < 0.0f || cv > 1.0f) code = 2;  // ColorOutOfRange
        }
    }
    if (code) atomicMin(p.issue + b, (static_cast<unsigned long long>(i) << 8) | code);
}

// Device-side geometry (bin_grid.cpp:45-60 with axis_cells 18-24), the same
// IEEE f64 operations as host_axis_cells: lets the hot path enqueue the whole
// binning without a host round trip.  Images whose bbox is not finite (a
// validation error is pending) get a 1x1 grid so the pipeline stays in
// bounds until gmi_ctx_synchronize / the sync point reports the error.
__device__ int dev_axis_cells(double span, double cell, int cap) {
    const double ideal = ceil(__ddiv_rn(span, cell)) + 2.0;
    if (!(ideal < static_cast<double>(cap))) return cap;
    const int v = x86_d2i(ideal);
    return v > 1 ? v : 1;
}

__global__ void k_geom(const uint32_t* __restrict__ bbox, int B, double cell, int cap,
                       int64_t stride, Geom* __restrict__ geom) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double mnx = ord2f(bbox[4 * b + 0]), mny = ord2f(bbox[4 * b + 1]);
    const double mxx = ord2f(bbox[4 * b + 2]), mxy = ord2f(bbox[4 * b + 3]);
    Geom g{};
    g.cell = cell;
    const bool ok = mnx <= mxx && mny <= mxy && fabs(mnx) < 1e300 && fabs(mxx) < 1e300 &&
                    fabs(mny) < 1e300 && fabs(mxy) < 1e300;
    if (ok) {
        g.ox = __dsub_rn(mnx, cell);
        g.oy = __dsub_rn(mny, cell);
        g.n_cols = dev_axis_cells(__dsub_rn(mxx, mnx), cell, cap);
        g.n_rows = dev_axis_cells(__dsub_rn(mxy, mny), cell, cap);
    } else {
        g.ox = 0.0;
        g.oy = 0.0;
        g.n_cols = 1;
        g.n_rows = 1;
    }
    g.capped = (g.n_cols >= cap || g.n_rows >= cap) ? 1 : 0;
    g.bin_off = static_cast<int64_t>(b) * stride;
    g.qx0 = static_cast<float>(g.ox);
    g.qscale = 2.0f;
    geom[b] = g;
}

// Boundary ambiguity with fp32 row geometry and a ~2 ulp reciprocal square
// root: the row crossing's nearest integers are found from s = sqrt(h^2),
// whose error only matters when mu -+ s is within ~1e-6 of a half-integer,
// i.e. when both neighbouring integers are ~1/2 away and far outside the
// 8e-6 r^2 band (same decision as point_ambiguous in gmi_common.cuh).
//
// Branch-free: the point is ambiguous iff the smallest |e| over the rows'
// candidate integers is <= tau.  Rows outside the disk need no mask: there
// h^2 < -tau, s = 0 and e = (n - mu)^2 - h^2 >= -h^2 > tau; so does the
// extra row an odd row count adds past y1 (its dy exceeds r + 0.02).
__device__ __forceinline__ bool point_ambiguous_fast(float mx, float my, float rf, float r2f) {
    if (!(fabsf(mx) < 1048576.f && fabsf(my) < 1048576.f)) return true;
    const float tau = kAmbRel * r2f;
    const float tx = truncf(mx), ty = truncf(my);
    const float fmu = mx - tx, fmy = my - ty;  // exact
    const int by = static_cast<int>(ty);
    const int y0 = static_cast<int>(floorf(my - rf - 0.02f));
    const int y1 = static_cast<int>(ceilf(my + rf + 0.02f));
    // two rows per step in f32x2; nearest integers by round-to-nearest adds
    // of 1.5 * 2^23 (|values| < 2^22), no conversions on the XU pipe
    constexpr float kM = 12582912.0f;
    const float2 fm2 = make_float2(fmu, fmu), mf2 = make_float2(-fmu, -fmu);
    const float2 M2 = make_float2(kM, kM), nM2 = make_float2(-kM, -kM);
    float2 dy = make_float2(static_cast<float>(y0 - by) - fmy, static_cast<float>(y0 + 1 - by) - fmy);
    const float2 two = make_float2(2.f, 2.f), r2 = make_float2(r2f, r2f);
    float emin = INFINITY;
#pragma unroll 2
    for (int y = y0; y <= y1; y += 2) {
        const float2 h2 = __ffma2_rn(make_float2(-dy.x, -dy.y), dy, r2);
        const float hx = fmaxf(h2.x, 1e-30f), hy = fmaxf(h2.y, 1e-30f);
        const float2 sq = __fmul2_rn(make_float2(hx, hy), make_float2(rsqrt_ftz(hx), rsqrt_ftz(hy)));
        const float2 lo = __fadd2_rn(fm2, make_float2(-sq.x, -sq.y));
        const float2 hi = __fadd2_rn(fm2, sq);
        const float2 nl = __fadd2_rn(__fadd2_rn(lo, M2), nM2);  // rint
        const float2 nr = __fadd2_rn(__fadd2_rn(hi, M2), nM2);
        const float2 dl = __fadd2_rn(nl, mf2), dr = __fadd2_rn(nr, mf2);
        const float2 el = __ffma2_rn(dl, dl, make_float2(-h2.x, -h2.y));
        const float2 er = __ffma2_rn(dr, dr, make_float2(-h2.x, -h2.y));
        emin = fminf(emin, fminf(fminf(fabsf(el.x), fabsf(er.x)), fminf(fabsf(el.y), fabsf(er.y))));
        dy = __fadd2_rn(dy, two);
    }
    return emin <= tau;
}

// Hot layout straight from atomic slots (no within-cell ordering: the fast
// gather canonicalises its own bins and the backward is order-independent):
// three points per thread, coalesced reads of the points, their cells
// recomputed (bit-identical to k_count_red) and slots taken by decrementing
// the cells' ends (the inclusive scan), so the ends become bin_start with no
// rank or cell-id arrays in between; the three slot atomics are in flight
// together while the colour validation (core.cpp:80-92) and the ambiguity
// test run; ONE 32-byte record per point — (x, y, c0, c1) (c2, c3, idx |
// ambiguity flag, 0) — written by one 256-bit store.
struct ScatterEmitParams {
    const float2* pos;
    const float* col;
    const Geom* geom;
    int32_t* bins;          // k_scatter_emit: cell ends, decremented to starts
    float4* rec;
    float* ccol;   // C > 4: [B][N][C] colours in bin order
    unsigned long long* issue;
    int32_t* inv;           // large images: slot of each original point (or null)
    int N, C;
    int classify;
    float rf, r2f;
};

#ifndef GMI_K1_EMIT_PER
#define GMI_K1_EMIT_PER 3
#endif
constexpr int kEmitPer = GMI_K1_EMIT_PER;

__global__ void __launch_bounds__(256) k_scatter_emit(ScatterEmitParams p) {
    const int b = blockIdx.y;
    const size_t base = static_cast<size_t>(b) * p.N;
    const Geom g = p.geom[b];
    const double inv = 1.0 / g.cell;
    const int i0 = blockIdx.x * (blockDim.x * kEmitPer) + threadIdx.x;
    const int istep = blockDim.x;
    int dst[kEmitPer];
    float2 v[kEmitPer];
    float c[kEmitPer][4];
    // straight-line code (indices past N clamped, their atomics add 0) so
    // the slot atomics are all in flight before anything consumes them:
    // their round trips overlap the colour checks and the ambiguity test
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = min(i0 + u * istep, p.N - 1);
        v[u] = p.pos[base + i];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) c[u][ch] = ch < p.C ? p.col[(base + i) * p.C + ch] : 0.f;
    }
    int old[kEmitPer];
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int cx = cell_of_fast(static_cast<double>(v[u].x), g.ox, g.cell, inv, g.n_cols);
        const int cy = cell_of_fast(static_cast<double>(v[u].y), g.oy, g.cell, inv, g.n_rows);
        old[u] = atomicSub(p.bins + g.bin_off + cy * g.n_cols + cx,
                           i0 + u * istep < p.N ? 1 : 0);  // bin_grid.cpp:67
    }
    uint32_t id[kEmitPer];
    unsigned code[kEmitPer];
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = i0 + u * istep;
        code[u] = 0;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            if (ch < p.C && code[u] == 0) {
                if (!is_finite_f(c[u][ch])) code[u] = 1;                   // NonFiniteValue
                else if (c[u][ch] < 0.0f || c[u][ch] > 1.0f) code[u] = 2;  // ColorOutOfRange
            }
        }
        const bool amb = p.classify && point_ambiguous_fast(v[u].x, v[u].y, p.rf, p.r2f);
        id[u] = static_cast<uint32_t>(i) | (amb ? kUnsafeBit : 0u);
    }
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = i0 + u * istep;
        if (i >= p.N) continue;
        dst[u] = old[u] - 1;
        GMI_CHECK(dst[u] >= 0 && dst[u] < p.N);
        if (p.ccol != nullptr) {
            // C > 4: every channel, validated in channel order, copied whole
            const float* src = p.col + (base + i) * p.C;
            float* dstc = p.ccol + (base + dst[u]) * p.C;
            for (int ch = 0; ch < p.C; ++ch) {
                const float cv = src[ch];
                dstc[ch] = cv;
                if (code[u] == 0) {
                    if (!is_finite_f(cv)) code[u] = 1;
                    else if (cv < 0.0f || cv > 1.0f) code[u] = 2;
                }
            }
        }
        if (code[u]) atomicMin(p.issue + b, (static_cast<unsigned long long>(i) << 8) | code[u]);
        if (p.inv != nullptr) p.inv[base + i] = dst[u];
        st_rec32(p.rec + (base + dst[u]) * 2, make_float4(v[u].x, v[u].y, c[u][0], c[u][1]),
                 make_float4(c[u][2], c[u][3], __uint_as_float(id[u]), 0.f));
    }
}

// Record layout in index-ordered cells (wide-channel path, C > 4): thread
// per slot, point i = tmp[slot]; the 32-byte record, all C colours and the
// colour validation, as k_scatter_emit but in the reference's bin order.
__global__ void __launch_bounds__(256) k_emit_rec(ScatterEmitParams p, const int32_t* __restrict__ tmp) {
    const int b = blockIdx.y;
    const size_t base = static_cast<size_t>(b) * p.N;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.N) return;
    const int i = tmp[base + k];
    const float2 v = p.pos[base + i];
    const float* src = p.col + (base + i) * p.C;
    float* dstc = p.ccol + (base + k) * p.C;
    unsigned code = 0;
    const bool vec = (p.C % 4) == 0 && (reinterpret_cast<uintptr_t>(p.col) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(p.ccol) & 15) == 0;
    float c4[4] = {0.f, 0.f, 0.f, 0.f};
    for (int ch = 0; ch < p.C; ch += 4) {
        float cv[4];
        if (vec) {
            const float4 t = *reinterpret_cast<const float4*>(src + ch);
            cv[0] = t.x; cv[1] = t.y; cv[2] = t.z; cv[3] = t.w;
            *reinterpret_cast<float4*>(dstc + ch) = t;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                cv[j] = ch + j < p.C ? src[ch + j] : 0.f;
                if (ch + j < p.C) dstc[ch + j] = cv[j];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (ch + j < p.C && code == 0) {
                if (!is_finite_f(cv[j])) code = 1;                // NonFiniteValue
                else if (cv[j] < 0.0f || cv[j] > 1.0f) code = 2;  // ColorOutOfRange
            }
        }
        if (ch == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) c4[j] = cv[j];
        }
    }
    if (code) atomicMin(p.issue + b, (static_cast<unsigned long long>(i) << 8) | code);
    const bool amb = p.classify && point_ambiguous_fast(v.x, v.y, p.rf, p.r2f);
    const uint32_t id = static_cast<uint32_t>(i) | (amb ? kUnsafeBit : 0u);
    st_rec32(p.rec + (base + k) * 2, make_float4(v.x, v.y, c4[0], c4[1]),
             make_float4(c4[2], c4[3], __uint_as_float(id), 0.f));
}

// Cells the fast gather may split across chunks (> its 640-candidate
// capacity) get their records in ascending original index, so chunk
// membership — and the summation order — is independent of the atomic
// arrival order (bit-deterministic results for clustered inputs).
constexpr int kBigRecCell = 640;    // = the fast gather's chunk capacity (kCap)
static_assert(kBigRecCell == kBigRecCellScan, "the scan lists the cells k_sort_big_recs sorts");
constexpr int kBigRecSmem = 4096;   // cells up to this size sort in shared memory

__device__ __forceinline__ uint32_t rec_idx(const float4& r1) {
    return __float_as_uint(r1.z) & 0x7fffffffu;
}

__global__ void __launch_bounds__(512) k_sort_big_recs(int N, const Geom* __restrict__ geom,
                                                       const int32_t* __restrict__ bins,
                                                       float4* __restrict__ rec,
                                                       const int2* __restrict__ big,
                                                       const int32_t* __restrict__ big_count,
                                                       int32_t* __restrict__ inv) {
    extern __shared__ float4 sr[];  // [2 kBigRecSmem] records, then the keys
    unsigned long long* key = reinterpret_cast<unsigned long long*>(sr + 2 * kBigRecSmem);
    const int nbig = *big_count;
    for (int job = blockIdx.x; job < nbig; job += gridDim.x) {
        const int b = big[job].x, cell = big[job].y;
        const Geom g = geom[b];
        const int s = bins[g.bin_off + cell], n = bins[g.bin_off + cell + 1] - s;
        float4* R = rec + (static_cast<size_t>(b) * N + s) * 2;
        int np2 = 1;
        while (np2 < n) np2 <<= 1;
        if (n <= kBigRecSmem) {
            for (int k = threadIdx.x; k < np2; k += blockDim.x) {
                if (k < n) {
                    sr[2 * k] = R[2 * k];
                    sr[2 * k + 1] = R[2 * k + 1];
                    key[k] = (static_cast<unsigned long long>(rec_idx(sr[2 * k + 1])) << 32) | k;
                } else {
                    key[k] = ~0ull;
                }
            }
            __syncthreads();
            for (int size = 2; size <= np2; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int k = threadIdx.x; k < np2; k += blockDim.x) {
                        const int partner = (stride == (size >> 1)) ? (k ^ (size - 1)) : (k ^ stride);
                        if (partner > k) {
                            const unsigned long long a = key[k], c = key[partner];
                            if (a > c) {
                                key[k] = c;
                                key[partner] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const int src = static_cast<int>(key[k] & 0xffffffffu);
                R[2 * k] = sr[2 * src];
                R[2 * k + 1] = sr[2 * src + 1];
                if (inv != nullptr) inv[static_cast<size_t>(b) * N + rec_idx(sr[2 * src + 1])] = s + k;
            }
            __syncthreads();
        } else {
            // in place in global memory (pathological cells): bitonic on the
            // records, partners past n skipped (all comparators ascending)
            for (int size = 2; size <= np2; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int k = threadIdx.x; k < np2; k += blockDim.x) {
                        const int partner = (stride == (size >> 1)) ? (k ^ (size - 1)) : (k ^ stride);
                        if (partner > k && partner < n) {
                            const float4 a1 = R[2 * k + 1], c1 = R[2 * partner + 1];
                            if (rec_idx(a1) > rec_idx(c1)) {
                                const float4 a0 = R[2 * k], c0 = R[2 * partner];
                                R[2 * k] = c0;
                                R[2 * k + 1] = c1;
                                R[2 * partner] = a0;
                                R[2 * partner + 1] = a1;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            if (inv != nullptr)
                for (int k = threadIdx.x; k < n; k += blockDim.x)
                    inv[static_cast<size_t>(b) * N + rec_idx(R[2 * k + 1])] = s + k;
            __syncthreads();
        }
    }
}

// Cell counts with a private shared-memory histogram (device geometry whose
// cell grid fits shared memory, e.g. configs[1]/[2]): CTA = one slice of one
// image's points, 1024 threads, the whole grid's counters in shared memory
// (native shared atomics instead of random L2 reductions), then one
// coalesced reduction per non-empty cell.  Same counts as k_count_red.
constexpr int kCountSmemCells = 56 * 1024;  // 224 KB of counters

__global__ void __launch_bounds__(1024, 1) k_count_smem(const float2* __restrict__ pos, int N,
                                                       const Geom* __restrict__ geom,
                                                       int32_t* __restrict__ bins, int parts) {
    extern __shared__ int hist[];
    const int b = blockIdx.y, tid = threadIdx.x;
    const Geom g = geom[b];
    const double inv = 1.0 / g.cell;
    const int cells = g.n_cols * g.n_rows;
    for (int k = tid; k < cells; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(b) * N;
    const int per = (N + parts - 1) / parts;
    const int i_beg = blockIdx.x * per, i_end = min(N, i_beg + per);
    for (int i = i_beg + tid; i < i_end; i += 4 * blockDim.x) {
        float2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = pos[base + min(i + u * static_cast<int>(blockDim.x), i_end - 1)];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i + u * static_cast<int>(blockDim.x) >= i_end) continue;
            const int cx = cell_of_fast(static_cast<double>(v[u].x), g.ox, g.cell, inv, g.n_cols);
            const int cy = cell_of_fast(static_cast<double>(v[u].y), g.oy, g.cell, inv, g.n_rows);
            atomicAdd(&hist[cy * g.n_cols + cx], 1);  // bin_grid.cpp:67
        }
    }
    __syncthreads();
    for (int k = tid; k < cells; k += blockDim.x) {
        const int h = hist[k];
        if (h != 0) atomicAdd(bins + g.bin_off + k, h);
    }
}

// Cell counts only (fire-and-forget reductions, no ranks stored): the fast
// path's count pass; k_scatter_emit recomputes the cell and takes its slot.
// Counts with 16-byte position loads (two points each) and kCountPer
// points per thread in flight: the count is a pure latency problem (its
// fire-and-forget RED.ADDs need no return).  N odd or unaligned positions:
// one point per load.
#ifndef GMI_K1_COUNT_PER
#define GMI_K1_COUNT_PER 4
#endif
constexpr int kCountPer = GMI_K1_COUNT_PER;
__global__ void __launch_bounds__(256) k_count_red(const float2* __restrict__ pos, int N,
                                                   const Geom* __restrict__ geom,
                                                   int32_t* __restrict__ bins) {
    const int b = blockIdx.y;
    const Geom g = geom[b];
    const double inv = 1.0 / g.cell;
    const size_t base = static_cast<size_t>(b) * N;
    const bool vec = (N % 2) == 0 && (reinterpret_cast<uintptr_t>(pos) & 15) == 0;
    if (vec) {
        const float4* p4 = reinterpret_cast<const float4*>(pos + base);
        const int k0 = blockIdx.x * (blockDim.x * kCountPer / 2) + threadIdx.x;
        float4 v[kCountPer / 2];
#pragma unroll
        for (int u = 0; u < kCountPer / 2; ++u) {
            const int k = k0 + u * blockDim.x;
            if (2 * k < N) v[u] = p4[k];
        }
#pragma unroll
        for (int u = 0; u < kCountPer / 2; ++u) {
            const int k = k0 + u * blockDim.x;
            if (2 * k >= N) continue;
            const float xs[2] = {v[u].x, v[u].z}, ys[2] = {v[u].y, v[u].w};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cx = cell_of_fast(static_cast<double>(xs[h]), g.ox, g.cell, inv, g.n_cols);
                const int cy = cell_of_fast(static_cast<double>(ys[h]), g.oy, g.cell, inv, g.n_rows);
                atomicAdd(bins + g.bin_off + cy * g.n_cols + cx, 1);  // bin_grid.cpp:67
            }
        }
        return;
    }
    const int i0 = blockIdx.x * (blockDim.x * kCountPer) + threadIdx.x;
    float2 v[kCountPer];
#pragma unroll
    for (int u = 0; u < kCountPer; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < N) v[u] = pos[base + i];
    }
#pragma unroll
    for (int u = 0; u < kCountPer; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < N) {
            const int cx = cell_of_fast(static_cast<double>(v[u].x), g.ox, g.cell, inv, g.n_cols);
            const int cy = cell_of_fast(static_cast<double>(v[u].y), g.oy, g.cell, inv, g.n_rows);
            atomicAdd(bins + g.bin_off + cy * g.n_cols + cx, 1);  // bin_grid.cpp:67
        }
    }
}

// k_count with 4 points per thread: 4 independent position loads and cell
// atomics in flight per thread (the single-point kernel is latency bound).
__global__ void __launch_bounds__(256) k_count4(const float2* __restrict__ pos, int N,
                                                const Geom* __restrict__ geom,
                                                int32_t* __restrict__ bins,
                                                int32_t* __restrict__ cellid,
                                                int32_t* __restrict__ rank) {
    const int b = blockIdx.y;
    const Geom g = geom[b];
    const double inv = 1.0 / g.cell;
    const size_t base = static_cast<size_t>(b) * N;
    const int i0 = blockIdx.x * (blockDim.x * kEmitPer) + threadIdx.x;
    float2 v[kEmitPer];
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < N) v[u] = pos[base + i];
    }
    int bin[kEmitPer], r[kEmitPer];
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < N) {
            const int cx = cell_of_fast(static_cast<double>(v[u].x), g.ox, g.cell, inv, g.n_cols);
            const int cy = cell_of_fast(static_cast<double>(v[u].y), g.oy, g.cell, inv, g.n_rows);
            bin[u] = cy * g.n_cols + cx;  // bin_grid.cpp:67
            r[u] = atomicAdd(bins + g.bin_off + bin[u], 1);
        }
    }
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < N) {
            cellid[base + i] = bin[u];
            rank[base + i] = r[u];
        }
    }
}

}  // namespace

namespace gmi_host {

// axis_cells (bin_grid.cpp:18-24) with a configurable cap
int host_axis_cells(double span, double cell, int cap) {
    const double ideal = std::ceil(span / cell) + 2.0;
    if (!(ideal < static_cast<double>(cap))) return cap;
    const int v = gmi_dev::x86_d2i(ideal);
    return std::max(1, v);
}

// Scan tiles over segments [seg_start[b], seg_start[b] + seg_len[b]).
// `equal`: all segments have the same length (device geometry); the tile
// table then depends only on (B, stride) and is cached in the context.
// inclusive: data[k] = sum of counts [0, k] (cell ends), else exclusive.
static void scan_segments(gmi_ctx* ctx, int32_t* data, const std::vector<int64_t>& seg_start,
                          const std::vector<int64_t>& seg_len, bool equal = false,
                          bool inclusive = false, const gmi_dev::Geom* geom = nullptr,
                          int2* big = nullptr, int32_t* big_count = nullptr) {
    cudaStream_t st = ctx->stream;
    const int B = static_cast<int>(seg_start.size());
    if (equal && ctx->eq_B == B && ctx->eq_stride == seg_len[0]) {
        const int nt = ctx->eq_nt;
        ScanTile* d_tiles = static_cast<ScanTile*>(ctx->ws_ptr[WS_TILES_EQ]);
        int32_t* d_segoff = static_cast<int32_t*>(ctx->ws_ptr[WS_SEGOFF_EQ]);
        int32_t* d_tsum = static_cast<int32_t*>(scratch(ctx, WS_TSUM, sizeof(int32_t) * nt));
        k_scan_reduce<<<nt, kScanThreads, 0, st>>>(data, d_tiles, d_tsum, geom, big, big_count);
        GMI_LAUNCHED(ctx);
        k_scan_segments<<<B, 1024, 0, st>>>(d_tsum, d_segoff);
        GMI_LAUNCHED(ctx);
        k_scan_apply<<<nt, kScanThreads, 0, st>>>(data, d_tiles, d_tsum, inclusive ? 1 : 0);
        GMI_LAUNCHED(ctx);
        return;
    }
    std::vector<ScanTile> tiles;
    std::vector<int32_t> seg_off(B + 1, 0);
    for (int b = 0; b < B; ++b) {
        for (int64_t s = 0; s < seg_len[b]; s += kScanTile)
            tiles.push_back({seg_start[b] + s,
                             static_cast<int32_t>(std::min<int64_t>(kScanTile, seg_len[b] - s)), b});
        seg_off[b + 1] = static_cast<int32_t>(tiles.size());
    }
    const int nt = static_cast<int>(tiles.size());
    ScanTile* d_tiles = static_cast<ScanTile*>(
        scratch(ctx, equal ? WS_TILES_EQ : WS_TILES, sizeof(ScanTile) * nt));
    int32_t* d_tsum = static_cast<int32_t*>(scratch(ctx, WS_TSUM, sizeof(int32_t) * nt));
    int32_t* d_segoff = static_cast<int32_t*>(
        scratch(ctx, equal ? WS_SEGOFF_EQ : WS_SEGOFF, sizeof(int32_t) * (B + 1)));
    if (equal) {
        ctx->eq_B = B;
        ctx->eq_stride = seg_len[0];
        ctx->eq_nt = nt;
    }
    GMI_CUDA(cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(ScanTile) * nt,
                             cudaMemcpyHostToDevice, st));
    GMI_CUDA(cudaMemcpyAsync(d_segoff, seg_off.data(), sizeof(int32_t) * (B + 1),
                             cudaMemcpyHostToDevice, st));
    k_scan_reduce<<<nt, kScanThreads, 0, st>>>(data, d_tiles, d_tsum, geom, big, big_count);
    GMI_LAUNCHED(ctx);
    k_scan_segments<<<B, 1024, 0, st>>>(d_tsum, d_segoff);
    GMI_LAUNCHED(ctx);
    k_scan_apply<<<nt, kScanThreads, 0, st>>>(data, d_tiles, d_tsum, inclusive ? 1 : 0);
    GMI_LAUNCHED(ctx);
}

void bin_points(gmi_ctx* ctx, gmi_cache* c, const float* pos, const float* col,
                int cap, bool hot, int32_t* point_index_out,
                unsigned long long* d_issue) {
    const int B = c->B, N = c->N;
    const double cell = c->cutoff;
    cudaStream_t st = ctx->stream;
    const float2* p2 = reinterpret_cast<const float2*>(pos);

    // ---- bbox + position validation ----
    uint32_t* d_bbox = static_cast<uint32_t*>(scratch(ctx, WS_BBOX, sizeof(uint32_t) * 4 * B));
    k_bbox_init<<<(B + 127) / 128, 128, 0, st>>>(d_bbox, d_issue, B);
    GMI_LAUNCHED(ctx);
#ifndef GMI_K1_BBOX_SCALAR
    if ((N % 2) == 0 && (reinterpret_cast<uintptr_t>(pos) & 15) == 0) {
        const int per_img = (N / 2 + 256 * kBboxPer - 1) / (256 * kBboxPer);
        k_bbox_validate4<<<dim3(per_img, B), 256, 0, st>>>(reinterpret_cast<const float4*>(pos), N,
                                                          d_bbox, d_issue);
        GMI_LAUNCHED(ctx);
    } else
#endif
    {
        const int per_img = std::max(1, std::min((N + 1023) / 1024,
                                                 (4 * ctx->num_sms + B - 1) / B));
        k_bbox_validate<<<dim3(per_img, B), 256, 0, st>>>(p2, N, d_bbox, d_issue);
        GMI_LAUNCHED(ctx);
    }
    c->geom_d = static_cast<gmi_dev::Geom*>(cache_alloc(c, sizeof(gmi_dev::Geom) * B));
    std::vector<int64_t> seg_start(B), seg_len(B);
    int max_bins = 0;
    // device geometry (no host round trip) when the frame-derived bin array
    // stays small; otherwise the exact host geometry with the reference cap
    const int64_t cells = static_cast<int64_t>(cap) * cap;
    if (hot && cells <= (int64_t(1) << 24) && cells * B <= (int64_t(1) << 27)) {
        const int64_t stride = cells + 1;
        c->geom_h.clear();
        c->grid_cap = cap;
        c->grid_stride = stride;
        k_geom<<<(B + 127) / 128, 128, 0, st>>>(d_bbox, B, cell, cap, stride, c->geom_d);
        GMI_LAUNCHED(ctx);
        c->total_bins = stride * B;
        for (int b = 0; b < B; ++b) {
            seg_start[b] = b * stride;
            seg_len[b] = stride;
        }
        max_bins = static_cast<int>(cells);
    } else {
        if (hot) cap = std::max(cap, 2048);
        // one sync: sizes are data dependent exactly as in the reference
        std::vector<uint32_t> bbox(4 * B);
        std::vector<unsigned long long> issue(B);
        GMI_CUDA(cudaMemcpyAsync(bbox.data(), d_bbox, sizeof(uint32_t) * 4 * B,
                                 cudaMemcpyDeviceToHost, st));
        GMI_CUDA(cudaMemcpyAsync(issue.data(), d_issue, sizeof(unsigned long long) * B,
                                 cudaMemcpyDeviceToHost, st));
        GMI_CUDA(cudaStreamSynchronize(st));
        for (int b = 0; b < B; ++b) {
            if (issue[b] != kNoIssue) {
                const long idx = static_cast<long>(issue[b] >> 8);
                throw GmiFail{GMI_ERR_NON_FINITE_VALUE,
                              "non-finite position at index " + std::to_string(idx) +
                                  (B > 1 ? " (image " + std::to_string(b) + ")" : "")};
            }
        }
        // geometry (bin_grid.cpp:45-60), f64 on the host (IEEE, same ops)
        c->geom_h.resize(B);
        int64_t off = 0;
        for (int b = 0; b < B; ++b) {
            const double mnx = ord2f(bbox[4 * b + 0]), mny = ord2f(bbox[4 * b + 1]);
            const double mxx = ord2f(bbox[4 * b + 2]), mxy = ord2f(bbox[4 * b + 3]);
            gmi_dev::Geom g{};
            g.cell = cell;
            g.ox = mnx - cell;
            g.oy = mny - cell;
            g.n_cols = host_axis_cells(mxx - mnx, cell, cap);
            g.n_rows = host_axis_cells(mxy - mny, cell, cap);
            g.capped = (g.n_cols >= cap || g.n_rows >= cap) ? 1 : 0;
            g.bin_off = off;
            g.qx0 = static_cast<float>(g.ox);
            g.qscale = 2.0f;
            seg_start[b] = off;
            seg_len[b] = static_cast<int64_t>(g.n_cols) * g.n_rows + 1;
            off += seg_len[b];
            max_bins = std::max(max_bins, g.n_cols * g.n_rows);
            c->geom_h[b] = g;
        }
        c->total_bins = off;
        GMI_CUDA(cudaMemcpyAsync(c->geom_d, c->geom_h.data(), sizeof(gmi_dev::Geom) * B,
                                 cudaMemcpyHostToDevice, st));
    }
    c->bins = static_cast<int32_t*>(cache_alloc(c, sizeof(int32_t) * c->total_bins));
    GMI_CUDA(cudaMemsetAsync(c->bins, 0, sizeof(int32_t) * c->total_bins, st));

    // ---- count (atomic arrival rank in the cell) + segmented scan ----
    const size_t BN = static_cast<size_t>(B) * N;
    const dim3 pgrid((N + 255) / 256, B);
    const dim3 pgrid4((N + 256 * kEmitPer - 1) / (256 * kEmitPer), B);
    const bool classify = c->wsum64 == nullptr;
    if (hot && !c->sort_cells) {
        // fast path: counts -> inclusive scan (cell ends) -> 32-byte records
        // at slots taken from the ends, which leaves bin_start behind
        if (c->geom_h.empty() && static_cast<int64_t>(c->grid_cap) * c->grid_cap <= kCountSmemCells &&
            std::getenv("GMI_K1_COUNT_RED") == nullptr) {
            // every image's grid fits shared memory: private histograms,
            // about one wave of CTAs (slices of the images' points)
            const int parts = std::max(1, std::min((N + 8191) / 8192, (ctx->num_sms + B - 1) / B));
            const int smem = static_cast<int>(sizeof(int) * c->grid_cap * c->grid_cap);
            GMI_SMEM_ONCE(ctx, k_count_smem, kCountSmemCells * static_cast<int>(sizeof(int)));
            k_count_smem<<<dim3(parts, B), 1024, smem, st>>>(p2, N, c->geom_d, c->bins, parts);
        } else {
            k_count_red<<<dim3((N + 256 * kCountPer - 1) / (256 * kCountPer), B), 256, 0, st>>>(
                p2, N, c->geom_d, c->bins);
        }
        GMI_LAUNCHED(ctx);
        host_trace("bin: count launched");
        // cells the gather may split (> its chunk capacity) are listed by the
        // scan's reduce pass and put in index order after the scatter
        int2* d_big = static_cast<int2*>(
            scratch(ctx, WS_BIG, sizeof(int2) * std::max<size_t>(1, BN / (kBigRecCell + 1) + 1)));
        int32_t* d_bigcount = static_cast<int32_t*>(scratch(ctx, WS_BIGCOUNT, sizeof(int32_t)));
        GMI_CUDA(cudaMemsetAsync(d_bigcount, 0, sizeof(int32_t), st));
        scan_segments(ctx, c->bins, seg_start, seg_len, c->geom_h.empty(), true, c->geom_d, d_big,
                      d_bigcount);
        if (c->ccol == nullptr && slot_grads(N, c->C))
            c->inv = static_cast<int32_t*>(cache_alloc(c, sizeof(int32_t) * BN));
        ScatterEmitParams e{};
        e.pos = p2;
        e.col = col;
        e.geom = c->geom_d;
        e.bins = c->bins;
        e.rec = c->rec;
        e.ccol = c->ccol;
        e.issue = d_issue;
        e.inv = c->inv;
        e.N = N;
        e.C = c->C;
        e.classify = classify ? 1 : 0;
        e.rf = static_cast<float>(c->cutoff);
        e.r2f = static_cast<float>(c->cutoff * c->cutoff);
        k_scatter_emit<<<pgrid4, 256, 0, st>>>(e);
        GMI_LAUNCHED(ctx);
        // cells the gather may split: index order
        const int rsmem = kBigRecSmem * (2 * sizeof(float4) + sizeof(unsigned long long));
        GMI_SMEM_ONCE(ctx, k_sort_big_recs, rsmem);
        k_sort_big_recs<<<ctx->num_sms, 512, rsmem, st>>>(N, c->geom_d, c->bins, c->rec, d_big, d_bigcount,
                                                           c->inv);
        GMI_LAUNCHED(ctx);
        host_trace("bin: scatter_emit launched");
        return;
    }

    // ---- count (atomic arrival rank) + scan + scatter + per-cell index order
    // (the reference's point_index) ----
    int32_t* cellid = static_cast<int32_t*>(scratch(ctx, WS_CELLID, sizeof(int32_t) * BN));
    int32_t* rank = static_cast<int32_t*>(scratch(ctx, WS_RANK, sizeof(int32_t) * BN));
    k_count4<<<pgrid4, 256, 0, st>>>(p2, N, c->geom_d, c->bins, cellid, rank);
    GMI_LAUNCHED(ctx);
    host_trace("bin: count launched");
    scan_segments(ctx, c->bins, seg_start, seg_len, c->geom_h.empty());
    int32_t* tmp = static_cast<int32_t*>(scratch(ctx, WS_TMP, sizeof(int32_t) * BN));
    k_scatter<<<pgrid, 256, 0, st>>>(N, c->geom_d, c->bins, cellid, rank, tmp);
    GMI_LAUNCHED(ctx);
    int2* d_big = static_cast<int2*>(scratch(ctx, WS_BIG, sizeof(int2) * std::max<size_t>(1, BN / (kSmallCell + 1) + 1)));
    int32_t* d_bigcount = static_cast<int32_t*>(scratch(ctx, WS_BIGCOUNT, sizeof(int32_t)));
    GMI_CUDA(cudaMemsetAsync(d_bigcount, 0, sizeof(int32_t), st));
    k_cellsort_small<<<dim3((max_bins + 127) / 128, B), 128, 0, st>>>(N, c->geom_d, c->bins, tmp,
                                                                      d_big, d_bigcount);
    GMI_LAUNCHED(ctx);
    const int smem = kBigSmemKeys * sizeof(int);
    GMI_CUDA(cudaFuncSetAttribute(k_cellsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_cellsort_big<<<ctx->num_sms, 1024, smem, st>>>(N, c->geom_d, c->bins, tmp, d_big, d_bigcount);
    GMI_LAUNCHED(ctx);
    if (!hot) {
        GMI_CUDA(cudaMemcpyAsync(point_index_out, tmp, sizeof(int32_t) * BN, cudaMemcpyDeviceToDevice, st));
    } else if (c->rec != nullptr) {
        // wide-channel path: records + colours in index-ordered cells
        ScatterEmitParams e{};
        e.pos = p2;
        e.col = col;
        e.geom = c->geom_d;
        e.bins = c->bins;
        e.rec = c->rec;
        e.ccol = c->ccol;
        e.issue = d_issue;
        e.N = N;
        e.C = c->C;
        e.classify = classify ? 1 : 0;
        e.rf = static_cast<float>(c->cutoff);
        e.r2f = static_cast<float>(c->cutoff * c->cutoff);
        k_emit_rec<<<pgrid, 256, 0, st>>>(e, tmp);
        GMI_LAUNCHED(ctx);
    } else {
        EmitParams e{};
        e.pos = p2;
        e.col = col;
        e.tmp = tmp;
        e.sx = c->sx;
        e.sy = c->sy;
        e.sidx = c->sidx;
        e.scol = c->scol;
        e.issue = d_issue;
        e.N = N;
        e.C = c->C;
        // f64 weight mode decides every pair in f64: no classification needed
        e.classify = classify ? 1 : 0;
        e.rf = static_cast<float>(c->cutoff);
        e.r2f = static_cast<float>(c->cutoff * c->cutoff);
        k_emit<<<pgrid, 256, 0, st>>>(e);
        GMI_LAUNCHED(ctx);
    }
    host_trace("bin: scan..cellsort launched");
}

}  // namespace gmi_host
