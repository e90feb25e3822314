// K2 fast path — forward gather (engine.cpp:44-103 forward_rows +
// query_radius bin_grid.cpp:84-105 + gaussian_weight core.cpp:49-53) for the
// fp32 weight mode (cutoff <= 6 sigma) with C <= 4 channels.
//
// CTA = 64x32 output pixels of one image, 8 warps; warp w owns rows
// y0+4w .. y0+4w+3, lane l the columns (x0+2l, x0+2l+1): 2x4 pixels per
// thread whose normaliser W and numerators live in f32x2 registers.  (Round
// 1 had 2x2 pixels per thread; the inner loop was bound by the shared-memory
// pipe — 80% of its wavefronts, half of them bank conflicts, from each lane
// reading its own candidate record — and one record read now serves 8
// pixels instead of 4: -13% gather time at configs[2].)
//
//  stage  The candidate points of the tile (reference cells overlapping the
//         tile grown by r: one contiguous run of 32-byte records per cell
//         row) arrive in shared memory by TMA — one cp.async.bulk per run,
//         completing on an mbarrier — and are counting-sorted there by
//         (1-px column, row-pair) bin into dense record arrays.  Bin geometry is exact (f64
//         differences of fp32 positions against integer / f64 anchors), so a
//         point that can reach the tile lands in the bins its pixels read.
//         Within a bin the order is canonicalised by original index, so the
//         summation order — and the result — is independent of K1's atomic
//         arrival order.
//  lists  Warp w needs the row-pair bins [2w, 2w + 1 + dyb] of every column:
//         per column one contiguous piece of the sorted array.  Lane-per-column
//         prefix sums give the warp's column-major index list and its column
//         starts; a lane's candidates (mu_x in (xa - r, xa + 1 + r)) are then
//         ONE contiguous range of that list.
//  gather Per candidate, 8 pixels with f32x2 ops: e = nk d^2, in-ball test
//         e >= nk r^2 (exact in fp32 for points K1 did not flag, see
//         gmi_common.cuh), 8 MUFU.EX2, W and C numerators.  Flagged
//         (boundary-ambiguous) points sit in one extra bin and take the f64
//         predicate in a warp-uniform pass.
//  store  out = num/W with one Newton step, W kept for the backward; pixels
//         with W == 0 go to the fallback list (K3).  Clustered tiles (several
//         staging chunks) fold their sums into f64 at each chunk end.
#include <algorithm>
#include <cmath>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

// rows per lane (each lane owns 2 columns x kRPL rows): 4 halves the shared-
// memory traffic per pixel evaluation against 2 (one staged candidate read
// serves 8 pixels); 2 is round 1's layout, kept for A/B builds
#ifndef GMI_GATHER_RPL
#define GMI_GATHER_RPL 4
#endif
constexpr int kRPL = GMI_GATHER_RPL;
constexpr int kNW = 8;             // warps
constexpr int kTW = 64, kTH = kNW * kRPL;
constexpr int kNT = kNW * 32;      // threads
constexpr int kCTAs = kRPL == 2 ? 4 : 3;  // resident CTAs per SM (registers, shared memory)
// staged candidates per chunk (>= K1's kBigRecCell: cells above it are
// index-ordered, so chunk membership never depends on arrival order)
constexpr int kCap = kRPL == 2 ? 640 : 1024;
constexpr int kRsMax = 32;         // cell-row runs per chunk
constexpr int kColMax = 128;       // 1-px columns across the tile's reach
constexpr int kBinMax = 2048;      // (column, row-pair) bins (+1 flag bin)
constexpr int kMultiCap = kNW * (kColMax + 1);  // multi-bin list, shares wcs
#ifndef GMI_GATHER_UNROLL
#define GMI_GATHER_UNROLL 1
#endif
constexpr int kLoopUnroll = GMI_GATHER_UNROLL;  // candidate loop unroll

template <int CC>
struct SmemGather {
    union {
        // the chunk's 32-byte records in run order, bulk-copied by TMA:
        // R[2k] = (x, y, c0, c1), R[2k+1] = (c2, c3, idx | flag, 0)
        float4 R[2 * kCap];
        uint16_t wl[kNW][kCap];            // per-warp column-major lists (after C)
    } u;
    float4 A[kCap];                        // mu_x, mu_y, c0, c1   (bin order)
    float2 Bc[CC > 2 ? kCap : 1];          // c2, c3
    int idx[kCap];                         // original index
    int bin[kBinMax + 2];                  // counts -> inclusive ends -> starts
    union {
        uint16_t wcs[kNW][kColMax + 1];    // per-warp column starts in wl
        uint16_t multi[kMultiCap];         // bins with >= 2 candidates (B..D)
    } v;
    int run_beg[kRsMax + 1];
    int run_g[kRsMax];
    int scan_w[kNW];
    int n_multi;
    int n_runs, cur_cy, cur_off, done, pre;
    int fold_slot;                         // multi-chunk tiles: f64 fold slot (-1: none)
    int cx0, cx1, cy1;
    unsigned long long mbar;               // TMA completion barrier
};

struct GatherParams {
    const Geom* geom;
    const int32_t* bins;
    const float4* rec;  // [B][N][2]: (x, y, c0, c1) (c2, c3, idx|flag, 0)
    int N, C, W, H;
    int ncol, nyb, dyb, rc;   // bin geometry (see launch_gather_fast)
    uint8_t qlo[32], qhi[32]; // per-lane column window [qlo, qhi]
    double r64, r2_64;
    float r2f, nk, thr;
    float* image;
    float* wsum;
    int32_t* counts;
    Special* special;
    int32_t* special_count;
    int special_cap;
    // multi-chunk (clustered) tiles fold their fp32 sums into private f64
    // totals at every chunk end: [slot][16][thread], slots from fold_count
    double* fold;
    int32_t* fold_count;
    int fold_cap;
};

constexpr int kFoldVals = 8 * kRPL;  // W and up to 3 numerators x 2 kRPL pixels (C <= 3)

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int CC, bool kCount>
__global__ void __launch_bounds__(kNT, kCTAs)
k_gather(GatherParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemGather<CC>& S = *reinterpret_cast<SmemGather<CC>*>(smem_raw);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = static_cast<int>(blockIdx.z);
    const int y0 = blockIdx.y * kTH;
    const int x0 = blockIdx.x * kTW;
    const size_t base = static_cast<size_t>(b) * p.N;
    const int ncol = p.ncol, nyb = p.nyb, nbins = ncol * nyb;
    // bin anchors: column = floor(mu_x - cxo), row pair = floor((mu_y - cyo)/2);
    // tile region and its reference cells (bin_grid.cpp:88-91 for the tile).
    // Recomputed from the parameters where used (not held in registers
    // across the candidate loop).
#define GMI_TILE_CXO (static_cast<double>(x0 - p.rc))
#define GMI_TILE_CYO (static_cast<double>(y0) - p.r64)
#define GMI_TILE_XLO (static_cast<double>(x0) - p.r64)
#define GMI_TILE_XHI (static_cast<double>(x0 + kTW - 1) + p.r64)
#define GMI_TILE_YLO (static_cast<double>(y0) - p.r64)
#define GMI_TILE_YHI (static_cast<double>(y0 + kTH - 1) + p.r64)

    // this thread's 2 x kRPL pixels: columns xa, xa + 1 of rows ya .. ya + kRPL - 1
    const int ya = y0 + kRPL * warp, xa = x0 + 2 * lane;
    const float2 X = f2(static_cast<float>(xa), static_cast<float>(xa + 1));
    float2 Y[kRPL / 2];  // row pairs (ya + 2j, ya + 2j + 1)
#pragma unroll
    for (int j = 0; j < kRPL / 2; ++j)
        Y[j] = f2(static_cast<float>(ya + 2 * j), static_cast<float>(ya + 2 * j + 1));
    const float2 nk2 = f2(p.nk, p.nk);
    const float thr = p.thr;
    float2 Wr[kRPL];       // per row: (xa, xa + 1)
    float2 Nr[kRPL][CC];
    int cnt[kRPL][2];
#pragma unroll
    for (int r = 0; r < kRPL; ++r) {
        Wr[r] = f2(0.f, 0.f);
        cnt[r][0] = cnt[r][1] = 0;
#pragma unroll
        for (int c = 0; c < CC; ++c) Nr[r][c] = f2(0.f, 0.f);
    }
    // the lane's column window (columns of mu_x in (xa - r, xa + 1 + r),
    // exact in f64, tabulated per lane on the host: p.qlo / p.qhi) and the
    // flagged points' generous band (fb_lo / fb_hi, decided exactly by the
    // f64 predicate) are read where used: registers are the candidate loop's
    const uint32_t mbar = smem_u32(&S.mbar);
    uint32_t phase = 0;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        // the f64 cell rectangle (four lanes in parallel)
        // one convergent call: lane 0/1 -> x bounds, lane 2/3 -> y bounds
        const Geom g = p.geom[b];
        const bool ax = lane < 2;
        const int cv = cell_of(ax ? ((lane & 1) ? GMI_TILE_XHI : GMI_TILE_XLO)
                                  : ((lane & 1) ? GMI_TILE_YHI : GMI_TILE_YLO),
                               ax ? g.ox : g.oy, g.cell, ax ? g.n_cols : g.n_rows);
        const int cx0 = __shfl_sync(0xffffffffu, cv, 0), cx1 = __shfl_sync(0xffffffffu, cv, 1);
        const int cy0 = __shfl_sync(0xffffffffu, cv, 2), cy1 = __shfl_sync(0xffffffffu, cv, 3);
        // common case: <= 32 cell rows and <= kCap candidates -> one chunk,
        // runs loaded by one lane each
        const int nrows = cy1 - cy0 + 1;
        bool one = false;
        if (nrows <= 32 && nrows <= kRsMax) {
            int gs = 0, len = 0;
            if (lane < nrows) {
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cy0 + lane) * g.n_cols;
                gs = p.bins[r0 + cx0];
                len = p.bins[r0 + cx1 + 1] - gs;
            }
            int incl = len;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            if (tot <= kCap) {
                one = true;
                if (lane < nrows) {
                    S.run_g[lane] = gs;
                    S.run_beg[lane] = incl - len;
                }
                if (lane == 0) {
                    S.run_beg[nrows] = tot;
                    S.n_runs = nrows;
                    S.pre = 1;
                }
            }
        }
        if (lane == 0) {
            S.cx0 = cx0;
            S.cx1 = cx1;
            S.cy1 = cy1;
            S.cur_cy = one ? cy1 + 1 : cy0;
            S.cur_off = 0;
            S.done = one ? 1 : 0;
            if (!one) S.pre = 0;
            int fs = -1;
            if (!one && CC <= 3 && p.fold != nullptr) {
                fs = atomicAdd(p.fold_count, 1);
                if (fs >= p.fold_cap) fs = -1;
            }
            S.fold_slot = fs;
        }
    }
    __syncthreads();
    // Clustered tiles (several chunks) sum thousands of candidates per pixel:
    // a plain fp32 running sum drifts by ~sqrt(n/3) ulp.  Their threads fold
    // the chunk's fp32 sums into private f64 totals at every chunk end, in
    // chunk order (deterministic), and normalise in f64.
    double* const fold = S.fold_slot >= 0
                             ? p.fold + static_cast<size_t>(S.fold_slot) * kFoldVals * kNT + tid
                             : nullptr;
    bool folded = false;
    auto fold_acc = [&](float& a, int k) {
        double* f = fold + static_cast<size_t>(k) * kNT;
        *f = (folded ? *f : 0.0) + static_cast<double>(a);
        a = 0.f;
    };
    while (true) {
        // ---- next chunk of runs (<= kRsMax runs, <= kCap candidates) ----
        if (tid == 0 && S.pre) {
            S.pre = 0;  // the single chunk was prepared above
        } else if (tid == 0) {
            const int cx0 = S.cx0, cx1 = S.cx1, cy1 = S.cy1;
            int n = 0, tot = 0, cy = S.cur_cy, off = S.cur_off;
            while (cy <= cy1 && n < kRsMax && tot < kCap) {
                const Geom& g = p.geom[b];  // (multi-chunk tiles only: reloaded)
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cy) * g.n_cols;
                const int gs = p.bins[r0 + cx0] + off, ge = p.bins[r0 + cx1 + 1];
                if (ge <= gs) {
                    ++cy;
                    off = 0;
                    continue;
                }
                int take = ge - gs;
                if (take > kCap - tot) {
                    // split at a cell boundary (chunk membership must not
                    // depend on K1's arrival order inside a cell): the
                    // longest prefix of whole cells that fits
                    const int room = kCap - tot;
                    int e = gs;
                    for (int cx = cx0 + 1; cx <= cx1 + 1; ++cx) {
                        const int bnd = p.bins[r0 + cx];
                        if (bnd - gs > room) break;
                        e = max(e, bnd);
                    }
                    if (e > gs) take = e - gs;
                    else if (tot > 0) break;  // the next cell opens the next chunk
                    else take = kCap;         // one cell > kCap: index-ordered by K1
                }
                S.run_g[n] = gs;
                S.run_beg[n] = tot;
                tot += take;
                ++n;
                if (take == ge - gs) {
                    ++cy;
                    off = 0;
                } else {
                    off += take;
                }
            }
            S.run_beg[n] = tot;
            S.n_runs = n;
            S.cur_cy = cy;
            S.cur_off = off;
            S.done = cy > cy1;
        }
        for (int k = tid; k <= nbins + 1; k += kNT) S.bin[k] = 0;
        if (tid == 0) S.n_multi = 0;
        __syncthreads();
        const int n_runs = S.n_runs;
        if (n_runs == 0) break;
        const int total = S.run_beg[n_runs];

        // ---- stage: one TMA bulk copy per run of consecutive records ----
        if (warp == 0) {
            if (lane == 0) {
                // order the previous chunk's generic reads of R before the
                // async-proxy writes, then announce the chunk's bytes
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(mbar), "r"(static_cast<uint32_t>(total) * 32u) : "memory");
            }
            __syncwarp();
            if (lane < n_runs) {
                const int rb = S.run_beg[lane], len = S.run_beg[lane + 1] - rb;
                GMI_CHECK(rb >= 0 && len >= 0 && rb + len <= kCap);
                if (len > 0)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        ::"r"(smem_u32(&S.u.R[2 * rb])), "l"(p.rec + (base + S.run_g[lane]) * 2),
                          "r"(static_cast<uint32_t>(len) * 32u), "r"(mbar)
                        : "memory");
            }
        }
        {
            uint32_t ok = 0;
            while (!ok) {
                asm volatile(
                    "{\n\t.reg .pred P1;\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                    "selp.b32 %0, 1, 0, P1;\n\t}"
                    : "=r"(ok) : "r"(mbar), "r"(phase) : "memory");
            }
            phase ^= 1u;
        }

        // ---- A: bin of every staged candidate + histogram ----
        for (int k = tid; k < total; k += kNT) {
            const float4 ra = S.u.R[2 * k];
            const float mx = ra.x, my = ra.y;
            const bool flag = (__float_as_uint(S.u.R[2 * k + 1].z) & kUnsafeBit) != 0;
            int key = -1;
            const double dx = static_cast<double>(mx) - GMI_TILE_CXO;
            const double dy = static_cast<double>(my) - GMI_TILE_CYO;
            if (!flag) {
                if (dx >= 0.0 && dy >= 0.0) {
                    const double qf = floor(dx), yf = floor(dy * 0.5);
                    if (qf < ncol && yf < nyb)
                        key = static_cast<int>(qf) * nyb + static_cast<int>(yf);
                }
            } else if (static_cast<double>(mx) >= GMI_TILE_XLO - 1.0 &&
                       static_cast<double>(mx) <= GMI_TILE_XHI + 1.0 &&
                       static_cast<double>(my) >= GMI_TILE_YLO - 1.0 &&
                       static_cast<double>(my) <= GMI_TILE_YHI + 1.0) {
                key = nbins;  // the flag bin
            }
            GMI_CHECK(key <= nbins && nbins + 1 < kBinMax + 2);
            if (key >= 0) atomicAdd(&S.bin[key], 1);
            S.u.R[2 * k + 1].w = __int_as_float(key);
        }
        __syncthreads();

        // ---- B: inclusive scan of the nbins + 1 counts (ends) ----
        {
            constexpr int kPer = (kBinMax + 1 + kNT - 1) / kNT;
            const int nb = nbins + 1;
            const int k0 = tid * kPer;
            int v[kPer];
            int s = 0;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                v[j] = (k0 + j < nb) ? S.bin[k0 + j] : 0;
                s += v[j];
            }
            int incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) S.scan_w[warp] = incl;
            __syncthreads();
            int run = incl - s;
            for (int w = 0; w < warp; ++w) run += S.scan_w[w];
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                run += v[j];
                if (k0 + j < nb) S.bin[k0 + j] = run;
                // bins holding 2+ candidates need the canonical-order pass
                if (v[j] > 1) {
                    const int m = atomicAdd(&S.n_multi, 1);
                    if (m < kMultiCap) S.v.multi[m] = static_cast<uint16_t>(k0 + j);
                }
            }
            if (tid == kNT - 1) S.bin[nb] = run;  // total kept
        }
        __syncthreads();

        // ---- C: scatter into bin order, dense (ends -> starts by decrement) ----
        for (int k = tid; k < total; k += kNT) {
            const int key = __float_as_int(S.u.R[2 * k + 1].w);
            if (key < 0) continue;
            const int pos = atomicSub(&S.bin[key], 1) - 1;
            GMI_CHECK(pos >= 0 && pos < kCap);
            const float4 ra = S.u.R[2 * k];
            const float4 rb = S.u.R[2 * k + 1];
            S.A[pos] = ra;
            if (CC > 2) S.Bc[pos] = f2(rb.x, rb.y);
            S.idx[pos] = static_cast<int>(__float_as_uint(rb.z) & 0x7fffffffu);
        }
        __syncthreads();

        // ---- D: canonical order inside each bin (ascending original index) ----
        const int n_multi = S.n_multi;
        const int n_sort = n_multi <= kMultiCap ? n_multi : nbins + 1;  // overflow: every bin
        for (int m = tid; m < n_sort; m += kNT) {
            const int k = n_multi <= kMultiCap ? S.v.multi[m] : m;
            const int s = S.bin[k], e = S.bin[k + 1];
            for (int i = s + 1; i < e; ++i) {
                const int vi = S.idx[i];
                if (S.idx[i - 1] <= vi) continue;
                const float4 va = S.A[i];
                const float2 vb = CC > 2 ? S.Bc[i] : f2(0.f, 0.f);
                int j = i;
                while (j > s && S.idx[j - 1] > vi) {
                    S.idx[j] = S.idx[j - 1];
                    S.A[j] = S.A[j - 1];
                    if (CC > 2) S.Bc[j] = S.Bc[j - 1];
                    --j;
                }
                S.idx[j] = vi;
                S.A[j] = va;
                if (CC > 2) S.Bc[j] = vb;
            }
        }
        __syncthreads();

        // ---- E: this warp's column-major list (row-pair bins [w, w+dyb]) ----
        {
            const int yb0 = warp * (kRPL / 2), yb1 = min(yb0 + kRPL / 2 - 1 + p.dyb, nyb - 1);
            // columns [c0, c1) of this lane: ncol spread evenly over the warp
            constexpr int kCpl = kColMax / 32;
            const int c0 = (lane * ncol) >> 5, c1 = ((lane + 1) * ncol) >> 5;
            int ps[kCpl], pl[kCpl];
            int s = 0;
#pragma unroll
            for (int j = 0; j < kCpl; ++j) {
                const int q = c0 + j;
                ps[j] = 0;
                pl[j] = 0;
                if (q < c1) {
                    ps[j] = S.bin[q * nyb + yb0];
                    pl[j] = S.bin[q * nyb + yb1 + 1] - ps[j];
                }
                s += pl[j];
            }
            int incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            int at = incl - s;
            uint16_t* wl = S.u.wl[warp];
#pragma unroll
            for (int j = 0; j < kCpl; ++j) {
                const int q = c0 + j;
                GMI_CHECK(q >= c1 || (q <= kColMax && at + pl[j] <= kCap));
                if (q < c1) S.v.wcs[warp][q] = static_cast<uint16_t>(at);
                for (int e = 0; e < pl[j]; ++e) wl[at + e] = static_cast<uint16_t>(ps[j] + e);
                at += pl[j];
            }
            if (lane == 31) S.v.wcs[warp][ncol] = static_cast<uint16_t>(at);
        }
        __syncwarp();

        // ---- gather: 2 x kRPL pixels per candidate, f32x2 ----
        {
            const int ts = S.v.wcs[warp][p.qlo[lane]], te = S.v.wcs[warp][p.qhi[lane] + 1];
            const uint16_t* lst = S.u.wl[warp];
            // the candidate's list entry loaded in its own iteration (a
            // one-ahead prefetch cost a register and a select: 1.625 vs 1.610 ms)
#pragma unroll kLoopUnroll
            for (int t = ts; t < te; ++t) {
                const int kc = lst[t];
                GMI_CHECK(kc >= 0 && kc < kCap && t < kCap);
                const float4 a = S.A[kc];
                const float2 bcur = CC > 2 ? S.Bc[kc] : f2(0.f, 0.f);
                const float2 dx = __fadd2_rn(X, f2(-a.x, -a.x));
                const float2 kx = __fmul2_rn(dx, nk2);

#pragma unroll
                for (int j = 0; j < kRPL / 2; ++j) {
                    const float2 dy = __fadd2_rn(Y[j], f2(-a.y, -a.y));
                    const float2 ey = __fmul2_rn(__fmul2_rn(dy, nk2), dy);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = 2 * j + h;
                        const float2 e = __ffma2_rn(kx, dx, h ? f2(ey.y, ey.y) : f2(ey.x, ey.x));
                        const bool i0 = e.x >= thr, i1 = e.y >= thr;
                        const float2 w = f2(i0 ? ex2(e.x) : 0.f, i1 ? ex2(e.y) : 0.f);
                        Wr[r] = __fadd2_rn(Wr[r], w);
#pragma unroll
                        for (int c = 0; c < CC; ++c) {
                            const float cc = c == 0 ? a.z : (c == 1 ? a.w : (c == 2 ? bcur.x : bcur.y));
                            Nr[r][c] = __ffma2_rn(w, f2(cc, cc), Nr[r][c]);
                        }
                        if (kCount) {
                            cnt[r][0] += i0;
                            cnt[r][1] += i1;
                        }
                    }
                }
            }
        }

        // ---- boundary-ambiguous points: f64 predicate (rare), index order ----
        {
            const int fs = S.bin[nbins], fe = S.bin[nbins + 1];
            const float fb_lo = static_cast<float>(ya) - static_cast<float>(p.r64) - 1.0f;
            const float fb_hi = static_cast<float>(ya + kRPL - 1) + static_cast<float>(p.r64) + 1.0f;
            for (int kk = fs; kk < fe; ++kk) {
                const float4 a = S.A[kk];
                if (!(a.y >= fb_lo && a.y <= fb_hi)) continue;  // warp-uniform
                float cc[4] = {a.z, a.w, 0.f, 0.f};
                if (CC > 2) {
                    const float2 bc = S.Bc[kk];
                    cc[2] = bc.x;
                    cc[3] = bc.y;
                }
#pragma unroll
                for (int r = 0; r < kRPL; ++r) {
#pragma unroll
                    for (int px = 0; px < 2; ++px) {
                        const int qx = xa + px, qy = ya + r;
                        if (d2_ref(qx, qy, a.x, a.y) > p.r2_64) continue;
                        const float ddx = static_cast<float>(qx) - a.x;
                        const float ddy = static_cast<float>(qy) - a.y;
                        const float w = ex2(fmaf(ddx * p.nk, ddx, (ddy * p.nk) * ddy));
                        if (px) Wr[r].y += w; else Wr[r].x += w;
#pragma unroll
                        for (int c = 0; c < CC; ++c) {
                            if (px) Nr[r][c].y = fmaf(w, cc[c], Nr[r][c].y);
                            else Nr[r][c].x = fmaf(w, cc[c], Nr[r][c].x);
                        }
                        if (kCount) ++cnt[r][px];
                    }
                }
            }
        }
        if (fold != nullptr) {
            // value k: W of pixel (row r, column h) at 2 r + h, numerator c
            // at 2 kRPL (c + 1) + 2 r + h
#pragma unroll
            for (int r = 0; r < kRPL; ++r) {
                fold_acc(Wr[r].x, 2 * r);
                fold_acc(Wr[r].y, 2 * r + 1);
#pragma unroll
                for (int c = 0; c < CC && c < 3; ++c) {
                    fold_acc(Nr[r][c].x, 2 * kRPL * (c + 1) + 2 * r);
                    fold_acc(Nr[r][c].y, 2 * kRPL * (c + 1) + 2 * r + 1);
                }
            }
            folded = true;
        }
        // the last chunk needs no barrier: a warp that is done goes straight
        // to its epilogue instead of waiting for the CTA's longest window
        // (S.done was published before this chunk's first barrier)
        if (S.done) break;
        __syncthreads();
    }

    // ---- fused normalisation + store (engine.cpp:74-100) ----
    // out = num / W with one Newton step; W kept for the backward
    auto norm = [](float num, float w, float inv) {
        const float q0 = num * inv;
        return fmaf(fmaf(-q0, w, num), inv, q0);
    };
    if (fold != nullptr && folded) {
        // folded tile: W and out = num / W from the f64 totals
#pragma unroll
        for (int pk = 0; pk < 2 * kRPL; ++pk) {
            const int r = pk >> 1, px = pk & 1;
            const int qx = xa + px, qy = ya + r;
            if (qx >= p.W || qy >= p.H) continue;
            const double w64 = fold[static_cast<size_t>(pk) * kNT];
            const size_t bp = (static_cast<size_t>(b) * p.H + qy) * p.W + qx;
            float* out = p.image + bp * p.C;
            if (w64 > 0.0) {
#pragma unroll
                for (int c = 0; c < CC; ++c)
                    out[c] = static_cast<float>(fold[static_cast<size_t>(2 * kRPL * (c + 1) + pk) * kNT] / w64);
                p.wsum[bp] = static_cast<float>(w64);
                if (kCount) p.counts[bp] = cnt[r][px];
            } else {
                p.wsum[bp] = 0.f;
                if (kCount) p.counts[bp] = 0;
                const int slot = atomicAdd(p.special_count, 1);
                if (slot < p.special_cap)
                    p.special[slot] = Special{b, static_cast<int32_t>(qy * p.W + qx), -1, 1};
            }
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < kRPL; ++r) {
        const int qy = ya + r;
        const float2 wr = Wr[r];
        // both pixels inside and non-fallback, 8-byte aligned: 64-bit stores
        // of the pixel pair
        const size_t bpr = (static_cast<size_t>(b) * p.H + qy) * p.W + xa;
        const bool al = ((reinterpret_cast<uintptr_t>(p.image + bpr * CC) |
                          reinterpret_cast<uintptr_t>(p.wsum + bpr)) & 7) == 0;
        if (qy < p.H && xa + 1 < p.W && wr.x > 0.f && wr.y > 0.f && !kCount && al) {
            const float ia = 1.0f / wr.x, ib = 1.0f / wr.y;
            float o[2 * CC];
#pragma unroll
            for (int c = 0; c < CC; ++c) {
                const float2 nm = Nr[r][c];
                o[c] = norm(nm.x, wr.x, ia);
                o[CC + c] = norm(nm.y, wr.y, ib);
            }
            float2* out2 = reinterpret_cast<float2*>(p.image + bpr * CC);
#pragma unroll
            for (int j = 0; j < CC; ++j) out2[j] = f2(o[2 * j], o[2 * j + 1]);
            *reinterpret_cast<float2*>(p.wsum + bpr) = wr;
            continue;
        }
#pragma unroll
        for (int px = 0; px < 2; ++px) {
            const int qx = xa + px;
            if (qx >= p.W || qy >= p.H) continue;
            const float w = px ? wr.y : wr.x;
            const size_t bp = (static_cast<size_t>(b) * p.H + qy) * p.W + qx;
            float* out = p.image + bp * p.C;
            if (w > 0.f) {
                const float inv = 1.0f / w;
#pragma unroll
                for (int c = 0; c < CC; ++c) {
                    const float num = px ? Nr[r][c].y : Nr[r][c].x;
                    out[c] = norm(num, w, inv);
                }
                p.wsum[bp] = w;
                if (kCount) p.counts[bp] = cnt[r][px];
            } else {
                // empty neighbourhood: fallback pixel (K3)
                p.wsum[bp] = 0.f;
                if (kCount) p.counts[bp] = 0;
                const int slot = atomicAdd(p.special_count, 1);
                if (slot < p.special_cap)
                    p.special[slot] = Special{b, static_cast<int32_t>(qy * p.W + qx), -1, 1};
            }
        }
    }
}
#undef GMI_TILE_CXO
#undef GMI_TILE_CYO
#undef GMI_TILE_XLO
#undef GMI_TILE_XHI
#undef GMI_TILE_YLO
#undef GMI_TILE_YHI

template <int CC, bool kCount>
void launch_cc(gmi_ctx* ctx, const GatherParams& p, dim3 grid) {
    const int smem = static_cast<int>(sizeof(SmemGather<CC>));
    GMI_SMEM_ONCE(ctx, (k_gather<CC, kCount>), smem);
    k_gather<CC, kCount><<<grid, kNT, smem, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

}  // namespace

namespace gmi_host {

static void gather_geometry(double r, int& rc, int& ncol, int& dyb, int& nyb) {
    // columns: floor(mu_x - (x0 - rc)), rc = ceil(r); lane windows are the
    // columns of (xa - r, xa + 1 + r), so ncol covers the last lane's
    rc = static_cast<int>(std::ceil(r));
    ncol = static_cast<int>(std::ceil(static_cast<double>(kTW - 2 + rc + 1) + r));
    // row pairs: floor((mu_y - (y0 - r)) / 2); warp w (rows y0 + kRPL w ..
    // + kRPL - 1) reads [w kRPL/2, w kRPL/2 + kRPL/2 - 1 + dyb]
    dyb = static_cast<int>(std::ceil(0.5 + r)) - 1;
    nyb = kNW * (kRPL / 2) + dyb;
}

// The fast gather applies: fp32 weight mode and a bin table that fits.
// C > 4 takes the wide-channel gather (gmi_wide.cu), which stages by cell
// rows and has no bin table: any radius of the fp32 mode.
bool gather_fast_ok(const gmi_cache* c) {
    if (c->wsum64 != nullptr || c->force_generic) return false;
    if (c->C > 4) return true;
    int rc, ncol, dyb, nyb;
    gather_geometry(c->cutoff, rc, ncol, dyb, nyb);
    return ncol < kColMax && ncol * nyb + 1 <= kBinMax;
}

// Returns false when the configuration needs the generic gather
// (f64 weight mode, or a radius whose bin table exceeds the staging tables).
bool launch_gather_fast(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts) {
    if (!gather_fast_ok(c)) return false;
    // C > 4: the wide-channel gather (gmi_wide.cu) on index-ordered cells
    if (launch_gather_wide(ctx, c, image, counts)) return true;
    if (c->C > 4) return false;
    const double r = c->cutoff;
    GatherParams p{};
    gather_geometry(r, p.rc, p.ncol, p.dyb, p.nyb);
    for (int l = 0; l < 32; ++l) {
        p.qlo[l] = static_cast<uint8_t>(std::max(0, static_cast<int>(std::floor(2.0 * l + p.rc - r))));
        p.qhi[l] = static_cast<uint8_t>(std::min(p.ncol - 1,
                                                 static_cast<int>(std::ceil(2.0 * l + p.rc + 1 + r)) - 1));
    }
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.rec = c->rec;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.r64 = r;
    p.r2_64 = r * r;
    p.r2f = static_cast<float>(p.r2_64);
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    // in-ball test on e = nk d^2: e >= nk r^2 (fp32 rounding of both sides is
    // ~3 ulp, far inside the 8e-6 r^2 safety band of unflagged points)
    p.thr = p.r2f * p.nk;
    p.image = image;
    p.wsum = c->wsum;
    p.counts = counts;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    const dim3 grid((c->W + kTW - 1) / kTW, (c->H + kTH - 1) / kTH, c->B);
    GMI_CUDA(cudaMemsetAsync(c->special_count_d, 0, sizeof(int32_t), ctx->stream));
    if (c->C <= 3) {
        // f64 folds of multi-chunk (clustered) tiles: up to 1024 per call
        // (128 KB each), slots handed out on the device
        p.fold_cap = 1024;
        char* f = static_cast<char*>(scratch(ctx, WS_FOLD, 256 + sizeof(double) * kFoldVals * kNT * p.fold_cap));
        p.fold_count = reinterpret_cast<int32_t*>(f);
        p.fold = reinterpret_cast<double*>(f + 256);
        GMI_CUDA(cudaMemsetAsync(p.fold_count, 0, sizeof(int32_t), ctx->stream));
    }
    const bool cnt = counts != nullptr;
    switch (c->C) {
        case 1: cnt ? launch_cc<1, true>(ctx, p, grid) : launch_cc<1, false>(ctx, p, grid); break;
        case 2: cnt ? launch_cc<2, true>(ctx, p, grid) : launch_cc<2, false>(ctx, p, grid); break;
        case 3: cnt ? launch_cc<3, true>(ctx, p, grid) : launch_cc<3, false>(ctx, p, grid); break;
        default: cnt ? launch_cc<4, true>(ctx, p, grid) : launch_cc<4, false>(ctx, p, grid); break;
    }
    return true;
}

}  // namespace gmi_host
