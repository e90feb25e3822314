// Wide-channel hot path (C > 4, fp32 weight mode): K2 forward gather and K4
// backward that compute each Gaussian weight once for 16 or more channels
// instead of once per group of 4 (configs[4]: C = 64, sigma = 4).
//
// K1 for this path keeps each cell in ascending original index (the
// reference's bin order, bin_grid.cpp:76-80) and writes the 32-byte records
// plus all colours [B][N][C] in that order, so both kernels visit candidates
// in a fixed order and the result is bit-deterministic without any in-CTA
// canonicalisation.
//
// K2 wide (engine.cpp:44-103, query_radius bin_grid.cpp:84-105):
//   CTA = 16x16 output pixels, 8 warps; warp = an 8x4 pixel block; lane =
//   one 2x2 pixel quad (lane & 7) x one block of CB channels (lane >> 3), so
//   4 * CB channels per pass (64 for CB = 16).  The tile's candidates (cells
//   overlapping the tile grown by r, runs per cell row) are staged in chunks
//   of 256: position + flag record and the pass's colours.  Each warp tests
//   32 candidates at a time against its block (one lane per candidate, a
//   ballot) and walks the hits: per hit, per lane, 7 f32x2 ops for the four
//   e = nk d^2, the exact in-ball test (fp32 for unflagged points, the f64
//   predicate for K1-flagged ones), 4 MUFU.EX2 and 2 CB f32x2 FMAs.  The
//   weight is the forward's e-form (bit-identical to the C <= 4 gather and
//   to the backward below).  Normalisation (one Newton step) and the store
//   are fused; W goes to the cache, W == 0 pixels to the fallback list (K3).
//
// K4 wide (engine.cpp:190-234): point-major and atomic-free like the C <= 4
//   backward.  CTA = a block of reference cells x a group of 16 channels; the
//   pixel region its points reach is staged once as u_c = up_c / W (16
//   floats, 64 B per pixel) and v = sum_c u_c out_c.  A warp owns one point
//   at a time: its 4 teams of 8 lanes take interleaved disk rows, a team
//   steps through a row two pixels at a time (lanes 0-3 the even pixel,
//   4-7 the odd one, 4 channels per lane: every LDS.128 phase reads 128
//   contiguous bytes, conflict-free).  Per pixel and lane:
//       R_c  += w u_c,   Gx_c += (w dx) u_c,   vx += (w dx) v,  vr += w v
//   and per row  d_col_c += R_c,  Gy_c += dy R_c,  vy += dy vr,  so that
//       d_pos = (sum_c c_ic G_c - (vx, vy)) / sigma^2
//   (= sum_p ratio * dot * (q - mu) / sigma^2, engine.cpp:219-230).  Group
//   partials of d_pos are summed in group order (deterministic).
#include <algorithm>
#include <cmath>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// ---------------------------------------------------------------------------
// K2 wide
// ---------------------------------------------------------------------------
constexpr int kWT = 16;          // tile side (pixels)
constexpr int kWThreads = 256;   // 8 warps
constexpr int kWCap = 384;       // staged candidates per chunk (tile-filtered)
constexpr int kWRuns = 32;       // cell rows per run group

template <int CB>
struct SmemWide {
    float4 pt[kWCap];            // x, y, idx|flag bits, 0
    float4 col[kWCap][CB];       // the pass's 4 CB channels
    int slot[kWCap];
    int run_beg[kWRuns + 1];
    int run_g[kWRuns];
    int rect[4];                 // cx0, cx1, cy0, cy1
    int wcnt[kWThreads / 32];    // kept candidates per warp (chunk fill)
    int e_resume;
};

struct GatherWideParams {
    const Geom* geom;
    const int32_t* bins;
    const float4* rec;   // [B][N][2] (x, y, c0, c1) (c2, c3, idx|flag, 0)
    const float* ccol;   // [B][N][C] colours in bin order
    int N, C, W, H;
    int nsg;             // channel passes of 4 CB channels
    int tiles_x, tiles_y;
    int heavy_cap;       // CTA slots reserved for heavy tiles (launched first)
    const int32_t* heavy_list;   // heavy tiles (linear b * ty * tx index)
    const int32_t* heavy_count;
    const uint8_t* heavy_mark;   // per tile: 1 = processed from the heavy list
    // f64 fold of the fp32 accumulators at every chunk end, for the first
    // fold_cap heavy tiles: [heavy slot][pass][4 + 4 CB][thread]
    double* fold;
    int fold_cap;
    double r64, r2_64;
    float rhit2;         // (r + 1e-3)^2: conservative block test
    float nk, thr;
    float* image;
    float* wsum;
    int32_t* counts;
    Special* special;
    int32_t* special_count;
    int special_cap;
};

template <int CB, bool kCount>
__global__ void __launch_bounds__(kWThreads, 2)
k_gather_wide(GatherWideParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemWide<CB>& S = *reinterpret_cast<SmemWide<CB>*>(smem_raw);
    constexpr int kJ = CB / 4;  // float4 of colours per lane per candidate

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cb = lane >> 3, q = lane & 7;
    // CTA -> tile: the first heavy_cap slots take the heavy (clustered)
    // tiles so that they start first; the rest walk the tiles in order and
    // skip the heavy ones
    const int sg = blockIdx.y;
    int tile;
    {
        const int slot = blockIdx.x;
        if (slot < p.heavy_cap) {
            if (slot >= min(*p.heavy_count, p.heavy_cap)) return;
            tile = p.heavy_list[slot];
        } else {
            tile = slot - p.heavy_cap;
            if (p.heavy_mark[tile]) return;
        }
    }
    const int ntx = p.tiles_x, nty = p.tiles_y;
    const int b = tile / (ntx * nty);
    const int tyx = tile - b * ntx * nty;
    const int sgc0 = sg * 4 * CB;
    const int ch0 = sgc0 + cb * CB;
    const int nch = max(0, min(CB, p.C - ch0));
    const int x0 = (tyx % ntx) * kWT, y0 = (tyx / ntx) * kWT;
    const int bx0 = x0 + 8 * (warp & 1), by0 = y0 + 4 * (warp >> 1);
    const int xa = bx0 + 2 * (q & 3), ya = by0 + 2 * (q >> 2);
    const Geom g = p.geom[b];
    const size_t base = static_cast<size_t>(b) * p.N;

    const float2 X = f2(static_cast<float>(xa), static_cast<float>(xa + 1));
    const float2 Y = f2(static_cast<float>(ya), static_cast<float>(ya + 1));
    const float2 nk2 = f2(p.nk, p.nk);
    const float thr = p.thr;
    // the warp's 8x4 block: centre and half extents (conservative hit test)
    const float wcx = static_cast<float>(bx0) + 3.5f, wcy = static_cast<float>(by0) + 1.5f;
    float2 Wa = f2(0.f, 0.f), Wb = f2(0.f, 0.f);
    float2 Na[CB], Nb[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) {
        Na[c] = f2(0.f, 0.f);
        Nb[c] = f2(0.f, 0.f);
    }
    int cnt00 = 0, cnt01 = 0, cnt10 = 0, cnt11 = 0;
    // Heavy (clustered) tiles sum tens of thousands of candidates per pixel:
    // a plain fp32 running sum drifts by ~sqrt(n/3) ulp (configs[4]'s
    // cluster: > 1e-5 relative).  Their lanes fold the fp32 accumulators of
    // every chunk (<= kWCap candidates) into private f64 totals, in chunk
    // order (deterministic), and normalise in f64.
    double* const fold = (p.fold != nullptr && blockIdx.x < p.fold_cap &&
                          static_cast<int>(blockIdx.x) < p.heavy_cap)
                             ? p.fold + (static_cast<size_t>(blockIdx.x) * gridDim.y + sg) *
                                            (4 + 4 * CB) * kWThreads + tid
                             : nullptr;
    bool folded = false;
    auto fold_acc = [&](float& a, int k) {
        double* f = fold + static_cast<size_t>(k) * kWThreads;
        *f = (folded ? *f : 0.0) + static_cast<double>(a);
        a = 0.f;
    };

    // the tile's reference cell rectangle (bin_grid.cpp:88-91 for the tile)
    if (tid < 4) {
        const bool ax = tid < 2;
        const double lo = static_cast<double>(ax ? x0 : y0) - p.r64;
        const double hi = static_cast<double>((ax ? x0 : y0) + kWT - 1) + p.r64;
        S.rect[tid] = cell_of((tid & 1) ? hi : lo, ax ? g.ox : g.oy, g.cell,
                              ax ? g.n_cols : g.n_rows);
    }
    __syncthreads();
    const int cx0 = S.rect[0], cx1 = S.rect[1], cy0 = S.rect[2], cy1 = S.rect[3];
    const bool vec = (p.C % 4) == 0 && (reinterpret_cast<uintptr_t>(p.ccol) & 15) == 0;

    for (int cya = cy0; cya <= cy1; cya += kWRuns) {
        const int nr = min(kWRuns, cy1 - cya + 1);
        __syncthreads();  // previous group's run table fully read
        if (warp == 0) {
            int gs = 0, len = 0;
            if (lane < nr) {
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cya + lane) * g.n_cols;
                gs = p.bins[r0 + cx0];
                len = p.bins[r0 + cx1 + 1] - gs;
            }
            int incl = len;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane < nr) {
                S.run_beg[lane] = incl - len;
                S.run_g[lane] = gs;
            }
            if (lane == nr - 1) S.run_beg[nr] = incl;
        }
        __syncthreads();
        const int total = S.run_beg[nr];
        // chunks: the candidates whose disk can reach the tile (conservative
        // fp32 test), compacted in run order, up to kWCap per chunk
        const float tcx = static_cast<float>(x0) + 7.5f, tcy = static_cast<float>(y0) + 7.5f;
        for (int e0 = 0; e0 < total;) {
            int n = 0;
            while (e0 < total && n < kWCap) {
                const int e = e0 + tid;
                bool keep = false;
                int slot = 0;
                float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
                if (e < total) {
                    int lo = 0, hi = nr;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (S.run_beg[mid] <= e) lo = mid;
                        else hi = mid;
                    }
                    slot = S.run_g[lo] + (e - S.run_beg[lo]);
                    const float4 ra = p.rec[(base + slot) * 2];
                    const float rz = p.rec[(base + slot) * 2 + 1].z;
                    pt = make_float4(ra.x, ra.y, rz, 0.f);
                    const float ddx = fmaxf(fabsf(ra.x - tcx) - 7.5f, 0.f);
                    const float ddy = fmaxf(fabsf(ra.y - tcy) - 7.5f, 0.f);
                    keep = fmaf(ddx, ddx, ddy * ddy) <= p.rhit2;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (lane == 0) S.wcnt[warp] = __popc(bal);
                __syncthreads();
                int woff = 0, blk = 0;
#pragma unroll
                for (int w = 0; w < kWThreads / 32; ++w) {
                    const int c = S.wcnt[w];
                    woff += w < warp ? c : 0;
                    blk += c;
                }
                const int pos = n + woff + __popc(bal & ((1u << lane) - 1u));
                GMI_CHECK(!keep || pos >= 0);
                if (keep && pos < kWCap) {
                    S.pt[pos] = pt;
                    S.slot[pos] = slot;
                }
                if (n + blk > kWCap) {
                    // full: the next chunk resumes at the first kept candidate left out
                    if (keep && pos == kWCap) S.e_resume = e;
                    __syncthreads();
                    e0 = S.e_resume;
                    n = kWCap;
                } else {
                    n += blk;
                    e0 += kWThreads;
                    __syncthreads();  // S.wcnt reused by the next block
                }
            }
            if (n == 0) break;
            // ---- stage this pass's colours ----
            for (int e = tid; e < n * CB; e += kWThreads) {
                const int k = e / CB, j = e % CB;
                const int c = sgc0 + 4 * j;
                const float* src = p.ccol + (base + S.slot[k]) * p.C + c;
                float4 v;
                if (vec && c + 3 < p.C) {
                    v = *reinterpret_cast<const float4*>(src);
                } else {
                    v.x = c < p.C ? src[0] : 0.f;
                    v.y = c + 1 < p.C ? src[1] : 0.f;
                    v.z = c + 2 < p.C ? src[2] : 0.f;
                    v.w = c + 3 < p.C ? src[3] : 0.f;
                }
                S.col[k][j] = v;
            }
            __syncthreads();
            // ---- gather: ballot the block's hits, 32 candidates at a time ----
            for (int kb = 0; kb < n; kb += 32) {
                bool hit = false;
                if (kb + lane < n) {
                    const float4 t = S.pt[kb + lane];
                    const float ddx = fmaxf(fabsf(t.x - wcx) - 3.5f, 0.f);
                    const float ddy = fmaxf(fabsf(t.y - wcy) - 1.5f, 0.f);
                    hit = fmaf(ddx, ddx, ddy * ddy) <= p.rhit2;
                }
                unsigned m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int k = kb + __ffs(m) - 1;
                    GMI_CHECK(k >= 0 && k < n && n <= kWCap);
                    m &= m - 1;
                    const float4 t = S.pt[k];
                    const float2 dx = __fadd2_rn(X, f2(-t.x, -t.x));
                    const float2 dy = __fadd2_rn(Y, f2(-t.y, -t.y));
                    const float2 kx = __fmul2_rn(dx, nk2);
                    const float2 ey = __fmul2_rn(__fmul2_rn(dy, nk2), dy);
                    const float2 ea = __ffma2_rn(kx, dx, f2(ey.x, ey.x));
                    const float2 eb = __ffma2_rn(kx, dx, f2(ey.y, ey.y));
                    bool i00, i01, i10, i11;
                    if (__float_as_uint(t.z) & kUnsafeBit) {
                        // boundary-ambiguous point: the reference's f64 predicate
                        const double mx = t.x, my = t.y;
                        i00 = d2_ref(xa, ya, mx, my) <= p.r2_64;
                        i01 = d2_ref(xa + 1, ya, mx, my) <= p.r2_64;
                        i10 = d2_ref(xa, ya + 1, mx, my) <= p.r2_64;
                        i11 = d2_ref(xa + 1, ya + 1, mx, my) <= p.r2_64;
                    } else {
                        i00 = ea.x >= thr;
                        i01 = ea.y >= thr;
                        i10 = eb.x >= thr;
                        i11 = eb.y >= thr;
                    }
                    // branch-free: ex2(-inf) = +0 for pairs outside the ball
                    const float2 wa = f2(ex2(i00 ? ea.x : -INFINITY), ex2(i01 ? ea.y : -INFINITY));
                    const float2 wb = f2(ex2(i10 ? eb.x : -INFINITY), ex2(i11 ? eb.y : -INFINITY));
                    Wa = __fadd2_rn(Wa, wa);
                    Wb = __fadd2_rn(Wb, wb);
                    const float4* cp = &S.col[k][cb * kJ];
#pragma unroll
                    for (int jj = 0; jj < kJ; ++jj) {
                        const float4 c4 = cp[jj];
                        Na[4 * jj + 0] = __ffma2_rn(wa, f2(c4.x, c4.x), Na[4 * jj + 0]);
                        Nb[4 * jj + 0] = __ffma2_rn(wb, f2(c4.x, c4.x), Nb[4 * jj + 0]);
                        Na[4 * jj + 1] = __ffma2_rn(wa, f2(c4.y, c4.y), Na[4 * jj + 1]);
                        Nb[4 * jj + 1] = __ffma2_rn(wb, f2(c4.y, c4.y), Nb[4 * jj + 1]);
                        Na[4 * jj + 2] = __ffma2_rn(wa, f2(c4.z, c4.z), Na[4 * jj + 2]);
                        Nb[4 * jj + 2] = __ffma2_rn(wb, f2(c4.z, c4.z), Nb[4 * jj + 2]);
                        Na[4 * jj + 3] = __ffma2_rn(wa, f2(c4.w, c4.w), Na[4 * jj + 3]);
                        Nb[4 * jj + 3] = __ffma2_rn(wb, f2(c4.w, c4.w), Nb[4 * jj + 3]);
                    }
                    if (kCount) {
                        cnt00 += i00;
                        cnt01 += i01;
                        cnt10 += i10;
                        cnt11 += i11;
                    }
                }
            }
            if (fold != nullptr) {
                fold_acc(Wa.x, 0);
                fold_acc(Wa.y, 1);
                fold_acc(Wb.x, 2);
                fold_acc(Wb.y, 3);
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    fold_acc(Na[c].x, 4 + 4 * c);
                    fold_acc(Na[c].y, 5 + 4 * c);
                    fold_acc(Nb[c].x, 6 + 4 * c);
                    fold_acc(Nb[c].y, 7 + 4 * c);
                }
                folded = true;
            }
            __syncthreads();  // chunk consumed before the next staging
        }
    }

    // ---- fused normalisation + store (engine.cpp:74-100) ----
    const bool owner = sg == 0 && cb == 0;
    const bool vst = (p.C % 4) == 0 && nch == CB &&
                     (reinterpret_cast<uintptr_t>(p.image) & 15) == 0;
#pragma unroll
    for (int py = 0; py < 2; ++py) {
#pragma unroll
        for (int px = 0; px < 2; ++px) {
            const int qx = xa + px, qy = ya + py;
            if (qx >= p.W || qy >= p.H) continue;
            float w = py ? (px ? Wb.y : Wb.x) : (px ? Wa.y : Wa.x);
            const size_t bp = (static_cast<size_t>(b) * p.H + qy) * p.W + qx;
            const int pk = 2 * py + px;
            double w64 = 0.0;
            if (fold != nullptr && folded) {
                w64 = fold[static_cast<size_t>(pk) * kWThreads];
                w = static_cast<float>(w64);
            }
            if (w > 0.f) {
                const float inv = 1.0f / w;
                float o[CB];
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    if (fold != nullptr && folded) {
                        o[c] = static_cast<float>(
                            fold[static_cast<size_t>(4 + 4 * c + pk) * kWThreads] / w64);
                        continue;
                    }
                    const float num = py ? (px ? Nb[c].y : Nb[c].x) : (px ? Na[c].y : Na[c].x);
                    const float q0 = num * inv;
                    o[c] = fmaf(fmaf(-q0, w, num), inv, q0);
                }
                float* out = p.image + bp * p.C + ch0;
                if (vst) {
#pragma unroll
                    for (int jj = 0; jj < kJ; ++jj)
                        reinterpret_cast<float4*>(out)[jj] =
                            make_float4(o[4 * jj], o[4 * jj + 1], o[4 * jj + 2], o[4 * jj + 3]);
                } else {
#pragma unroll
                    for (int c = 0; c < CB; ++c)
                        if (c < nch) out[c] = o[c];
                }
                if (owner) {
                    p.wsum[bp] = w;
                    if (kCount) p.counts[bp] = py ? (px ? cnt11 : cnt10) : (px ? cnt01 : cnt00);
                }
            } else if (owner) {
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

// Per tile: the number of candidates (cells overlapping the tile grown by r);
// tiles above kHeavy go to the heavy list (processed by the first CTAs).
constexpr int kHeavy = 8 * kWCap;

__global__ void k_wide_tile_load(const Geom* __restrict__ geom, const int32_t* __restrict__ bins,
                                 int tiles_x, int tiles_y, int B, double r64, int cap,
                                 int32_t* __restrict__ heavy_list, int32_t* heavy_count,
                                 uint8_t* __restrict__ mark) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B * tiles_x * tiles_y) return;
    const int b = t / (tiles_x * tiles_y), tyx = t - b * tiles_x * tiles_y;
    const int x0 = (tyx % tiles_x) * kWT, y0 = (tyx / tiles_x) * kWT;
    const Geom g = geom[b];
    const int cx0 = cell_of(static_cast<double>(x0) - r64, g.ox, g.cell, g.n_cols);
    const int cx1 = cell_of(static_cast<double>(x0 + kWT - 1) + r64, g.ox, g.cell, g.n_cols);
    const int cy0 = cell_of(static_cast<double>(y0) - r64, g.oy, g.cell, g.n_rows);
    const int cy1 = cell_of(static_cast<double>(y0 + kWT - 1) + r64, g.oy, g.cell, g.n_rows);
    long tot = 0;
    for (int cy = cy0; cy <= cy1 && tot <= kHeavy; ++cy) {
        const int64_t r0 = g.bin_off + static_cast<int64_t>(cy) * g.n_cols;
        tot += bins[r0 + cx1 + 1] - bins[r0 + cx0];
    }
    uint8_t m = 0;
    if (tot > kHeavy) {
        const int slot = atomicAdd(heavy_count, 1);
        if (slot < cap) {
            heavy_list[slot] = t;
            m = 1;
        }
    }
    mark[t] = m;
}

template <int CB, bool kCount>
void launch_wide_cb(gmi_ctx* ctx, const GatherWideParams& p, dim3 grid) {
    const int smem = static_cast<int>(sizeof(SmemWide<CB>));
    GMI_SMEM_ONCE(ctx, (k_gather_wide<CB, kCount>), smem);
    k_gather_wide<CB, kCount><<<grid, kWThreads, smem, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

// ---------------------------------------------------------------------------
// K4 wide
// ---------------------------------------------------------------------------
constexpr int kBG = 16;                 // channels per group
constexpr int kBThreads = 256;          // 8 warps (one point each) x 4 squads
constexpr int kPlanePx = 1600;          // ring capacity in pixels (68 B each): 2 CTAs/SM
constexpr int kBSmem = kPlanePx * 68;
constexpr int kBSeg = 16;               // cell rows per CTA

struct BwdWideParams {
    const Geom* geom;
    const int32_t* bins;
    const int32_t* blk_off;  // [B+1] CTA offsets per image
    const float4* rec;
    const float* ccol;       // [B][N][C]
    const float* wsum;       // [B][H][W]
    const float* image;      // [B][H][W][C]
    const float* upstream;   // [B][H][W][C]
    int B, N, C, W, H;
    int seg;                 // cell rows per CTA (one cell column)
    int nseg_cap;            // row segments per column (unit = column * nseg_cap + segment)
    int heavy_cap;           // CTA slots reserved for heavy units (launched first)
    const int32_t* heavy_list;
    const int32_t* heavy_count;
    const uint8_t* heavy_mark;
    double r64, r2_64;
    float nk, inv_s2;
    float* d_col;            // [B][N][C]
    float* d_pos;            // partial [groups][B][N][2]
};

__device__ __forceinline__ bool in_ref_w(int x, int y, float mx, float my, double r2_64) {
    return d2_ref(static_cast<double>(x), static_cast<double>(y), static_cast<double>(mx),
                  static_cast<double>(my)) <= r2_64;
}

// The 16 channels of group ch0 at one pixel: w (W of the pixel), up and out.
__device__ __forceinline__ void load_px16(const BwdWideParams& p, size_t pix, int ch0, bool full,
                                          float& w, float* up, float* im) {
    w = p.wsum[pix];
    if (full) {
        const float4* u4 = reinterpret_cast<const float4*>(p.upstream + pix * p.C + ch0);
        const float4* o4 = reinterpret_cast<const float4*>(p.image + pix * p.C + ch0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4 a = u4[j], o = o4[j];
            up[4 * j] = a.x; up[4 * j + 1] = a.y; up[4 * j + 2] = a.z; up[4 * j + 3] = a.w;
            im[4 * j] = o.x; im[4 * j + 1] = o.y; im[4 * j + 2] = o.z; im[4 * j + 3] = o.w;
        }
    } else {
#pragma unroll
        for (int c = 0; c < kBG; ++c) {
            up[c] = ch0 + c < p.C ? p.upstream[pix * p.C + ch0 + c] : 0.f;
            im[c] = ch0 + c < p.C ? p.image[pix * p.C + ch0 + c] : 0.f;
        }
    }
}

// sum_c u_c x_c over the group's 16 channels as four chains (c mod 4) in
// f32x2, combined in a fixed order.  The backward forms both v = sum u out
// and sum u c_i with it, so t = sum u c_i - v is exactly 0 where a pixel's
// output equals the point's colour (a sole contributor).
__device__ __forceinline__ float chain16(const float2* uu, const float2* xx) {
    float2 ta = make_float2(0.f, 0.f), tb = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < kBG / 2; k += 2) {
        ta = __ffma2_rn(uu[k], xx[k], ta);
        tb = __ffma2_rn(uu[k + 1], xx[k + 1], tb);
    }
    return (ta.x + ta.y) + (tb.x + tb.y);
}

// u_c = up_c / W and v = sum_c u_c out_c (zeros for W == 0: fallback pixel)
__device__ __forceinline__ float pixel_uv(float w, float* u, const float* im) {
    const float inv = w > 0.f ? 1.0f / w : 0.f;
    float2 uu[kBG / 2], oo[kBG / 2];
#pragma unroll
    for (int k = 0; k < kBG / 2; ++k) {
        u[2 * k] *= inv;
        u[2 * k + 1] *= inv;
        uu[k] = make_float2(u[2 * k], u[2 * k + 1]);
        oo[k] = make_float2(im[2 * k], im[2 * k + 1]);
    }
    return chain16(uu, oo);
}

// Column walk: CTA = (image, cell column, segment of kBSeg cell rows, group).
// The pixel rows a cell's points reach (the cell grown by r) live in a ring
// of rows in shared memory: 4 planes of float4 (u, 16 channels) + 1 plane of
// v, pixel-major inside a plane, so 8 lanes on 8 consecutive pixels read 128
// contiguous bytes per LDS.128 (conflict-free).  Consecutive cells of the
// column share all but cell rows, which are the only ones staged.
// A warp owns one point; its 4 squads of 8 lanes take interleaved rows of the
// point's exact disk, lane l of a squad the pixels xl + l, xl + l + 8, ..;
// per pixel
//     t = sum_c u_c c_ic - v,  d_col_c += w u_c,  d_pos += w t (q - mu)
// with all 16 channels of the group in the lane's registers (no cross-lane
// work per pixel).  Lane sums are combined by a fixed shuffle tree.
__global__ void __launch_bounds__(kBThreads, 2)
k_backward_wide(BwdWideParams p) {
    extern __shared__ float4 s_u4[];      // planes [4][kPlanePx] float4, then s_v[kPlanePx]
    float* s_v = reinterpret_cast<float*>(s_u4 + 4 * kPlanePx);
    __shared__ float s_red[4][kBThreads / 32];
    __shared__ int s_reg[5];

    // ---- image, cell column and row segment of this CTA: the first
    // heavy_cap slots take the heavy (clustered) units so they start first ----
    int unit;
    if (static_cast<int>(blockIdx.x) < p.heavy_cap) {
        if (static_cast<int>(blockIdx.x) >= min(*p.heavy_count, p.heavy_cap)) return;
        unit = p.heavy_list[blockIdx.x];
    } else {
        unit = blockIdx.x - p.heavy_cap;
        if (p.heavy_mark[unit]) return;
    }
    int b = 0;
    {
        int lo = 0, hi = p.B;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (p.blk_off[mid] <= unit) lo = mid;
            else hi = mid;
        }
        b = lo;
    }
    const Geom g = p.geom[b];
    const int local = unit - p.blk_off[b];
    const int cx = local / p.nseg_cap, sgm = local % p.nseg_cap;
    const int cyA = sgm * p.seg;
    if (cx >= g.n_cols || cyA >= g.n_rows) return;  // past this image's grid
    const int cyB = min(cyA + p.seg, g.n_rows);
    const int cg = blockIdx.y, ch0 = cg * kBG;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sq = lane >> 3, sl = lane & 7;
    const size_t base = static_cast<size_t>(b) * p.N;
    const size_t img_base = static_cast<size_t>(b) * p.H * p.W;
    const float nk = p.nk;
    const float r2f = static_cast<float>(p.r2_64), rf = static_cast<float>(p.r64);
    const double r2_64 = p.r2_64;
    // a point's in-ball pixels lie within its cell grown by r
    const double pad = p.r64 + 0.25;
    const bool full = (p.C % 4) == 0 && ch0 + kBG <= p.C &&
                      (reinterpret_cast<uintptr_t>(p.upstream) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(p.image) & 15) == 0;
    const bool cfull = (p.C % 4) == 0 && ch0 + kBG <= p.C &&
                       (reinterpret_cast<uintptr_t>(p.ccol) & 15) == 0;

    // uncapped grids bound a cell's points by the cell: the column's x-range
    // is fixed and consecutive cells share rows
    int rx0 = 0, rx1 = -1, wd = 0, rb = 0;
    if (!g.capped) {
        rx0 = max(0, static_cast<int>(floor(g.ox + cx * g.cell - pad)));
        rx1 = min(p.W - 1, static_cast<int>(ceil(g.ox + (cx + 1) * g.cell + pad)));
        wd = rx1 - rx0 + 1;
        rb = wd > 0 ? kPlanePx / wd : 0;
    }
    int st_hi = -1;  // last staged row: the ring holds rows (st_hi - rb, st_hi]

    for (int cy = cyA; cy < cyB; ++cy) {
        const int64_t ci = g.bin_off + static_cast<int64_t>(cy) * g.n_cols + cx;
        const int s0 = p.bins[ci], cnt = p.bins[ci + 1] - s0;
        if (cnt == 0) continue;
        int ry0, ry1, mode;  // mode 1: staged, 0: from global, -1: no pixel reachable
        if (!g.capped) {
            ry0 = max(0, static_cast<int>(floor(g.oy + cy * g.cell - pad)));
            ry1 = min(p.H - 1, static_cast<int>(ceil(g.oy + (cy + 1) * g.cell + pad)));
            mode = (wd <= 0 || ry1 < ry0) ? -1 : (ry1 - ry0 + 1 <= rb ? 1 : 0);
        } else {
            // clamped edge cells: the bbox of the cell's points grown by r
            float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
            for (int k = tid; k < cnt; k += kBThreads) {
                const float4 ra = p.rec[(base + s0 + k) * 2];
                mnx = fminf(mnx, ra.x);
                mny = fminf(mny, ra.y);
                mxx = fmaxf(mxx, ra.x);
                mxy = fmaxf(mxy, ra.y);
            }
            for (int o = 16; o > 0; o >>= 1) {
                mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
                mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
                mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
                mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
            }
            __syncthreads();  // s_red / s_reg and the ring free
            if (lane == 0) {
                s_red[0][warp] = mnx;
                s_red[1][warp] = mny;
                s_red[2][warp] = mxx;
                s_red[3][warp] = mxy;
            }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < kBThreads / 32; ++w) {
                    mnx = fminf(mnx, s_red[0][w]);
                    mny = fminf(mny, s_red[1][w]);
                    mxx = fmaxf(mxx, s_red[2][w]);
                    mxy = fmaxf(mxy, s_red[3][w]);
                }
                const float rr = static_cast<float>(p.r64) + 1.0f;
                const int x0 = max(0, static_cast<int>(floorf(fmaxf(mnx - rr, -1.0e9f))));
                const int y0 = max(0, static_cast<int>(floorf(fmaxf(mny - rr, -1.0e9f))));
                const int x1 = min(p.W - 1, static_cast<int>(ceilf(fminf(mxx + rr, 1.0e9f))));
                const int y1 = min(p.H - 1, static_cast<int>(ceilf(fminf(mxy + rr, 1.0e9f))));
                s_reg[0] = x0;
                s_reg[1] = x1;
                s_reg[2] = y0;
                s_reg[3] = y1;
                s_reg[4] = (mnx <= mxx && x1 >= x0 && y1 >= y0) ? 1 : -1;
            }
            __syncthreads();
            rx0 = s_reg[0];
            rx1 = s_reg[1];
            ry0 = s_reg[2];
            ry1 = s_reg[3];
            wd = rx1 - rx0 + 1;
            rb = wd > 0 ? kPlanePx / wd : 0;
            st_hi = -1;  // new x-range: nothing reusable
            mode = s_reg[4] < 0 ? -1 : (ry1 - ry0 + 1 <= rb ? 1 : 0);
        }
        if (mode < 0) {
            // no frame pixel is reachable: gradients are zero
            for (int k = tid; k < cnt; k += kBThreads) {
                const int i = static_cast<int>(
                    __float_as_uint(p.rec[(base + s0 + k) * 2 + 1].z) & 0x7fffffffu);
                for (int c = ch0; c < min(p.C, ch0 + kBG); ++c) p.d_col[(base + i) * p.C + c] = 0.f;
                float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
                dp[0] = 0.f;
                dp[1] = 0.f;
            }
            continue;
        }
        if (mode == 1 && ry1 > st_hi) {
            // ---- stage the rows this cell adds (lane per pixel) ----
            const int ys = max(st_hi + 1, ry0);
            const int area = (ry1 - ys + 1) * wd;
            __syncthreads();  // the previous cell's points are done with the ring
            int r = tid / wd, cc = tid - r * wd;
            int pr = (ys + r) % rb;
            for (int k = tid; k < area; k += kBThreads) {
                const int yy = ys + r, xx = rx0 + cc;
                float w = 0.f, u[kBG], im[kBG];
#pragma unroll
                for (int c = 0; c < kBG; ++c) {
                    u[c] = 0.f;
                    im[c] = 0.f;
                }
                if (xx < p.W && yy < p.H)
                    load_px16(p, img_base + static_cast<size_t>(yy) * p.W + xx, ch0, full, w, u, im);
                const float v = pixel_uv(w, u, im);
                const int q = pr * wd + cc;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    s_u4[j * kPlanePx + q] = make_float4(u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
                s_v[q] = v;
                cc += kBThreads;
                while (cc >= wd) {
                    cc -= wd;
                    ++r;
                    if (++pr == rb) pr = 0;
                }
            }
            st_hi = ry1;
            __syncthreads();
        }
        const bool staged = mode == 1;
        const int xmin = max(rx0, 0), xmax = min(rx1, p.W - 1);

        // ---- per point: one warp, its 4 squads on interleaved rows ----
        for (int k = warp; k < cnt; k += kBThreads / 32) {
            const int s = s0 + k;
            if (k + kBThreads / 32 < cnt && lane < 3) {
                // the warp's next point: record and colour lines into L1
                const int sn = s + kBThreads / 32;
                const char* a = lane == 0 ? reinterpret_cast<const char*>(p.rec + (base + sn) * 2)
                                          : reinterpret_cast<const char*>(p.ccol + (base + sn) * p.C + ch0) +
                                                (lane - 1) * 32;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
            }
            const float4 ra = p.rec[(base + s) * 2];
            const uint32_t raw = __float_as_uint(p.rec[(base + s) * 2 + 1].z);
            const float mx = ra.x, my = ra.y;
            const int i = static_cast<int>(raw & 0x7fffffffu);
            const bool unsafe = (raw & kUnsafeBit) != 0;
            // channel pairs in f32x2: the 32 FMAs per pixel as 16 FFMA2 (half
            // the issue slots, the same per-channel operations)
            float2 cc2[kBG / 2];
            if (cfull) {
                const float4* c4 = reinterpret_cast<const float4*>(p.ccol + (base + s) * p.C + ch0);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 t = c4[j];
                    cc2[2 * j] = f2(t.x, t.y);
                    cc2[2 * j + 1] = f2(t.z, t.w);
                }
            } else {
#pragma unroll
                for (int k = 0; k < kBG / 2; ++k) {
                    const int c = ch0 + 2 * k;
                    cc2[k] = f2(c < p.C ? p.ccol[(base + s) * p.C + c] : 0.f,
                                c + 1 < p.C ? p.ccol[(base + s) * p.C + c + 1] : 0.f);
                }
            }
            float2 dc2[kBG / 2];
#pragma unroll
            for (int k = 0; k < kBG / 2; ++k) dc2[k] = f2(0.f, 0.f);
            float gx = 0.f, gy = 0.f;
            const float tx = truncf(mx);
            const float fmu = mx - tx;  // exact
            const int bx = static_cast<int>(tx);
            const float pd = unsafe ? 1.0f : 1e-2f;
            const int ya = max(ry0, static_cast<int>(ceilf(my - rf - pd))) + sq;
            const int yb = min(ry1, static_cast<int>(floorf(my + rf + pd)));
            int prow = staged && ya <= yb ? ya % rb : 0;
            float yf = static_cast<float>(ya);
            for (int y = ya; y <= yb; y += 4, yf += 4.f) {
                const int pr = prow;
                if (staged) {
                    prow += 4;
                    while (prow >= rb) prow -= rb;
                }
                float dy;
                int xl, xr;
                if (!unsafe) {
                    dy = yf - my;
                    const float h2f = fmaf(-dy, dy, r2f);
                    if (h2f < 0.f) continue;
                    const float sqv = h2f * rsqrt_ftz(fmaxf(h2f, 1e-30f));
                    constexpr float kMagic = 12582912.0f;
                    constexpr int kMagicBits = 0x4B400000;
                    xl = bx + (__float_as_int(__fadd_ru(fmu - sqv, kMagic)) - kMagicBits);
                    xr = bx + (__float_as_int(__fadd_rd(fmu + sqv, kMagic)) - kMagicBits);
                } else {
                    const double dy64 = __dsub_rn(static_cast<double>(y), static_cast<double>(my));
                    const double h2 = __dsub_rn(r2_64, __dmul_rn(dy64, dy64));
                    if (h2 < 0.0) continue;
                    const float sqv = sqrtf(static_cast<float>(h2));
                    xl = bx + static_cast<int>(ceilf(fmu - sqv));
                    xr = bx + static_cast<int>(floorf(fmu + sqv));
                    int a = xl - 2;
                    while (a <= xl + 2 && !in_ref_w(a, y, mx, my, r2_64)) ++a;
                    int z = xr + 2;
                    while (z >= xr - 2 && !in_ref_w(z, y, mx, my, r2_64)) --z;
                    xl = a;
                    xr = z;
                    dy = static_cast<float>(dy64);
                }
                xl = max(xl, xmin);
                xr = min(xr, xmax);
                // e = nk dx^2 + nk dy^2 with the forward's fp32 operations
                const float ey = (dy * nk) * dy;
                const int x0l = xl + sl;
                float xf = static_cast<float>(x0l);
                if (staged) {
                    const int q0 = pr * wd - rx0;
                    for (int x = x0l; x <= xr; x += 8, xf += 8.f) {
                        const int q = q0 + x;
                        const float4 u0 = s_u4[q], u1 = s_u4[kPlanePx + q];
                        const float4 u2 = s_u4[2 * kPlanePx + q], u3 = s_u4[3 * kPlanePx + q];
                        const float v = s_v[q];
                        const float2 uu[kBG / 2] = {f2(u0.x, u0.y), f2(u0.z, u0.w), f2(u1.x, u1.y),
                                                    f2(u1.z, u1.w), f2(u2.x, u2.y), f2(u2.z, u2.w),
                                                    f2(u3.x, u3.y), f2(u3.z, u3.w)};
                        const float dx = xf - mx;
                        const float w = ex2(fmaf(dx * nk, dx, ey));
                        // t = sum_c c_ic u_c - v  (= dot / W, engine.cpp:219-221):
                        // four partial sums (chains c mod 4) as two f32x2, the
                        // chain of the staged v (chain16)
                        const float t = chain16(uu, cc2) - v;
                        const float a = w * t;
                        gx = fmaf(a, dx, gx);
                        gy = fmaf(a, dy, gy);
                        const float2 w2 = f2(w, w);
#pragma unroll
                        for (int k = 0; k < kBG / 2; ++k) dc2[k] = __ffma2_rn(w2, uu[k], dc2[k]);
                    }
                } else {
                    for (int x = x0l; x <= xr; x += 8, xf += 8.f) {
                        float w0, u[kBG], im[kBG];
                        load_px16(p, img_base + static_cast<size_t>(y) * p.W + x, ch0, full, w0, u, im);
                        const float v = pixel_uv(w0, u, im);
                        const float dx = xf - mx;
                        const float w = ex2(fmaf(dx * nk, dx, ey));
                        float2 uu[kBG / 2];
#pragma unroll
                        for (int k = 0; k < kBG / 2; ++k) uu[k] = f2(u[2 * k], u[2 * k + 1]);
                        const float t = chain16(uu, cc2) - v;
                        const float a = w * t;
                        gx = fmaf(a, dx, gx);
                        gy = fmaf(a, dy, gy);
                        const float2 w2 = f2(w, w);
#pragma unroll
                        for (int k = 0; k < kBG / 2; ++k)
                            dc2[k] = __ffma2_rn(w2, f2(u[2 * k], u[2 * k + 1]), dc2[k]);
                    }
                }
            }
            float dcol[kBG];
#pragma unroll
            for (int k = 0; k < kBG / 2; ++k) {
                dcol[2 * k] = dc2[k].x;
                dcol[2 * k + 1] = dc2[k].y;
            }
            // ---- warp sums: the 4 squads, then a reduce-scatter of d_col
            // inside the squad (lane sl keeps channels 2 sl, 2 sl + 1) ----
#pragma unroll
            for (int o = 8; o < 32; o <<= 1) {
#pragma unroll
                for (int c = 0; c < kBG; ++c) dcol[c] += __shfl_xor_sync(0xffffffffu, dcol[c], o);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const bool up = (sl & 4) != 0;
                const float send = up ? dcol[c] : dcol[c + 8];
                const float keep = up ? dcol[c + 8] : dcol[c];
                dcol[c] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const bool up = (sl & 2) != 0;
                const float send = up ? dcol[c] : dcol[c + 4];
                const float keep = up ? dcol[c + 4] : dcol[c];
                dcol[c] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const bool up = (sl & 1) != 0;
                const float send = up ? dcol[c] : dcol[c + 2];
                const float keep = up ? dcol[c + 2] : dcol[c];
                dcol[c] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                gx += __shfl_xor_sync(0xffffffffu, gx, o);
                gy += __shfl_xor_sync(0xffffffffu, gy, o);
            }
            if (sq == 0) {
                const int c0 = ch0 + 2 * sl;
                float* dc = p.d_col + (base + i) * p.C + c0;
                if (c0 < p.C) dc[0] = dcol[0];
                if (c0 + 1 < p.C) dc[1] = dcol[1];
                if (sl == 0) {
                    float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
                    dp[0] = gx * p.inv_s2;
                    dp[1] = gy * p.inv_s2;
                }
            }
        }
    }
}

// Per backward unit (cell column segment): its number of points; units
// above kHeavyB go to the heavy list (processed by the first CTAs).
constexpr int kHeavyB = 4096;

__global__ void k_wide_unit_load(const Geom* __restrict__ geom, const int32_t* __restrict__ bins,
                                 const int32_t* __restrict__ blk_off, int B, int seg, int nseg_cap,
                                 int cap, int32_t* __restrict__ heavy_list, int32_t* heavy_count,
                                 uint8_t* __restrict__ mark) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= blk_off[B]) return;
    int lo = 0, hi = B;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (blk_off[mid] <= u) lo = mid;
        else hi = mid;
    }
    const Geom g = geom[lo];
    const int local = u - blk_off[lo];
    const int cx = local / nseg_cap, cyA = (local % nseg_cap) * seg;
    uint8_t m = 0;
    if (cx < g.n_cols && cyA < g.n_rows) {
        long tot = 0;
        for (int cy = cyA; cy < min(cyA + seg, g.n_rows); ++cy) {
            const int64_t ci = g.bin_off + static_cast<int64_t>(cy) * g.n_cols + cx;
            tot += bins[ci + 1] - bins[ci];
        }
        if (tot > kHeavyB) {
            const int slot = atomicAdd(heavy_count, 1);
            if (slot < cap) {
                heavy_list[slot] = u;
                m = 1;
            }
        }
    }
    mark[u] = m;
}

// d_pos = sum over channel groups, in group order (deterministic)
__global__ void k_sum_groups_w(const float* __restrict__ part, float* __restrict__ d_pos,
                               size_t n2, int groups) {
    const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (k >= n2) return;
    float s = 0.f;
    for (int gi = 0; gi < groups; ++gi) s += part[gi * n2 + k];
    d_pos[k] = s;
}

}  // namespace

namespace gmi_host {

bool launch_gather_wide(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts) {
    if (c->C <= 4 || c->rec == nullptr || c->ccol == nullptr || c->wsum64 != nullptr) return false;
    GatherWideParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.rec = c->rec;
    p.ccol = c->ccol;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    const double r = c->cutoff;
    p.r64 = r;
    p.r2_64 = r * r;
    const float rh = static_cast<float>(r) + 1e-3f;
    p.rhit2 = rh * rh;
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    // in-ball test on e = nk d^2 (see gmi_gather.cu)
    p.thr = static_cast<float>(p.r2_64) * p.nk;
    p.image = image;
    p.wsum = c->wsum;
    p.counts = counts;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    // channels per lane: the smallest block with 4 CB >= min(C, 64)
    const int cb = c->C <= 16 ? 4 : (c->C <= 32 ? 8 : 16);
    p.nsg = (c->C + 4 * cb - 1) / (4 * cb);
    p.tiles_x = (c->W + kWT - 1) / kWT;
    p.tiles_y = (c->H + kWT - 1) / kWT;
    const int ntiles = c->B * p.tiles_x * p.tiles_y;
    p.heavy_cap = std::min(4096, ntiles);
    // scratch: [heavy count][heavy list][marks]
    char* ws = static_cast<char*>(scratch(ctx, WS_TMP, sizeof(int32_t) * (1 + p.heavy_cap) + ntiles));
    int32_t* d_cnt = reinterpret_cast<int32_t*>(ws);
    p.heavy_count = d_cnt;
    p.heavy_list = d_cnt + 1;
    p.heavy_mark = reinterpret_cast<uint8_t*>(ws + sizeof(int32_t) * (1 + p.heavy_cap));
    GMI_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int32_t), ctx->stream));
    k_wide_tile_load<<<(ntiles + 255) / 256, 256, 0, ctx->stream>>>(
        c->geom_d, c->bins, p.tiles_x, p.tiles_y, c->B, r, p.heavy_cap, d_cnt + 1, d_cnt,
        reinterpret_cast<uint8_t*>(ws + sizeof(int32_t) * (1 + p.heavy_cap)));
    GMI_LAUNCHED(ctx);
    const dim3 grid(p.heavy_cap + ntiles, p.nsg);
    // f64 folds for up to 512 heavy tiles per call (~140 KB each at C = 64)
    p.fold_cap = std::min(p.heavy_cap, 512);
    p.fold = static_cast<double*>(scratch(ctx, WS_FOLD, sizeof(double) * p.fold_cap * p.nsg *
                                                            (4 + 4 * cb) * kWThreads));
    GMI_CUDA(cudaMemsetAsync(c->special_count_d, 0, sizeof(int32_t), ctx->stream));
    const bool cnt = counts != nullptr;
    switch (cb) {
        case 4: cnt ? launch_wide_cb<4, true>(ctx, p, grid) : launch_wide_cb<4, false>(ctx, p, grid); break;
        case 8: cnt ? launch_wide_cb<8, true>(ctx, p, grid) : launch_wide_cb<8, false>(ctx, p, grid); break;
        default: cnt ? launch_wide_cb<16, true>(ctx, p, grid) : launch_wide_cb<16, false>(ctx, p, grid); break;
    }
    return true;
}

bool launch_backward_wide(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                          float* d_colors, float* d_positions) {
    if (c->C <= 4 || c->rec == nullptr || c->ccol == nullptr || c->wsum64 != nullptr) return false;
    cudaStream_t st = ctx->stream;
    const int groups = (c->C + kBG - 1) / kBG;
    // CTA = one cell column x a segment of kBSeg cell rows
    int max_rows = c->grid_cap;
    if (!c->geom_h.empty()) {
        max_rows = 1;
        for (const auto& g : c->geom_h) max_rows = std::max(max_rows, g.n_rows);
    }
    const int nseg_cap = (max_rows + kBSeg - 1) / kBSeg;
    std::vector<int32_t> off(c->B + 1, 0);
    for (int b = 0; b < c->B; ++b) {
        const int ncols = c->geom_h.empty() ? c->grid_cap : c->geom_h[b].n_cols;
        off[b + 1] = off[b] + ncols * nseg_cap;
    }
    const int32_t* d_off = upload_table(ctx, WS_BLKOFF, off);
    BwdWideParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.blk_off = d_off;
    p.rec = c->rec;
    p.ccol = c->ccol;
    p.wsum = c->wsum;
    p.image = c->image;
    p.upstream = upstream;
    p.B = c->B;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.seg = kBSeg;
    p.nseg_cap = nseg_cap;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    p.inv_s2 = static_cast<float>(1.0 / (c->sigma * c->sigma));
    p.d_col = d_colors;
    const size_t n2 = static_cast<size_t>(c->B) * c->N * 2;
    float* part = static_cast<float*>(scratch(ctx, WS_PART, sizeof(float) * n2 * groups));
    p.d_pos = groups > 1 ? part : d_positions;
    if (off[c->B] > 0) {
        GMI_SMEM_ONCE(ctx, k_backward_wide, kBSmem);
        const int nunits = off[c->B];
        p.heavy_cap = std::min(2048, nunits);
        char* ws = static_cast<char*>(scratch(ctx, WS_TMP, sizeof(int32_t) * (1 + p.heavy_cap) + nunits));
        int32_t* d_cnt = reinterpret_cast<int32_t*>(ws);
        uint8_t* d_mark = reinterpret_cast<uint8_t*>(ws + sizeof(int32_t) * (1 + p.heavy_cap));
        p.heavy_count = d_cnt;
        p.heavy_list = d_cnt + 1;
        p.heavy_mark = d_mark;
        GMI_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int32_t), st));
        k_wide_unit_load<<<(nunits + 255) / 256, 256, 0, st>>>(c->geom_d, c->bins, d_off, c->B, kBSeg,
                                                                nseg_cap, p.heavy_cap, d_cnt + 1, d_cnt,
                                                                d_mark);
        GMI_LAUNCHED(ctx);
        k_backward_wide<<<dim3(p.heavy_cap + nunits, groups), kBThreads, kBSmem, st>>>(p);
        GMI_LAUNCHED(ctx);
    }
    if (groups > 1) {
        k_sum_groups_w<<<static_cast<unsigned>((n2 + 255) / 256), 256, 0, st>>>(part, d_positions, n2,
                                                                                groups);
        GMI_LAUNCHED(ctx);
    }
    return true;
}

}  // namespace gmi_host
