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
constexpr int kWCap = 256;       // staged candidates per chunk
constexpr int kWRuns = 32;       // cell rows per run group

template <int CB>
struct SmemWide {
    float4 pt[kWCap];            // x, y, idx|flag bits, 0
    float4 col[kWCap][CB];       // the pass's 4 CB channels
    int slot[kWCap];
    int run_beg[kWRuns + 1];
    int run_g[kWRuns];
    int rect[4];                 // cx0, cx1, cy0, cy1
};

struct GatherWideParams {
    const Geom* geom;
    const int32_t* bins;
    const float4* rec;   // [B][N][2] (x, y, c0, c1) (c2, c3, idx|flag, 0)
    const float* ccol;   // [B][N][C] colours in bin order
    int N, C, W, H;
    int nsg;             // channel passes of 4 CB channels
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
    const int sg = static_cast<int>(blockIdx.z) % p.nsg;
    const int b = static_cast<int>(blockIdx.z) / p.nsg;
    const int sgc0 = sg * 4 * CB;
    const int ch0 = sgc0 + cb * CB;
    const int nch = max(0, min(CB, p.C - ch0));
    const int x0 = blockIdx.x * kWT, y0 = blockIdx.y * kWT;
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
        for (int c0 = 0; c0 < total; c0 += kWCap) {
            const int n = min(kWCap, total - c0);
            // ---- stage positions / flags ----
            for (int k = tid; k < n; k += kWThreads) {
                const int e = c0 + k;
                int lo = 0, hi = nr;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (S.run_beg[mid] <= e) lo = mid;
                    else hi = mid;
                }
                const int slot = S.run_g[lo] + (e - S.run_beg[lo]);
                S.slot[k] = slot;
                const float4 ra = p.rec[(base + slot) * 2];
                const float rz = p.rec[(base + slot) * 2 + 1].z;
                S.pt[k] = make_float4(ra.x, ra.y, rz, 0.f);
            }
            __syncthreads();
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
            const float w = py ? (px ? Wb.y : Wb.x) : (px ? Wa.y : Wa.x);
            const size_t bp = (static_cast<size_t>(b) * p.H + qy) * p.W + qx;
            if (w > 0.f) {
                const float inv = 1.0f / w;
                float o[CB];
#pragma unroll
                for (int c = 0; c < CB; ++c) {
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

template <int CB, bool kCount>
void launch_wide_cb(gmi_ctx* ctx, const GatherWideParams& p, dim3 grid) {
    const int smem = static_cast<int>(sizeof(SmemWide<CB>));
    static int set_dev = -1;  // attribute set once per device
    if (set_dev != ctx->device) {
        set_dev = ctx->device;
        GMI_CUDA(cudaFuncSetAttribute(k_gather_wide<CB, kCount>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    k_gather_wide<CB, kCount><<<grid, kWThreads, smem, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

// ---------------------------------------------------------------------------
// K4 wide
// ---------------------------------------------------------------------------
constexpr int kBG = 16;                 // channels per group
constexpr int kBThreads = 256;          // 8 warps, one point each at a time
constexpr int kBSmem = 110 * 1024;      // staged bytes (68 per pixel), 2 CTAs/SM
constexpr int kBRunMax = 64;            // cell rows per block

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
    int bs;                  // cells per block side
    double r64, r2_64;
    float nk, inv_s2;
    float* d_col;            // [B][N][C]
    float* d_pos;            // partial [groups][B][N][2]
};

__device__ __forceinline__ bool in_ref_w(int x, int y, float mx, float my, double r2_64) {
    return d2_ref(static_cast<double>(x), static_cast<double>(y), static_cast<double>(mx),
                  static_cast<double>(my)) <= r2_64;
}

// u (this lane's 4 channels of the group) and the group's v at one pixel,
// straight from global memory (unstaged blocks); v is summed over the 4
// channel lanes of the pixel (lanes cl = 0..3 of the calling quad).
__device__ __forceinline__ void pixel_u4(const BwdWideParams& p, size_t img_base, int c0, int x,
                                         int y, float4& u, float& v, unsigned qmask) {
    u = make_float4(0.f, 0.f, 0.f, 0.f);
    float vp = 0.f;
    if (x >= 0 && x < p.W && y >= 0 && y < p.H) {
        const size_t pix = img_base + static_cast<size_t>(y) * p.W + x;
        const float wv = p.wsum[pix];
        if (wv > 0.f) {
            const float inv = 1.0f / wv;
            float uu[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uu[c] = 0.f;
                if (c0 + c < p.C) {
                    uu[c] = p.upstream[pix * p.C + c0 + c] * inv;
                    vp = fmaf(uu[c], p.image[pix * p.C + c0 + c], vp);
                }
            }
            u = make_float4(uu[0], uu[1], uu[2], uu[3]);
        }
    }
    vp += __shfl_xor_sync(qmask, vp, 1);
    vp += __shfl_xor_sync(qmask, vp, 2);
    v = vp;
}

__global__ void __launch_bounds__(kBThreads, 2)
k_backward_wide(BwdWideParams p) {
    extern __shared__ float4 s_u4[];      // [area][4] float4, then s_v[area]
    __shared__ int s_run[kBRunMax + 1];
    __shared__ int s_rung[kBRunMax];
    __shared__ float s_red[4][kBThreads / 32];
    __shared__ int s_region[5];

    // ---- image / cell block of this CTA ----
    int b = 0;
    {
        int lo = 0, hi = p.B;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (p.blk_off[mid] <= static_cast<int>(blockIdx.x)) lo = mid;
            else hi = mid;
        }
        b = lo;
    }
    const Geom g = p.geom[b];
    const int local = blockIdx.x - p.blk_off[b];
    const int nbx = (g.n_cols + p.bs - 1) / p.bs;
    const int cx0 = (local % nbx) * p.bs, cy0 = (local / nbx) * p.bs;
    if (cy0 >= g.n_rows) return;  // past this image's grid (device geometry)
    const int cx1 = min(cx0 + p.bs, g.n_cols), cy1 = min(cy0 + p.bs, g.n_rows);
    const int cg = blockIdx.y, ch0 = cg * kBG;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t base = static_cast<size_t>(b) * p.N;

    // ---- point runs (one per cell row of the block) ----
    const int nrun = cy1 - cy0;
    if (tid < 32) {
        int carry = 0;
        for (int k0 = 0; k0 < nrun; k0 += 32) {
            const int k = k0 + tid;
            int len = 0, gs = 0;
            if (k < nrun) {
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cy0 + k) * g.n_cols;
                gs = p.bins[r0 + cx0];
                len = p.bins[r0 + cx1] - gs;
            }
            int incl = len;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += t;
            }
            if (k < nrun) {
                s_run[k] = carry + incl - len;
                s_rung[k] = gs;
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (tid == 0) s_run[nrun] = carry;
    }
    __syncthreads();
    const int total = s_run[nrun];
    if (total == 0) return;
    auto slot_of = [&](int k) -> int {
        int lo = 0, hi = nrun;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_run[mid] <= k) lo = mid;
            else hi = mid;
        }
        return s_rung[lo] + (k - s_run[lo]);
    };

    // ---- pixel region reached by the block's points (as k_backward_points) ----
    if (tid == 0) {
        s_region[4] = -2;
        if (!g.capped) {
            const double pad = p.r64 + 1.0;
            const int x0 = max(0, static_cast<int>(floor(g.ox + cx0 * g.cell - pad))) & ~1;
            const int y0 = max(0, static_cast<int>(floor(g.oy + cy0 * g.cell - pad)));
            const int x1 = min(p.W - 1, static_cast<int>(ceil(g.ox + cx1 * g.cell + pad))) | 1;
            const int y1 = min(p.H - 1, static_cast<int>(ceil(g.oy + cy1 * g.cell + pad)));
            const long wd = (x1 >= x0) ? (x1 - x0 + 1) : 0;
            const long area = (y1 >= y0) ? wd * (y1 - y0 + 1) : 0;
            if (area <= 0) {
                s_region[4] = -1;
            } else if (area * 68 <= kBSmem) {
                s_region[0] = x0;
                s_region[1] = y0;
                s_region[2] = x1;
                s_region[3] = y1;
                s_region[4] = 1;
            }
        }
    }
    __syncthreads();
    if (s_region[4] == -2) {
        float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
        for (int k = tid; k < total; k += kBThreads) {
            const float4 ra = p.rec[(base + slot_of(k)) * 2];
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
            const float rr = static_cast<float>(p.r64) + 2.0f;
            int x0 = max(0, static_cast<int>(floorf(fmaxf(mnx - rr, -1.0e9f))));
            const int y0 = max(0, static_cast<int>(floorf(fmaxf(mny - rr, -1.0e9f))));
            int x1 = min(p.W - 1, static_cast<int>(ceilf(fminf(mxx + rr, 1.0e9f))));
            const int y1 = min(p.H - 1, static_cast<int>(ceilf(fminf(mxy + rr, 1.0e9f))));
            x0 &= ~1;
            x1 |= 1;
            s_region[0] = x0;
            s_region[1] = y0;
            s_region[2] = x1;
            s_region[3] = y1;
            const long wd = (x1 >= x0) ? (x1 - x0 + 1) : 0;
            const long area = (y1 >= y0) ? wd * (y1 - y0 + 1) : 0;
            s_region[4] = (mnx <= mxx && area > 0 && area * 68 <= kBSmem) ? 1 : (area > 0 ? 0 : -1);
        }
        __syncthreads();
    }
    const int rx0 = s_region[0], ry0 = s_region[1], rx1 = s_region[2], ry1 = s_region[3];
    const int mode = s_region[4];
    if (mode < 0) {
        // no frame pixel is reachable: gradients are zero
        for (int k = tid; k < total; k += kBThreads) {
            const int sk = slot_of(k);
            const int i = static_cast<int>(__float_as_uint(p.rec[(base + sk) * 2 + 1].z) & 0x7fffffffu);
            for (int c = ch0; c < min(p.C, ch0 + kBG); ++c) p.d_col[(base + i) * p.C + c] = 0.f;
            float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
            dp[0] = 0.f;
            dp[1] = 0.f;
        }
        return;
    }
    const bool staged = mode == 1;
    const int wd = rx1 - rx0 + 1;  // even
    const int area = wd * (ry1 - ry0 + 1);
    float* s_v = reinterpret_cast<float*>(s_u4 + (staged ? 4 * area : 0));
    const size_t img_base = static_cast<size_t>(b) * p.H * p.W;
    const int cl = lane & 3;           // channel quad of the lane
    const int c4 = ch0 + 4 * cl;       // its first channel

    if (staged) {
        // 4 lanes per pixel (16 channels), pixels row-major over the region,
        // two pixels per thread and iteration with all loads issued up front
        const bool full = (p.C % 4) == 0 && c4 + 3 < p.C &&
                          (reinterpret_cast<uintptr_t>(p.upstream) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(p.image) & 15) == 0;
        constexpr int kStep = kBThreads / 4;
        auto adv = [&](int& r, int& cc) {
            cc += kStep;
            while (cc >= wd) {
                cc -= wd;
                ++r;
            }
        };
        auto load = [&](bool live, int r, int cc, float& w, float4& up, float4& im) {
            const int yy = ry0 + r, xx = rx0 + cc;
            const bool in = live && xx < p.W && yy < p.H;
            const size_t pix = img_base + (in ? static_cast<size_t>(yy) * p.W + xx : 0);
            w = 0.f;
            up = make_float4(0.f, 0.f, 0.f, 0.f);
            im = up;
            if (in) {
                w = p.wsum[pix];
                if (full) {
                    up = *reinterpret_cast<const float4*>(p.upstream + pix * p.C + c4);
                    im = *reinterpret_cast<const float4*>(p.image + pix * p.C + c4);
                } else {
                    float t[8];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        t[c] = c4 + c < p.C ? p.upstream[pix * p.C + c4 + c] : 0.f;
                        t[4 + c] = c4 + c < p.C ? p.image[pix * p.C + c4 + c] : 0.f;
                    }
                    up = make_float4(t[0], t[1], t[2], t[3]);
                    im = make_float4(t[4], t[5], t[6], t[7]);
                }
            }
        };
        auto put = [&](bool live, int k, float w, const float4& up, const float4& im) {
            const float inv = w > 0.f ? 1.0f / w : 0.f;  // W == 0: fallback pixel, zeros
            const float4 u = make_float4(up.x * inv, up.y * inv, up.z * inv, up.w * inv);
            float vp = fmaf(u.w, im.w, fmaf(u.z, im.z, fmaf(u.y, im.y, u.x * im.x)));
            vp += __shfl_xor_sync(0xffffffffu, vp, 1);
            vp += __shfl_xor_sync(0xffffffffu, vp, 2);
            if (live) {
                s_u4[4 * k + cl] = u;
                if (cl == 0) s_v[k] = vp;
            }
        };
        int rA = (tid >> 2) / wd, cA = (tid >> 2) - rA * wd;
        int rB = rA, cB = cA;
        adv(rB, cB);
        for (int kb = 0; kb < area; kb += 2 * kStep) {
            const int kA = kb + (tid >> 2), kB = kA + kStep;
            float wA, wB;
            float4 uA, oA, uB, oB;
            load(kA < area, rA, cA, wA, uA, oA);
            load(kB < area, rB, cB, wB, uB, oB);
            put(kA < area, kA, wA, uA, oA);
            put(kB < area, kB, wB, uB, oB);
            adv(rA, cA);
            adv(rA, cA);
            adv(rB, cB);
            adv(rB, cB);
        }
        __syncthreads();
    }

    // ---- per point: one warp, 4 teams of 8 lanes on interleaved rows ----
    const float nk = p.nk;
    const float r2f = static_cast<float>(p.r2_64), rf = static_cast<float>(p.r64);
    const double r2_64 = p.r2_64;
    const int xmin = max(rx0, 0), xmax = min(rx1, p.W - 1);
    const int team = lane >> 3, h = (lane >> 2) & 1;
    const unsigned qmask = 0xfu << (lane & ~3);
    for (int k = warp; k < total; k += kBThreads / 32) {
        const int s = slot_of(k);
        const float4 ra = p.rec[(base + s) * 2];
        const uint32_t raw = __float_as_uint(p.rec[(base + s) * 2 + 1].z);
        const float mx = ra.x, my = ra.y;
        const int i = static_cast<int>(raw & 0x7fffffffu);
        const bool unsafe = (raw & kUnsafeBit) != 0;
        float cc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) cc[c] = c4 + c < p.C ? p.ccol[(base + s) * p.C + c4 + c] : 0.f;
        float dcol[4] = {0.f, 0.f, 0.f, 0.f}, gxc[4] = {0.f, 0.f, 0.f, 0.f},
              gyc[4] = {0.f, 0.f, 0.f, 0.f};
        float vx = 0.f, vy = 0.f;
        const float tx = truncf(mx);
        const float fmu = mx - tx;  // exact
        const int bx = static_cast<int>(tx);
        const float pad = unsafe ? 1.0f : 1e-2f;
        const int ya = max(ry0, static_cast<int>(ceilf(my - rf - pad))) + team;
        const int yb = min(ry1, static_cast<int>(floorf(my + rf + pad)));
        float yf = static_cast<float>(ya);
        for (int y = ya; y <= yb; y += 4, yf += 4.f) {
            float dy;
            int xl, xr;
            if (!unsafe) {
                dy = yf - my;
                const float h2f = fmaf(-dy, dy, r2f);
                if (h2f < 0.f) continue;
                const float sq = h2f * rsqrtf(fmaxf(h2f, 1e-30f));
                constexpr float kMagic = 12582912.0f;
                constexpr int kMagicBits = 0x4B400000;
                xl = bx + (__float_as_int(__fadd_ru(fmu - sq, kMagic)) - kMagicBits);
                xr = bx + (__float_as_int(__fadd_rd(fmu + sq, kMagic)) - kMagicBits);
            } else {
                const double dy64 = __dsub_rn(static_cast<double>(y), static_cast<double>(my));
                const double h2 = __dsub_rn(r2_64, __dmul_rn(dy64, dy64));
                if (h2 < 0.0) continue;
                const float sq = sqrtf(static_cast<float>(h2));
                xl = bx + static_cast<int>(ceilf(fmu - sq));
                xr = bx + static_cast<int>(floorf(fmu + sq));
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
            if (xl > xr) continue;
            const float ey = (dy * nk) * dy;
            // pair-aligned span: pairs xs, xs+2, ..; the lane takes x = xs+2j+h
            const int xs = xl - ((xl - rx0) & 1);
            const int np = ((xr - xs) >> 1) + 1;
            const bool mfirst = h == 0 && ((xl - rx0) & 1);
            const bool mlast = h == 1 && !((xr - rx0) & 1);
            float xf = static_cast<float>(xs + h);
            float R[4] = {0.f, 0.f, 0.f, 0.f};
            float vr = 0.f;
            if (staged) {
                // this lane's pixels x = xs + h + 2j, j in [j0, j1), all in [xl, xr]
                const int j0 = mfirst ? 1 : 0, j1 = mlast ? np - 1 : np;
                const int kk0 = (y - ry0) * wd + (xs - rx0) + h + 2 * j0;
                const float4* pu = s_u4 + 4 * kk0 + cl;
                const float* pv = s_v + kk0;
                xf += static_cast<float>(2 * j0);
#pragma unroll 2
                for (int j = j0; j < j1; ++j) {
                    const float4 u = *pu;
                    const float v = *pv;
                    const float dx = xf - mx;
                    const float w = ex2(fmaf(dx * nk, dx, ey));
                    const float wdx = w * dx;
                    R[0] = fmaf(w, u.x, R[0]);
                    R[1] = fmaf(w, u.y, R[1]);
                    R[2] = fmaf(w, u.z, R[2]);
                    R[3] = fmaf(w, u.w, R[3]);
                    gxc[0] = fmaf(wdx, u.x, gxc[0]);
                    gxc[1] = fmaf(wdx, u.y, gxc[1]);
                    gxc[2] = fmaf(wdx, u.z, gxc[2]);
                    gxc[3] = fmaf(wdx, u.w, gxc[3]);
                    vx = fmaf(wdx, v, vx);
                    vr = fmaf(w, v, vr);
                    xf += 2.f;
                    pu += 8;
                    pv += 2;
                }
            } else {
                for (int j = 0; j < np; ++j) {
                    float4 u;
                    float v;
                    pixel_u4(p, img_base, c4, xs + 2 * j + h, y, u, v, qmask);
                    const float dx = xf - mx;
                    float w = ex2(fmaf(dx * nk, dx, ey));
                    if ((j == 0 && mfirst) || (j == np - 1 && mlast)) w = 0.f;
                    const float wdx = w * dx;
                    R[0] = fmaf(w, u.x, R[0]);
                    R[1] = fmaf(w, u.y, R[1]);
                    R[2] = fmaf(w, u.z, R[2]);
                    R[3] = fmaf(w, u.w, R[3]);
                    gxc[0] = fmaf(wdx, u.x, gxc[0]);
                    gxc[1] = fmaf(wdx, u.y, gxc[1]);
                    gxc[2] = fmaf(wdx, u.z, gxc[2]);
                    gxc[3] = fmaf(wdx, u.w, gxc[3]);
                    vx = fmaf(wdx, v, vx);
                    vr = fmaf(w, v, vr);
                    xf += 2.f;
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                dcol[c] += R[c];
                gyc[c] = fmaf(dy, R[c], gyc[c]);
            }
            vy = fmaf(dy, vr, vy);
        }
        // combine the two pixel halves and the four teams (fixed tree)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                dcol[c] += __shfl_xor_sync(0xffffffffu, dcol[c], o);
                gxc[c] += __shfl_xor_sync(0xffffffffu, gxc[c], o);
                gyc[c] += __shfl_xor_sync(0xffffffffu, gyc[c], o);
            }
            vx += __shfl_xor_sync(0xffffffffu, vx, o);
            vy += __shfl_xor_sync(0xffffffffu, vy, o);
        }
        // d_pos of this group: sum_c c_ic G_c over the 4 channel lanes - v
        float gx = cc[0] * gxc[0], gy = cc[0] * gyc[0];
#pragma unroll
        for (int c = 1; c < 4; ++c) {
            gx = fmaf(cc[c], gxc[c], gx);
            gy = fmaf(cc[c], gyc[c], gy);
        }
        gx += __shfl_xor_sync(0xffffffffu, gx, 1);
        gy += __shfl_xor_sync(0xffffffffu, gy, 1);
        gx += __shfl_xor_sync(0xffffffffu, gx, 2);
        gy += __shfl_xor_sync(0xffffffffu, gy, 2);
        if (lane < 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c4 + c < p.C) p.d_col[(base + i) * p.C + c4 + c] = dcol[c];
        }
        if (lane == 0) {
            float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
            dp[0] = (gx - vx) * p.inv_s2;
            dp[1] = (gy - vy) * p.inv_s2;
        }
    }
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
    const dim3 grid((c->W + kWT - 1) / kWT, (c->H + kWT - 1) / kWT, c->B * p.nsg);
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
    // cells per block side so that the staged region (~(bs cell + 2r + 4)^2
    // pixels of 68 B) fits the budget
    const double cell = c->cutoff;
    const double side_px = std::sqrt(static_cast<double>(kBSmem) / 68.0);
    int bs = static_cast<int>(std::floor((side_px - 2.0 * c->cutoff - 4.0) / cell));
    bs = std::max(1, std::min(bs, kBRunMax));
    std::vector<int32_t> off(c->B + 1, 0);
    for (int b = 0; b < c->B; ++b) {
        int nb;
        if (c->geom_h.empty()) {
            const int side = (c->grid_cap + bs - 1) / bs;
            nb = side * side;
        } else {
            const auto& g = c->geom_h[b];
            nb = ((g.n_cols + bs - 1) / bs) * ((g.n_rows + bs - 1) / bs);
        }
        off[b + 1] = off[b] + nb;
    }
    int32_t* d_off = static_cast<int32_t*>(scratch(ctx, WS_BLKOFF, sizeof(int32_t) * (c->B + 1)));
    GMI_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * (c->B + 1),
                             cudaMemcpyHostToDevice, st));
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
    p.bs = bs;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    p.inv_s2 = static_cast<float>(1.0 / (c->sigma * c->sigma));
    p.d_col = d_colors;
    const size_t n2 = static_cast<size_t>(c->B) * c->N * 2;
    float* part = static_cast<float*>(scratch(ctx, WS_PART, sizeof(float) * n2 * groups));
    p.d_pos = groups > 1 ? part : d_positions;
    if (off[c->B] > 0) {
        static int set_dev = -1;
        if (set_dev != ctx->device) {
            set_dev = ctx->device;
            GMI_CUDA(cudaFuncSetAttribute(k_backward_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kBSmem));
        }
        k_backward_wide<<<dim3(off[c->B], groups), kBThreads, kBSmem, st>>>(p);
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
