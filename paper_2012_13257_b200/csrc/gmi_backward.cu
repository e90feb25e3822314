// K4 — backward (engine.cpp:190-234 backward_rows, engine.cpp:238-309).
//
// Point-major and atomic-free.  A CTA takes a block of reference cells and
// stages, for every pixel those points can reach,
//     u_c = upstream_c / W      and      -v = -sum_c u_c out_c
// (zeros on fallback pixels) in shared memory as interleaved PIXEL PAIRS
// (x even, x+1): (CG + 1) float2 = 16 bytes per pixel for C = 3, so two
// pixels are processed per f32x2 instruction (FFMA2 / FMUL2 / FADD2, sm_100).
// Every thread owns whole points and walks the point's exact disk row by row
// — the reference's closed ball d^2 <= r^2 (bin_grid.cpp:98; exact spans from
// one fp32 reciprocal-sqrt per row, or the f64 predicate for points K1
// flagged as boundary-ambiguous) — recomputing the Gaussian weight with the
// forward's own fp32 operations (bit-identical to the weight summed into W)
// instead of storing it.  Per pair it accumulates in registers
//     d_col_c += w * u_c                         (= up_c w/W, engine.cpp:222)
//     d_pos   += w * (sum_c c_ic u_c - v) * (q - mu) / sigma^2
//                                     (= ratio * dot / sigma^2 * (q-mu), engine.cpp:219-230)
// and writes each point's gradients once.  One owner per point: the result
// is bit-deterministic with no atomics and no reduction pass.  Images of
// >= 2^20 points write the gradients in slot order instead and
// k_permute_grads moves them to the original indices (slot_grads).
//
// K5 — fallback pixels under NearestPoint route their upstream to the nearest
// point's colour (engine.cpp:200-211), summed in per-point fixed point
// (deterministic whatever the arrival order).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

#ifndef GMI_BWD_WARPS
#define GMI_BWD_WARPS 8
#endif
constexpr int kThreads = 32 * GMI_BWD_WARPS;
#ifndef GMI_BWD_CTAS
#define GMI_BWD_CTAS (32 / GMI_BWD_WARPS)
#endif
constexpr int kCtasPerSm = GMI_BWD_CTAS;  // 8 warps x 4 CTAs: 64 registers, 32 warps per SM
constexpr int kSmemBudget = (208 / kCtasPerSm) * 1024;  // staged pixel bytes per CTA (4 CTAs/SM: 52 KB)
constexpr int kRunMax = 64;             // cell rows per block
#ifndef GMI_BWD_STAGE_UNROLL
#define GMI_BWD_STAGE_UNROLL 1
#endif
constexpr int kStageUnroll = GMI_BWD_STAGE_UNROLL;  // staging pairs in flight per lane

struct BwdParams {
    const Geom* geom;
    const int32_t* bins;
    const float* sx;
    const float* sy;
    const int32_t* sidx;
    const float* scol;      // [B][C][N]
    const float4* rec;      // fast layout [B][N][2] (replaces sx/sy/sidx/scol)
    const float* ccol;      // C > 4 with the fast layout: [B][N][C] colours
    int lpp;                // lanes per point (1, 2, 4, 8): rows split over lanes
    const float* wsum;      // [B][H][W]
    const float* image;     // [B][H][W][C]
    const double* image64;  // [B][H][W][C] f64 image (precise mode) or null
    const float* upstream;  // [B][H][W][C]
    int B, N, C, W, H;
    int b0;                 // first image of this launch (grid z <= 65535)
    int bs;                 // cells per block side
    double r64, r2_64;
    float nk;               // -log2(e) / (2 sigma^2)
    float r2f;              // float(r^2) (kept in the constant bank: no per-row conversion)
    float inv_s2;
    float* d_col;           // [B][N][C]
    float* d_pos;           // [B][N][2] or partial [G][B][N][2]
    float4* gslot;          // large images: [B][N][2] gradients in SLOT order
                            // (d_col[0..3], d_pos), permuted by k_permute_grads
};

__device__ __forceinline__ bool in_ref(int x, int y, float mx, float my, double r2_64) {
    return d2_ref(static_cast<double>(x), static_cast<double>(y), static_cast<double>(mx),
                  static_cast<double>(my)) <= r2_64;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// float4 slots per staged pixel pair: CG u-pairs + the (-v) pair, as float2
template <int CG>
struct PairLayout {
    static constexpr int kF2 = CG + 1;
    static constexpr int kF4 = (kF2 + 1) / 2;
};

// Per-pixel terms of the backward (engine.cpp:213-231), for this channel
// group:  u_c = up_c / W  and  v = sum_c u_c * out_c, so that per pair
//     ratio * up_c = w * u_c,   ratio * dot = w * (sum_c c_ic u_c - v).
// Fallback pixels (W == 0) and off-frame pixels stage zeros (K5 routes the
// fallback upstream).
template <int CG>
__device__ __forceinline__ void pixel_terms(const BwdParams& p, size_t img_base, int ch0, int nch,
                                            int x, int y, float* u, float& v) {
#pragma unroll
    for (int c = 0; c < CG; ++c) u[c] = 0.f;
    v = 0.f;
    if (x < 0 || x >= p.W || y < 0 || y >= p.H) return;
    const size_t pix = img_base + static_cast<size_t>(y) * p.W + x;
    const float wv = p.wsum[pix];
    if (!(wv > 0.f)) return;
    const float inv = 1.0f / wv;
#pragma unroll
    for (int c = 0; c < CG; ++c) {
        if (c < nch) {
            u[c] = p.upstream[pix * p.C + ch0 + c] * inv;
            v = fmaf(u[c], p.image[pix * p.C + ch0 + c], v);
        }
    }
}

template <int CG, int LPP>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
k_backward_points(BwdParams p) {
    using L = PairLayout<CG>;
    // slot-major planes at a FIXED stride (the budget's share per plane), so
    // the pair loop's second plane is an immediate offset from the first
    constexpr int kPlane = kSmemBudget / (L::kF4 * static_cast<int>(sizeof(float4)));
    extern __shared__ float4 s_pair[];   // [L::kF4][kPlane]: rows x pairs in each
    __shared__ int s_run[kRunMax + 1];   // prefix of the block's cell-row runs
    __shared__ int s_rung[kRunMax];      // first slot of each run
    __shared__ float s_red[4][kThreads / 32];
    __shared__ int s_region[5];

    // ---- image / cell block of this CTA (grid: blocks x groups x images;
    // blocks past this image's own grid exit at once) ----
    const int b = p.b0 + static_cast<int>(blockIdx.z);
    const Geom g = p.geom[b];
    const int local = blockIdx.x;
    const int nbx = (g.n_cols + p.bs - 1) / p.bs;
    const int cx0 = (local % nbx) * p.bs, cy0 = (local / nbx) * p.bs;
    if (cy0 >= g.n_rows) return;
    const int cx1 = min(cx0 + p.bs, g.n_cols), cy1 = min(cy0 + p.bs, g.n_rows);
    const int cg = blockIdx.y, ch0 = cg * CG, nch = min(CG, p.C - ch0);
    const int tid = threadIdx.x, lane = tid & 31;
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
    // k-th point of the block -> slot (binary search over the runs)
    auto slot_of = [&](int k) -> int {
        int lo = 0, hi = nrun;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_run[mid] <= k) lo = mid;
            else hi = mid;
        }
        const int s = s_rung[lo] + (k - s_run[lo]);
        GMI_CHECK(s >= 0 && s < p.N);
        return s;
    };

    // ---- pixel region reached by the block's points ----
    // Uncapped grids: the block's cells bound its points' positions exactly
    // (cell_of = floor((v - origin) / cell), no clamping in use), so the
    // region is the cell rectangle grown by r — no pass over the points.
    // Capped grids (clamped edge cells) or an oversized rectangle: the
    // points' bbox grown by r.
    if (tid == 0) {
        s_region[4] = -2;
        if (!g.capped) {
            const double pad = p.r64 + 1.0;
            const int x0 = max(0, static_cast<int>(floor(g.ox + cx0 * g.cell - pad))) & ~1;
            const int y0 = max(0, static_cast<int>(floor(g.oy + cy0 * g.cell - pad)));
            const int x1 = min(p.W - 1, static_cast<int>(ceil(g.ox + cx1 * g.cell + pad))) | 1;
            const int y1 = min(p.H - 1, static_cast<int>(ceil(g.oy + cy1 * g.cell + pad)));
            const long npairs = (x1 >= x0) ? (x1 - x0 + 1) / 2 : 0;
            const long area = (y1 >= y0) ? npairs * (y1 - y0 + 1) : 0;
            if (area <= 0) {
                s_region[4] = -1;
            } else if (area * L::kF4 * static_cast<long>(sizeof(float4)) <= kSmemBudget) {
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
    for (int k = tid; k < total; k += kThreads) {
        const int s = slot_of(k);
        float x, y;
        if (p.rec) {
            const float4 ra = p.rec[(base + s) * 2];
            x = ra.x;
            y = ra.y;
        } else {
            x = p.sx[base + s];
            y = p.sy[base + s];
        }
        mnx = fminf(mnx, x);
        mny = fminf(mny, y);
        mxx = fmaxf(mxx, x);
        mxy = fmaxf(mxy, y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    if (lane == 0) {
        s_red[0][tid >> 5] = mnx;
        s_red[1][tid >> 5] = mny;
        s_red[2][tid >> 5] = mxx;
        s_red[3][tid >> 5] = mxy;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kThreads / 32; ++w) {
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
        x0 &= ~1;        // pairs start at even x
        x1 |= 1;         // and end at odd x (may exceed the frame: zero-staged)
        s_region[0] = x0;
        s_region[1] = y0;
        s_region[2] = x1;
        s_region[3] = y1;
        const long npairs = (x1 >= x0) ? (x1 - x0 + 1) / 2 : 0;
        const long area = (y1 >= y0) ? npairs * (y1 - y0 + 1) : 0;
        s_region[4] = (mnx <= mxx && area > 0 &&
                       area * L::kF4 * static_cast<long>(sizeof(float4)) <= kSmemBudget)
                          ? 1
                          : (area > 0 ? 0 : -1);
    }
    __syncthreads();
    }
    const int rx0 = s_region[0], ry0 = s_region[1], rx1 = s_region[2], ry1 = s_region[3];
    const int mode = s_region[4];
    if (mode < 0) {
        // no frame pixel is reachable: gradients are zero
        for (int k = tid; k < total; k += kThreads) {
            const int sk = slot_of(k);
            const int i = (p.rec ? static_cast<int>(__float_as_uint(p.rec[(base + sk) * 2 + 1].z))
                                 : p.sidx[base + sk]) & 0x7fffffff;
            for (int c = 0; c < nch; ++c) p.d_col[(base + i) * p.C + ch0 + c] = 0.f;
            float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
            dp[0] = 0.f;
            dp[1] = 0.f;
        }
        return;
    }
    const bool staged = mode == 1;
    const int npairs = (rx1 - rx0 + 1) / 2;
    const int area = npairs * (ry1 - ry0 + 1);  // <= kPlane when staged (bounds checks)
    (void)area;
    const size_t img_base = static_cast<size_t>(b) * p.H * p.W;

    if (staged) {
        // 8-byte alignment of a pixel pair in W / upstream / image rows
        // (64-bit loads: the caller's upstream / image may be any float
        // pointer, e.g. a view at an odd element offset)
        const bool vec = (p.W % 2 == 0) && (CG == p.C) &&
                         ((reinterpret_cast<uintptr_t>(p.upstream) |
                           reinterpret_cast<uintptr_t>(p.image)) & 7) == 0;
        const bool vec4 = CG == 4 && (p.C % 4) == 0 && (p.W % 2) == 0 &&
                          (reinterpret_cast<uintptr_t>(p.upstream) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(p.image) & 15) == 0;
        // rows by warps, pixel pairs by lanes (coalesced, no index division)
        const int nrows = ry1 - ry0 + 1;
        for (int row = tid >> 5; row < nrows; row += kThreads / 32)
#pragma unroll kStageUnroll
        for (int pp = lane; pp < npairs; pp += 32) {
            const int k = row * npairs + pp, yy = ry0 + row;
            const int xa = rx0 + 2 * pp;
            float ua[CG], ub[CG], va = 0.f, vb = 0.f;
            if (vec && xa >= 0 && xa + 1 < p.W && yy < p.H) {
                // both pixels in the frame: 64-bit loads of the pair
                const size_t pix = img_base + static_cast<size_t>(yy) * p.W + xa;
                const float2 wv = *reinterpret_cast<const float2*>(p.wsum + pix);
                const float2* up2 = reinterpret_cast<const float2*>(p.upstream + pix * CG);
                const float2* im2 = reinterpret_cast<const float2*>(p.image + pix * CG);
                float upv[2 * CG], imv[2 * CG];
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    const float2 a = up2[j], c2 = im2[j];
                    upv[2 * j] = a.x;
                    upv[2 * j + 1] = a.y;
                    imv[2 * j] = c2.x;
                    imv[2 * j + 1] = c2.y;
                }
                const float ia = wv.x > 0.f ? 1.0f / wv.x : 0.f;
                const float ib = wv.y > 0.f ? 1.0f / wv.y : 0.f;
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    ua[c] = upv[c] * ia;
                    ub[c] = upv[CG + c] * ib;
                    va = fmaf(ua[c], imv[c], va);
                    vb = fmaf(ub[c], imv[CG + c], vb);
                }
            } else if (vec4 && xa >= 0 && xa + 1 < p.W && yy < p.H) {
                // channel group of 4 inside C % 4 == 0 channels: 128-bit
                // loads of the group's slice of both pixels
                const size_t pix = img_base + static_cast<size_t>(yy) * p.W + xa;
                const float2 wv = *reinterpret_cast<const float2*>(p.wsum + pix);
                const float4 ua4 = *reinterpret_cast<const float4*>(p.upstream + pix * p.C + ch0);
                const float4 ub4 = *reinterpret_cast<const float4*>(p.upstream + (pix + 1) * p.C + ch0);
                const float4 oa4 = *reinterpret_cast<const float4*>(p.image + pix * p.C + ch0);
                const float4 ob4 = *reinterpret_cast<const float4*>(p.image + (pix + 1) * p.C + ch0);
                const float ia = wv.x > 0.f ? 1.0f / wv.x : 0.f;
                const float ib = wv.y > 0.f ? 1.0f / wv.y : 0.f;
                const float uav[4] = {ua4.x, ua4.y, ua4.z, ua4.w}, ubv[4] = {ub4.x, ub4.y, ub4.z, ub4.w};
                const float oav[4] = {oa4.x, oa4.y, oa4.z, oa4.w}, obv[4] = {ob4.x, ob4.y, ob4.z, ob4.w};
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    ua[c] = uav[c] * ia;
                    ub[c] = ubv[c] * ib;
                    va = fmaf(ua[c], oav[c], va);
                    vb = fmaf(ub[c], obv[c], vb);
                }
            } else {
                pixel_terms<CG>(p, img_base, ch0, nch, xa, yy, ua, va);
                pixel_terms<CG>(p, img_base, ch0, nch, xa + 1, yy, ub, vb);
            }
            float2 e[2 * L::kF4];
#pragma unroll
            for (int c = 0; c < CG; ++c) e[c] = f2(ua[c], ub[c]);
            e[CG] = f2(-va, -vb);
#pragma unroll
            for (int c = CG + 1; c < 2 * L::kF4; ++c) e[c] = f2(0.f, 0.f);
            // slot-major planes (16-byte stride: conflict-light LDS.128)
#pragma unroll
            for (int j = 0; j < L::kF4; ++j)
            {
                GMI_CHECK(k >= 0 && k < area);
                s_pair[j * kPlane + k] = make_float4(e[2 * j].x, e[2 * j].y, e[2 * j + 1].x, e[2 * j + 1].y);
            }
        }
        __syncthreads();
    }

    // ---- per point ----
    const float nk = p.nk, inv_s2 = p.inv_s2;
    const float r2f = p.r2f, rf = static_cast<float>(p.r64);
    const double r2_64 = p.r2_64;
    const int xmin = max(rx0, 0), xmax = min(rx1, p.W - 1);
    const float2 nk2 = f2(nk, nk), two = f2(2.f, 2.f);
    // warp tasks of 32/lpp consecutive points (bin order keeps a warp's points
    // adjacent), dealt round-robin.
    // With lpp > 1 (wide radii) the lpp lanes of a point take interleaved rows
    // of its disk and their partial sums are combined by a fixed shuffle tree.
    const int warp = tid >> 5;
    constexpr int lpp = LPP;
    const int sub = lane & (lpp - 1);
    const int ppw = 32 / lpp;                 // points per warp task
    const int pstep = (kThreads / 32) * ppw;  // points per CTA round
    for (int kb = warp * ppw; kb < total; kb += pstep) {
        const int k = kb + lane / lpp;
        // the task's own record, loaded at its start (other warps hide the
        // latency; a register prefetch of the next task's record cost 9
        // registers and spills: 1.993 vs 1.962 ms)
        float4 cra = make_float4(0.f, 0.f, 0.f, 0.f), crb = cra;
        const int cs = p.rec && k < total ? slot_of(k) : 0;
        if (p.rec && k < total) {
            cra = p.rec[(base + cs) * 2];
            crb = p.rec[(base + cs) * 2 + 1];
        }
        const bool live = k < total;
        if (lpp == 1 && !live) continue;
        const int s = p.rec ? cs : slot_of(min(k, total - 1));
        float mx, my;
        uint32_t raw;
        float cc[CG];
        if (p.rec) {
            // fast layout: C <= 4, one channel group
            const float4 ra = cra;
            const float4 rb = crb;
            mx = ra.x;
            my = ra.y;
            raw = __float_as_uint(rb.z);
            if (p.ccol != nullptr) {
#pragma unroll
                for (int c = 0; c < CG; ++c)
                    cc[c] = c < nch ? p.ccol[(base + s) * p.C + ch0 + c] : 0.f;
            } else {
                const float cv[4] = {ra.z, ra.w, rb.x, rb.y};
#pragma unroll
                for (int c = 0; c < CG; ++c) cc[c] = cv[c];
            }
        } else {
            mx = p.sx[base + s];
            my = p.sy[base + s];
            raw = static_cast<uint32_t>(p.sidx[base + s]);
#pragma unroll
            for (int c = 0; c < CG; ++c)
                cc[c] = c < nch ? p.scol[(static_cast<size_t>(b) * p.C + ch0 + c) * p.N + s] : 0.f;
        }
        const int i = static_cast<int>(raw & 0x7fffffffu);
        const bool unsafe = (raw & kUnsafeBit) != 0;
        float2 dcol[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) dcol[c] = f2(0.f, 0.f);
        // d_pos: fp32 pair sums over the whole disk, a * dx and a * dy per
        // pixel (round 2 first formed per-row sums and folded them in f64;
        // the strict fuzz shows no difference at the same seeds — the same 0
        // images over 1x in the BASELINE regimes, the same contract-domain
        // misses — and the per-row folds cost registers and ~10 SASS a row)
        float2 gx2 = f2(0.f, 0.f), gy2 = f2(0.f, 0.f);
        const float tx = truncf(mx);
        const float fmu = mx - tx;  // exact
        const int bx = static_cast<int>(tx);
        // rows that can hold an in-ball pixel: a safe point's boundary rows are
        // decided by the fp32 test below, so a small pad (>> fp32 rounding of
        // my +- r) suffices; flagged points keep a one-row margin for the f64
        // predicate
        const float pad = unsafe ? 1.0f : 1e-2f;
        const int ya = max(ry0, static_cast<int>(ceilf(my - rf - pad))) + sub;
        const int yb = live ? min(ry1, static_cast<int>(floorf(my + rf + pad))) : ya - 1;

        // the disk walk, compiled twice: warps without a flagged point (all
        // but ~0.3% at random inputs) run a copy with no f64 branch in it
        auto walk = [&](auto safe_only, auto staged_c) {
        float yf = static_cast<float>(ya);  // exact row coordinate
        // the row's staged pairs, advanced with the row (ya >= ry0 when the
        // region is staged; unused otherwise)
        const float4* rowp = s_pair + (ya - ry0) * npairs;
        for (int y = ya; y <= yb; y += lpp, yf += static_cast<float>(lpp), rowp += lpp * npairs) {
            float dy;
            int xl, xr;
            if (decltype(safe_only)::value || !unsafe) {
                // safe point: fp32 row geometry decides the reference's ball;
                // dy = y - my is the forward's own operation (bit-identical)
                dy = yf - my;
                const float h2f = fmaf(-dy, dy, r2f);
                if (h2f < 0.f) continue;
                // ~2 ulp: a safe point's row ends are >= 8e-6 r^2 from the ball
                const float sq = h2f * rsqrt_ftz(fmaxf(h2f, 1e-30f));
                // ceil / floor of small values by directed-rounding adds of
                // 1.5 * 2^23 (FMA pipe, no conversion on the XU pipe)
                constexpr float kMagic = 12582912.0f;
                constexpr int kMagicBits = 0x4B400000;
                xl = bx + (__float_as_int(__fadd_ru(fmu - sq, kMagic)) - kMagicBits);
                xr = bx + (__float_as_int(__fadd_rd(fmu + sq, kMagic)) - kMagicBits);
            } else {
                const double dy64 = __dsub_rn(static_cast<double>(y), static_cast<double>(my));
                const double h2 = __dsub_rn(r2_64, __dmul_rn(dy64, dy64));
                if (h2 < 0.0) continue;  // fl(dy^2) > r^2: no pixel of this row is in
                const float sq = sqrtf(static_cast<float>(h2));
                xl = bx + static_cast<int>(ceilf(fmu - sq));
                xr = bx + static_cast<int>(floorf(fmu + sq));
                int a = xl - 2;
                while (a <= xl + 2 && !in_ref(a, y, mx, my, r2_64)) ++a;
                int z = xr + 2;
                while (z >= xr - 2 && !in_ref(z, y, mx, my, r2_64)) --z;
                xl = a;
                xr = z;
                dy = static_cast<float>(dy64);
            }
            xl = max(xl, xmin);
            xr = min(xr, xmax);
            if (xl > xr) continue;
            // e = nk dx^2 + nk dy^2 with the forward's fp32 operations, so a
            // pair's weight is bit-identical to the one summed into W
            const float ey = (dy * nk) * dy;
            if (!decltype(staged_c)::value) {
                for (int x = xl; x <= xr; ++x) {
                    const float dx = static_cast<float>(x) - mx;
                    const float w = ex2(fmaf(dx * nk, dx, ey));
                    float u[CG], v;
                    // (the image base recomputed here: not held across the point loop)
                    pixel_terms<CG>(p, static_cast<size_t>(p.b0 + static_cast<int>(blockIdx.z)) * p.H * p.W,
                                    ch0, nch, x, y, u, v);
                    // t = sum_c c_ic u_c - v with the sum formed by the same
                    // chain as v (pixel_terms): exactly 0 where c_i == out
                    float t = u[0] * cc[0];
#pragma unroll
                    for (int c = 1; c < CG; ++c) t = fmaf(u[c], cc[c], t);
                    t -= v;
                    const float a = w * t;
#pragma unroll
                    for (int c = 0; c < CG; ++c) dcol[c].x = fmaf(w, u[c], dcol[c].x);
                    gx2.x = fmaf(a, dx, gx2.x);
                    gy2.x = fmaf(a, dy, gy2.x);
                }
                continue;
            }
            // pair-aligned span (rx0 is even): pairs xs..xs+2(np-1); the end
            // pixels outside [xl, xr] get weight 0 in the first / last pair
            const int xs = xl - ((xl - rx0) & 1);
            const int np = ((xr - xs) >> 1) + 1;
            const float mf = ((xl - rx0) & 1) ? 0.f : 1.f;
            const float ml = ((xr - rx0) & 1) ? 1.f : 0.f;
            const float xsf = static_cast<float>(xs);
            float2 X = f2(xsf, xsf + 1.f);  // |x| < 2^24: exact
            const float2 ey2 = f2(ey, ey), mmx = f2(-mx, -mx), dy2 = f2(dy, dy);
            const float4* pr = rowp + ((xs - rx0) >> 1);
            GMI_CHECK(y >= ry0 && xs >= rx0 && (y - ry0) * npairs + ((xs - rx0) >> 1) + np <= area &&
                      area * L::kF4 * static_cast<int>(sizeof(float4)) <= kSmemBudget);
            // np >= 1 (xl <= xr): a do-while on the pair pointer; the last-pair
            // test doubles as the loop condition
            const float4* const p0 = pr;
            const float4* const plast = pr + (np - 1);
#pragma unroll 1
            do {
                const bool last = pr == plast;
                float4 q4[L::kF4];
#pragma unroll
                for (int c = 0; c < L::kF4; ++c) q4[c] = pr[c * kPlane];  // immediate offsets
                const float2* q = reinterpret_cast<const float2*>(q4);
                const float2 dx = __fadd2_rn(X, mmx);
                const float2 arg = __ffma2_rn(__fmul2_rn(dx, nk2), dx, ey2);
                float2 w = f2(ex2(arg.x), ex2(arg.y));
                if (pr == p0) w.x *= mf;
                if (last) w.y *= ml;
                // t = sum_c c_ic u_c - v  (= dot / W, engine.cpp:219-221);
                // the sum is formed by the same operation chain as the staged
                // v = sum_c u_c out_c, so t is exactly 0 where the pixel's
                // output equals the point's colour (a sole contributor): the
                // reference's dot is 0 there up to f64 rounding
                float2 t = __fmul2_rn(q[0], f2(cc[0], cc[0]));
#pragma unroll
                for (int c = 1; c < CG; ++c) t = __ffma2_rn(q[c], f2(cc[c], cc[c]), t);
                t = __fadd2_rn(t, q[CG]);
                const float2 a = __fmul2_rn(w, t);
#pragma unroll
                for (int c = 0; c < CG; ++c) dcol[c] = __ffma2_rn(w, q[c], dcol[c]);
                gx2 = __ffma2_rn(a, dx, gx2);
                gy2 = __ffma2_rn(a, dy2, gy2);
                X = __fadd2_rn(X, two);
                if (last) break;
                ++pr;
            } while (true);
        }
        };
#ifndef GMI_BWD_NO_SAFE_SPLIT
        if (!staged) walk(std::false_type{}, std::false_type{});
        else if (__any_sync(__activemask(), unsafe)) walk(std::false_type{}, std::true_type{});
        else walk(std::true_type{}, std::true_type{});
#else
        if (!staged) walk(std::false_type{}, std::false_type{});
        else walk(std::false_type{}, std::true_type{});
#endif
        float gxs = gx2.x + gx2.y, gy = gy2.x + gy2.y;
        float dcs[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) dcs[c] = dcol[c].x + dcol[c].y;
        for (int o = lpp >> 1; o > 0; o >>= 1) {
#pragma unroll
            for (int c = 0; c < CG; ++c) dcs[c] += __shfl_xor_sync(0xffffffffu, dcs[c], o);
            gxs += __shfl_xor_sync(0xffffffffu, gxs, o);
            gy += __shfl_xor_sync(0xffffffffu, gy, o);
        }
        if (!live || sub != 0) continue;
        GMI_CHECK(i >= 0 && i < p.N);
        if (p.gslot != nullptr) {
            // large images: one 32-byte record at the point's slot (the
            // block's points are runs of consecutive slots: full sectors);
            // k_permute_grads moves it to the original index
            st_rec32(p.gslot + (base + s) * 2,
                     make_float4(dcs[0], CG > 1 ? dcs[1] : 0.f, CG > 2 ? dcs[2] : 0.f, CG > 3 ? dcs[3] : 0.f),
                     make_float4(gxs * inv_s2, gy * inv_s2, 0.f, 0.f));
            continue;
        }
        // each point's gradients land at its original index (random against
        // the cell order): as few store transactions as alignment allows
        float* dc = p.d_col + (base + i) * p.C + ch0;
        if (CG == 3 && nch == 3 && p.C == 3 && (reinterpret_cast<uintptr_t>(p.d_col) & 7) == 0) {
            // 12-byte rows: one 8-byte and one 4-byte store (the 8-byte half
            // is the first two channels for an even row, the last two for an
            // odd one)
            if (((base + i) & 1) == 0) {
                *reinterpret_cast<float2*>(dc) = f2(dcs[0], dcs[1]);
                dc[2] = dcs[2];
            } else {
                dc[0] = dcs[0];
                *reinterpret_cast<float2*>(dc + 1) = f2(dcs[1], dcs[2]);
            }
        } else {
            for (int c = 0; c < nch; ++c) dc[c] = dcs[c];
        }
        float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
        const float2 g2 = f2(gxs * inv_s2, gy * inv_s2);
        if ((reinterpret_cast<uintptr_t>(p.d_pos) & 7) == 0) {
            *reinterpret_cast<float2*>(dp) = g2;
        } else {
            dp[0] = g2.x;
            dp[1] = g2.y;
        }
    }
}

// Large images: gradients from slot order to the original point order.
// Thread per point i: its slot from K1's inverse map, one 32-byte record
// read (random, whole sectors), coalesced d_col / d_pos writes — instead of
// the backward scattering partial sectors over a gradient array far larger
// than L2 (read-modify-write traffic in DRAM).
__global__ void __launch_bounds__(256) k_permute_grads(const float4* __restrict__ gslot,
                                                       const int32_t* __restrict__ inv,
                                                       float* __restrict__ d_col,
                                                       float* __restrict__ d_pos, int N, int C,
                                                       size_t total) {
    const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (k >= total) return;
    const size_t base = k - k % N;
    const int s = inv[k];
    GMI_CHECK(s >= 0 && s < N);
    float4 a, b;
    ld_rec32(gslot + (base + s) * 2, a, b);
    const float v[4] = {a.x, a.y, a.z, a.w};
    for (int c = 0; c < C; ++c) d_col[k * C + c] = v[c];
    d_pos[2 * k] = b.x;
    d_pos[2 * k + 1] = b.y;
}

// d_pos = sum over channel groups, in group order (deterministic)
__global__ void k_sum_groups(const float* __restrict__ part, float* __restrict__ d_pos,
                             size_t n2, int groups) {
    const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (k >= n2) return;
    float s = 0.f;
    for (int gi = 0; gi < groups; ++gi) s += part[gi * n2 + k];
    d_pos[k] = s;
}

// Precise mode (cutoff > 6 sigma): one thread per point, f64 weights and
// ratios straight from the reference formulas (engine.cpp:213-231) against the
// f64 normaliser; inclusion by the exact predicate.  A correctness path for
// untruncated / wide-radius calls, not the hot path.
constexpr int kCG64 = 4;
__global__ void k_backward_points_f64(BwdParams p, const double* __restrict__ wsum64,
                                      double inv2s2) {
    const size_t total = static_cast<size_t>(p.B) * p.N;
    const int cg = blockIdx.y, ch0 = cg * kCG64, nch = min(kCG64, p.C - ch0);
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(k / p.N);
        const size_t base = static_cast<size_t>(b) * p.N;
        const double mx = p.sx[k], my = p.sy[k];
        const int i = p.sidx[k] & 0x7fffffff;
        const int s = static_cast<int>(k - base);
        double dcol[kCG64] = {0, 0, 0, 0};
        double gx = 0.0, gy = 0.0;
        double cc[kCG64];
        for (int c = 0; c < kCG64; ++c)
            cc[c] = c < nch ? p.scol[(static_cast<size_t>(b) * p.C + ch0 + c) * p.N + s] : 0.0;
        const int y0 = max(0, static_cast<int>(floor(my - p.r64)) - 1);
        const int y1 = min(p.H - 1, static_cast<int>(ceil(my + p.r64)) + 1);
        const int x0 = max(0, static_cast<int>(floor(mx - p.r64)) - 1);
        const int x1 = min(p.W - 1, static_cast<int>(ceil(mx + p.r64)) + 1);
        for (int y = y0; y <= y1; ++y) {
            for (int x = x0; x <= x1; ++x) {
                const double d2 = d2_ref(x, y, mx, my);
                if (!(d2 <= p.r2_64)) continue;
                const size_t pix = static_cast<size_t>(b) * p.H * p.W + static_cast<size_t>(y) * p.W + x;
                const double W64 = wsum64[pix];
                if (!(W64 > 0.0)) continue;
                const double ratio = exp(-d2 * inv2s2) / W64;
                double dot = 0.0;
                for (int c = 0; c < nch; ++c) {
                    const double u = p.upstream[pix * p.C + ch0 + c];
                    dcol[c] += u * ratio;
                    const double o = p.image64 ? p.image64[pix * p.C + ch0 + c]
                                               : static_cast<double>(p.image[pix * p.C + ch0 + c]);
                    dot += u * (cc[c] - o);
                }
                const double coef = ratio * dot;
                gx += coef * (x - mx);
                gy += coef * (y - my);
            }
        }
        for (int c = 0; c < nch; ++c) p.d_col[(base + i) * p.C + ch0 + c] = static_cast<float>(dcol[c]);
        float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
        dp[0] = static_cast<float>(gx * p.inv_s2);
        dp[1] = static_cast<float>(gy * p.inv_s2);
    }
}

// ---------------------------------------------------------------------------
struct SpecBwdParams {
    const float* upstream;
    const Special* special;
    const int32_t* special_count;
    int special_cap;
    int N, C, W, H;
    int fallback;
    float* d_col;
};

// engine.cpp:200-211: fallback pixels route their upstream to the nearest
// point's colour only (no position gradient).  Sparse inputs route hundreds
// of O(1) upstream values into one point, whose sum may cancel to ~1e-2, so
// it is formed exactly-ordered-independent and added to the point's fp32
// d_col with ONE rounding.  Deterministic by construction: each routed
// value is converted to a 64-bit FIXED-POINT integer on a per-(point,
// channel) scale — 2^(60 - hb - emax), emax the largest exponent among the
// point's routed values and 2^hb > their count, so no sum can overflow — and
// summed with integer atomics, which commute.  Terms below 2^-(60 - hb) of the
// largest one are rounded to that resolution (~1e-15 relative for hundreds of
// terms); a non-finite value switches its (point, channel) to an f64 sum,
// whose inf / NaN result does not depend on the order either.  Four passes
// with fixed grids that read the special count on the device (no host round
// trip, capturable in a CUDA graph), touching only the routed points: reset
// their slots, statistics (count, owner = largest list position, exponent
// maxima), accumulate, then the owner entry adds the point's sum once.
constexpr int kNonFinite = 0x7fffffff;  // emax sentinel: f64 sum instead

__device__ __forceinline__ bool special_route(const SpecBwdParams& p, int si, size_t& pixb,
                                              size_t& pt) {
    const Special sp = p.special[si];
    if (sp.kind != 1 || sp.nearest < 0) return false;
    pixb = static_cast<size_t>(sp.b) * p.H * p.W + sp.pix;
    pt = static_cast<size_t>(sp.b) * p.N + sp.nearest;
    return true;
}

// fixed-point shift of a (point, channel): |v| < 2^(emax+1), count < 2^hb
__device__ __forceinline__ int special_shift(int emax, int count) {
    const int hb = 32 - __clz(count);
    return 60 - hb - emax;
}

__global__ void k_special_zero(SpecBwdParams p, unsigned long long* __restrict__ acc,
                               int* __restrict__ emax, int* __restrict__ own, int* __restrict__ cnt) {
    const int n = min(*p.special_count, p.special_cap);
    for (int si = blockIdx.x * blockDim.x + threadIdx.x; si < n; si += gridDim.x * blockDim.x) {
        size_t pixb, pt;
        if (!special_route(p, si, pixb, pt)) continue;
        own[pt] = -1;
        cnt[pt] = 0;
        for (int c = 0; c < p.C; ++c) {
            acc[pt * p.C + c] = 0ull;
            emax[pt * p.C + c] = INT_MIN;
        }
    }
}

__global__ void k_special_stats(SpecBwdParams p, int* __restrict__ emax, int* __restrict__ own,
                                int* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = min(*p.special_count, p.special_cap);
    for (int si = warp; si < n; si += nwarps) {
        size_t pixb, pt;
        if (!special_route(p, si, pixb, pt)) continue;
        if (lane == 0) {
            atomicMax(own + pt, si);
            atomicAdd(cnt + pt, 1);
        }
        for (int c = lane; c < p.C; c += 32) {
            const float v = p.upstream[pixb * p.C + c];
            if (v != 0.f) atomicMax(emax + pt * p.C + c, is_finite_f(v) ? ilogbf(v) : kNonFinite);
        }
    }
}

__global__ void k_special_accumulate(SpecBwdParams p, unsigned long long* __restrict__ acc,
                                     const int* __restrict__ emax, const int* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = min(*p.special_count, p.special_cap);
    for (int si = warp; si < n; si += nwarps) {
        size_t pixb, pt;
        if (!special_route(p, si, pixb, pt)) continue;
        const int count = cnt[pt];
        for (int c = lane; c < p.C; c += 32) {
            const float v = p.upstream[pixb * p.C + c];
            const int e = emax[pt * p.C + c];
            if (v == 0.f || e == INT_MIN) continue;
            unsigned long long* a = acc + pt * p.C + c;
            if (e == kNonFinite) {
                atomicAdd(reinterpret_cast<double*>(a), static_cast<double>(v));
            } else {
                const long long t = llrint(ldexp(static_cast<double>(v), special_shift(e, count)));
                atomicAdd(a, static_cast<unsigned long long>(t));
            }
        }
    }
}

__global__ void k_special_merge(SpecBwdParams p, const unsigned long long* __restrict__ acc,
                                const int* __restrict__ emax, const int* __restrict__ own,
                                const int* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = min(*p.special_count, p.special_cap);
    for (int si = warp; si < n; si += nwarps) {
        size_t pixb, pt;
        if (!special_route(p, si, pixb, pt) || own[pt] != si) continue;
        for (int c = lane; c < p.C; c += 32) {
            const int e = emax[pt * p.C + c];
            if (e == INT_MIN) continue;  // all routed values were 0
            const unsigned long long a = acc[pt * p.C + c];
            const double sum = e == kNonFinite
                                   ? __longlong_as_double(static_cast<long long>(a))
                                   : ldexp(static_cast<double>(static_cast<long long>(a)),
                                           -special_shift(e, cnt[pt]));
            float* d = p.d_col + pt * p.C + c;
            *d = static_cast<float>(static_cast<double>(*d) + sum);
        }
    }
}

// float4 slots of one staged pixel pair (PairLayout<CG>::kF4)
inline int pair_f4(int cg) { return (cg + 2) / 2; }

template <int CG, int LPP>
void launch_points_lpp(gmi_ctx* ctx, const BwdParams& p, int nblocks, int groups) {
    const int smem = kSmemBudget;
    GMI_SMEM_ONCE(ctx, (k_backward_points<CG, LPP>), smem);
    for (int b0 = 0; b0 < p.B; b0 += 65535) {
        BwdParams q = p;
        q.b0 = b0;
        const unsigned nz = static_cast<unsigned>(std::min(p.B - b0, 65535));
        k_backward_points<CG, LPP><<<dim3(nblocks, groups, nz), kThreads, smem, ctx->stream>>>(q);
        GMI_LAUNCHED(ctx);
    }
}

template <int CG>
void launch_points(gmi_ctx* ctx, const BwdParams& p, int nblocks, int groups) {
    if (p.lpp > 1) launch_points_lpp<CG, 8>(ctx, p, nblocks, groups);
    else launch_points_lpp<CG, 1>(ctx, p, nblocks, groups);
}

}  // namespace

namespace gmi_host {

void launch_backward(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                     float* d_colors, float* d_positions) {
    // C > 4 with the record layout: the wide-channel backward (gmi_wide.cu)
    if (launch_backward_wide(ctx, c, upstream, d_colors, d_positions)) return;
    cudaStream_t st = ctx->stream;
    const int CG = c->C <= 4 ? c->C : 4;
    const int groups = (c->C + CG - 1) / CG;
    // cells per block side so that the staged pixel pairs fit the budget
    const double cell = c->cutoff;
    const double pix_bytes = 8.0 * pair_f4(CG);  // staged bytes per pixel
    const double side_px = std::sqrt(static_cast<double>(kSmemBudget) / pix_bytes);
    int bs = static_cast<int>(std::floor((side_px - 2.0 * cell - 8.0) / cell));
    bs = std::max(1, std::min(bs, kRunMax));
    // CTAs per image: device geometry = a grid of at most grid_cap^2 cells;
    // host geometry = the largest image's grid (smaller images' extra CTAs
    // exit at once)
    int nb_max = 0;
    if (c->geom_h.empty()) {
        const int side = (c->grid_cap + bs - 1) / bs;
        nb_max = side * side;
    } else {
        for (const auto& g : c->geom_h)
            nb_max = std::max(nb_max, ((g.n_cols + bs - 1) / bs) * ((g.n_rows + bs - 1) / bs));
    }
    BwdParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.sx = c->sx;
    p.sy = c->sy;
    p.sidx = c->sidx;
    p.scol = c->scol;
    p.rec = c->rec;
    p.ccol = c->ccol;
    // lanes per point: a point's disk has ~2r+1 rows; split them over lanes
    // once they outnumber what keeps a 256-thread block busy
    p.lpp = c->cutoff >= 6.0 ? 8 : 1;
    p.wsum = c->wsum;
    p.image = c->image;
    p.image64 = c->image64;
    p.upstream = upstream;
    p.B = c->B;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.bs = bs;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.r2f = static_cast<float>(p.r2_64);
    const double nk = -1.4426950408889634 / (2.0 * c->sigma * c->sigma);
    p.nk = static_cast<float>(nk);
    p.inv_s2 = static_cast<float>(1.0 / (c->sigma * c->sigma));
    p.d_col = d_colors;
    const size_t n2 = static_cast<size_t>(c->B) * c->N * 2;
    float* part = nullptr;
    if (groups > 1) {
        part = static_cast<float*>(scratch(ctx, WS_PART, sizeof(float) * n2 * groups));
        p.d_pos = part;
    } else {
        p.d_pos = d_positions;
    }
    if (c->wsum64 != nullptr) {
        const int g64 = (c->C + kCG64 - 1) / kCG64;
        p.d_pos = d_positions;
        if (g64 > 1) {
            part = static_cast<float*>(scratch(ctx, WS_PART, sizeof(float) * n2 * g64));
            p.d_pos = part;
        }
        k_backward_points_f64<<<dim3(4 * ctx->num_sms, g64), 128, 0, st>>>(
            p, c->wsum64, 1.0 / (2.0 * c->sigma * c->sigma));
        GMI_LAUNCHED(ctx);
        if (g64 > 1) {
            k_sum_groups<<<static_cast<unsigned>((n2 + 255) / 256), 256, 0, st>>>(part, d_positions, n2, g64);
            GMI_LAUNCHED(ctx);
        }
        return;
    }
    // large images: gradients in slot order, then one permutation pass
    const bool permute = c->inv != nullptr && c->rec != nullptr && groups == 1;
    if (permute)
        p.gslot = static_cast<float4*>(scratch(ctx, WS_PART, sizeof(float4) * 2 * c->B * c->N));
    if (nb_max > 0) {
        switch (CG) {
            case 1: launch_points<1>(ctx, p, nb_max, groups); break;
            case 2: launch_points<2>(ctx, p, nb_max, groups); break;
            case 3: launch_points<3>(ctx, p, nb_max, groups); break;
            default: launch_points<4>(ctx, p, nb_max, groups); break;
        }
    }
    if (groups > 1) {
        k_sum_groups<<<static_cast<unsigned>((n2 + 255) / 256), 256, 0, st>>>(part, d_positions, n2, groups);
        GMI_LAUNCHED(ctx);
    }
    if (permute) {
        const size_t total = static_cast<size_t>(c->B) * c->N;
        k_permute_grads<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
            p.gslot, c->inv, d_colors, d_positions, c->N, c->C, total);
        GMI_LAUNCHED(ctx);
    }
}

bool slot_grads(int N, int C) {
    const char* e = std::getenv("GMI_SLOT_GRADS_MIN_N");  // read per call (tests flip it)
    const long min_n = e != nullptr ? std::atol(e) : (1L << 20);
    return C <= 4 && N >= min_n;
}

void launch_special_backward(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                             float* d_colors, float* /*d_positions*/) {
    SpecBwdParams p{};
    p.upstream = upstream;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.fallback = c->fallback;
    p.d_col = d_colors;
    // count 0 known on the host (synchronous API): nothing to route
    if (c->special_count == 0 || c->fallback != GMI_FALLBACK_NEAREST) return;
    const size_t npt = static_cast<size_t>(c->B) * c->N;
    // slots touched only for routed points (never cleared wholesale)
    auto* acc = static_cast<unsigned long long*>(
        scratch(ctx, WS_PART, sizeof(unsigned long long) * npt * c->C));
    int* emax = static_cast<int*>(scratch(ctx, WS_RANK, sizeof(int) * npt * c->C));
    int* own = static_cast<int*>(scratch(ctx, WS_TMP, sizeof(int) * 2 * npt));
    int* cnt = own + npt;
    const int grid = 8 * ctx->num_sms;  // many routed pixels in flight (dependent loads)
    k_special_zero<<<grid, 256, 0, ctx->stream>>>(p, acc, emax, own, cnt);
    GMI_LAUNCHED(ctx);
    k_special_stats<<<grid, 256, 0, ctx->stream>>>(p, emax, own, cnt);
    GMI_LAUNCHED(ctx);
    k_special_accumulate<<<grid, 256, 0, ctx->stream>>>(p, acc, emax, cnt);
    GMI_LAUNCHED(ctx);
    k_special_merge<<<grid, 256, 0, ctx->stream>>>(p, acc, emax, own, cnt);
    GMI_LAUNCHED(ctx);
}

}  // namespace gmi_host
