// K2 fast path — forward gather (engine.cpp:44-103 forward_rows +
// query_radius bin_grid.cpp:84-105 + gaussian_weight core.cpp:49-53) for the
// fp32 weight mode (cutoff <= 6 sigma) with C <= 4 channels.
//
// CTA = 64x16 output pixels of one image, 8 warps; warp w owns the row pair
// (y0+2w, y0+2w+1), lane l the columns (x0+2l, x0+2l+1): 2x2 pixels per thread
// whose normaliser W and numerators live in f32x2 registers.
//
//  stage  The candidate points of the tile (reference cells overlapping the
//         tile grown by r) come from the bin-ordered SoA.  Inside a cell row
//         the SoA is sorted by fine x-column (K1), so each cell row is an
//         x-sorted run.  The runs are merged COLUMN-MAJOR into shared memory
//         — position = column start + earlier rows in that column + rank —
//         with deterministic ranks (__match_any_sync), no sort and no atomics.
//  band   Each warp compacts (ballot) the candidates of its row pair's band
//         |y - mu_y| <= r into an x-sorted index list.
//  window Each lane's candidates are then ONE contiguous range of that list:
//         mu_x in [x - r, x + 1 + r], found from the column starts and the
//         warp's ballot words — no per-lane search.
//  gather Per candidate, 4 pixels with f32x2 ops: d^2, in-ball test (fp32 is
//         exact for points K1 did not flag, see gmi_common.cuh), 4 MUFU.EX2,
//         W and C numerators.  Flagged (boundary-ambiguous) points take the f64
//         predicate in a separate warp-uniform pass.
//  store  out = num/W with one Newton step, W kept for the backward; pixels
//         with W == 0 go to the fallback list (K3).
#include <algorithm>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

constexpr int kTW = 64, kTH = 16;
constexpr int kNW = kTH / 2;       // warps (row pairs)
constexpr int kNT = kNW * 32;      // threads
constexpr int kCap = 1024;         // staged candidates per chunk
constexpr int kRsMax = 32;         // cell-row runs per chunk
constexpr int kNqMax = 256;        // fine x-columns across the tile's region
constexpr int kChunks = kCap / 32;

template <int CC>
struct SmemGather {
    float4 A[kCap];                        // mu_x, mu_y, c0, c1
    float2 Bc[CC > 2 ? kCap : 1];          // c2, c3
    uint8_t flag[kCap];                    // boundary-ambiguous point
    uint16_t cnt[kRsMax][kNqMax];          // per (run, column) count -> offset
    int colstart[kNqMax + 1];
    uint16_t srank[kCap];
    uint16_t list[kNW][kCap];
    uint32_t bal[kNW][kChunks + 1];
    uint16_t balpre[kNW][kChunks + 1];
    int run_beg[kRsMax + 1];
    int run_g[kRsMax];
    int scan_w[kNT / 32];
    int n_runs, cur_cy, cur_off, done, any_flag;
    int cx0, cx1, cy1, pre;
};

struct GatherParams {
    const Geom* geom;
    const int32_t* bins;
    const float* sx;
    const float* sy;
    const int32_t* sidx;
    const float* scol;  // [B][C][N]
    int N, C, W, H;
    double r64, r2_64;
    float rf, r2f, nk;
    float* image;
    float* wsum;
    int32_t* counts;
    Special* special;
    int32_t* special_count;
    int special_cap;
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

template <int CC, bool kCount>
__global__ void __launch_bounds__(kNT)
k_gather(GatherParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemGather<CC>& S = *reinterpret_cast<SmemGather<CC>*>(smem_raw);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // channel group of this CTA (C > 4: grid.z groups, weights recomputed per
    // group; group 0 owns W, counts and the fallback list)
    const int ch0 = blockIdx.z * CC, nch = min(CC, p.C - ch0);
    const int tiles_y = (p.H + kTH - 1) / kTH;
    const int b = blockIdx.y / tiles_y;
    const int y0 = (blockIdx.y % tiles_y) * kTH;
    const int x0 = blockIdx.x * kTW;
    const Geom g = p.geom[b];
    const size_t base = static_cast<size_t>(b) * p.N;
    const unsigned lt = (1u << lane) - 1u;

    // tile region and its reference cells (bin_grid.cpp:88-91 for the tile)
    const double xlo = static_cast<double>(x0) - p.r64;
    const double xhi = static_cast<double>(x0 + kTW - 1) + p.r64;
    const double ylo = static_cast<double>(y0) - p.r64;
    const double yhi = static_cast<double>(y0 + kTH - 1) + p.r64;
    // fp32 region bounds, padded outward (monotone filters stay supersets)
    const float epsx = 2e-3f + 1e-6f * fabsf(static_cast<float>(xhi));
    const float epsy = 2e-3f + 1e-6f * fabsf(static_cast<float>(yhi));
    const float fxlo = static_cast<float>(xlo) - epsx, fxhi = static_cast<float>(xhi) + epsx;
    const float fylo = static_cast<float>(ylo) - epsy, fyhi = static_cast<float>(yhi) + epsy;
    const int q_lo = fine_col(fxlo, g.qx0, g.qscale);
    const int nq = min(kNqMax, fine_col(fxhi, g.qx0, g.qscale) - q_lo + 1);

    // this thread's 2x2 pixels
    const int ya = y0 + 2 * warp, xa = x0 + 2 * lane;
    const float2 X = f2(static_cast<float>(xa), static_cast<float>(xa + 1));
    const float2 Y = f2(static_cast<float>(ya), static_cast<float>(ya + 1));
    const float2 nk2 = f2(p.nk, p.nk);
    float2 Wa = f2(0.f, 0.f), Wb = f2(0.f, 0.f);  // rows ya, ya+1; (xa, xa+1)
    float2 Na[CC], Nb[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) {
        Na[c] = f2(0.f, 0.f);
        Nb[c] = f2(0.f, 0.f);
    }
    int cnt00 = 0, cnt01 = 0, cnt10 = 0, cnt11 = 0;
    // lane window in fine columns: mu_x in [xa - r, xa + 1 + r]
    const float wlo = X.x - p.rf - epsx, whi = X.y + p.rf + epsx;
    const int wq0 = max(0, fine_col(wlo, g.qx0, g.qscale) - q_lo);
    const int wq1 = min(nq - 1, fine_col(whi, g.qx0, g.qscale) - q_lo);
    const float band_lo = Y.x - p.rf - epsy, band_hi = Y.y + p.rf + epsy;

    if (warp == 0) {
        // the f64 cell rectangle (four lanes in parallel)
        int cv = 0;
        if (lane == 0) cv = cell_of(xlo, g.ox, g.cell, g.n_cols);
        if (lane == 1) cv = cell_of(xhi, g.ox, g.cell, g.n_cols);
        if (lane == 2) cv = cell_of(ylo, g.oy, g.cell, g.n_rows);
        if (lane == 3) cv = cell_of(yhi, g.oy, g.cell, g.n_rows);
        const int cx0 = __shfl_sync(0xffffffffu, cv, 0), cx1 = __shfl_sync(0xffffffffu, cv, 1);
        const int cy0 = __shfl_sync(0xffffffffu, cv, 2), cy1 = __shfl_sync(0xffffffffu, cv, 3);
        // common case: <= 32 cell rows and <= kCap candidates -> one chunk,
        // runs loaded by one lane each (no serial chain of dependent loads)
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
        }
    }
    __syncthreads();
    while (true) {
        // ---- next chunk of runs (<= kRsMax runs, <= kCap candidates) ----
        if (tid == 0 && S.pre) {
            S.pre = 0;  // the single chunk was prepared above
        } else if (tid == 0) {
            const int cx0 = S.cx0, cx1 = S.cx1, cy1 = S.cy1;
            int n = 0, tot = 0, cy = S.cur_cy, off = S.cur_off;
            while (cy <= cy1 && n < kRsMax && tot < kCap) {
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cy) * g.n_cols;
                const int gs = p.bins[r0 + cx0] + off, ge = p.bins[r0 + cx1 + 1];
                if (ge <= gs) {
                    ++cy;
                    off = 0;
                    continue;
                }
                const int take = min(ge - gs, kCap - tot);
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
        __syncthreads();
        const int n_runs = S.n_runs;
        if (n_runs == 0) break;
        for (int k = tid; k < n_runs * kNqMax; k += kNT) (&S.cnt[0][0])[k] = 0;
        if (tid == 0) S.any_flag = 0;
        __syncthreads();

        // ---- A: deterministic rank of each kept candidate in its (run, column)
        for (int rs = warp; rs < n_runs; rs += kNW) {
            const int gs = S.run_g[rs], rb = S.run_beg[rs], len = S.run_beg[rs + 1] - rb;
            for (int j0 = 0; j0 < len; j0 += 32) {
                const int j = j0 + lane;
                float mx = 0.f, my = 0.f;
                bool keep = false;
                int q = 0;
                if (j < len) {
                    mx = p.sx[base + gs + j];
                    my = p.sy[base + gs + j];
                    keep = mx >= fxlo && mx <= fxhi && my >= fylo && my <= fyhi;
                    q = fine_col(mx, g.qx0, g.qscale) - q_lo;
                    keep = keep && q >= 0 && q < nq;
                }
                const int key = keep ? q : (0x10000 + lane);
                const unsigned peers = __match_any_sync(0xffffffffu, key);
                const int leader = __ffs(peers) - 1;
                int bcnt = 0;
                if (keep && lane == leader) {
                    bcnt = S.cnt[rs][q];
                    S.cnt[rs][q] = static_cast<uint16_t>(bcnt + __popc(peers));
                }
                bcnt = __shfl_sync(0xffffffffu, bcnt, leader);
                if (j < len)
                    S.srank[rb + j] = keep ? static_cast<uint16_t>(bcnt + __popc(peers & lt)) : 0xFFFFu;
                __syncwarp();
            }
        }
        __syncthreads();

        // ---- B: column starts and per-column run offsets ----
        {
            int colsum = 0;
            if (tid < nq) {
                for (int rs = 0; rs < n_runs; ++rs) {
                    const int v = S.cnt[rs][tid];
                    S.cnt[rs][tid] = static_cast<uint16_t>(colsum);
                    colsum += v;
                }
            }
            int incl = colsum;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) S.scan_w[warp] = incl;
            __syncthreads();
            int wbase = 0;
            for (int w = 0; w < warp; ++w) wbase += S.scan_w[w];
            if (tid < nq) S.colstart[tid] = wbase + incl - colsum;
            if (tid == kNT - 1) S.colstart[nq] = wbase + incl;
        }
        __syncthreads();

        // ---- C: scatter the records column-major ----
        for (int rs = warp; rs < n_runs; rs += kNW) {
            const int gs = S.run_g[rs], rb = S.run_beg[rs], len = S.run_beg[rs + 1] - rb;
            for (int j = lane; j < len; j += 32) {
                const int r = S.srank[rb + j];
                if (r == 0xFFFF) continue;
                const size_t slot = base + gs + j;
                const float mx = p.sx[slot], my = p.sy[slot];
                const int q = fine_col(mx, g.qx0, g.qscale) - q_lo;
                const int dst = S.colstart[q] + S.cnt[rs][q] + r;
                float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int ch = 0; ch < CC; ++ch)
                    if (ch < nch)
                        c[ch] = p.scol[(static_cast<size_t>(b) * p.C + ch0 + ch) * p.N + gs + j];
                S.A[dst] = make_float4(mx, my, c[0], c[1]);
                if (CC > 2) S.Bc[dst] = f2(c[2], c[3]);
                const uint8_t fl = static_cast<uint8_t>(static_cast<uint32_t>(p.sidx[slot]) >> 31);
                S.flag[dst] = fl;
                if (fl) S.any_flag = 1;
            }
        }
        __syncthreads();
        const bool any_flag = S.any_flag != 0;

        // ---- D: per-warp band list and per-lane windows ----
        const int T = S.colstart[nq];
        int nf = 0;
        for (int k0 = 0; k0 < T; k0 += 32) {
            const int k = k0 + lane;
            bool fast = false;
            if (k < T) {
                const float my = S.A[k].y;
                fast = my >= band_lo && my <= band_hi && !S.flag[k];
            }
            const unsigned bf = __ballot_sync(0xffffffffu, fast);
            if (fast) S.list[warp][nf + __popc(bf & lt)] = static_cast<uint16_t>(k);
            if (lane == 0) {
                S.bal[warp][k0 >> 5] = bf;
                S.balpre[warp][k0 >> 5] = static_cast<uint16_t>(nf);
            }
            nf += __popc(bf);
        }
        if (lane == 0) {
            S.bal[warp][(T + 31) >> 5] = 0u;
            S.balpre[warp][(T + 31) >> 5] = static_cast<uint16_t>(nf);
        }
        __syncwarp();
        auto prefix_kept = [&](int pos) -> int {
            const int c = pos >> 5, bit = pos & 31;
            return S.balpre[warp][c] + __popc(S.bal[warp][c] & ((1u << bit) - 1u));
        };
        int ts = 0, te = 0;
        if (wq0 <= wq1) {
            ts = prefix_kept(S.colstart[wq0]);
            te = prefix_kept(S.colstart[wq1 + 1]);
        }

        // ---- gather: 4 pixels per candidate, f32x2 ----
        const uint16_t* lst = S.list[warp];
#pragma unroll 2
        for (int t = ts; t < te; ++t) {
            const int kc = lst[t];
            const float4 a = S.A[kc];
            const float2 bcur = CC > 2 ? S.Bc[kc] : f2(0.f, 0.f);
            const float2 dx = __fadd2_rn(X, f2(-a.x, -a.x));
            const float2 dy = __fadd2_rn(Y, f2(-a.y, -a.y));
            const float2 sxx = __fmul2_rn(dx, dx);
            const float2 syy = __fmul2_rn(dy, dy);
            const float2 da = __fadd2_rn(sxx, f2(syy.x, syy.x));
            const float2 db = __fadd2_rn(sxx, f2(syy.y, syy.y));
            const float2 aa = __fmul2_rn(da, nk2);
            const float2 ab = __fmul2_rn(db, nk2);
            const bool i00 = da.x <= p.r2f, i01 = da.y <= p.r2f;
            const bool i10 = db.x <= p.r2f, i11 = db.y <= p.r2f;
            const float2 wa = f2(i00 ? ex2(aa.x) : 0.f, i01 ? ex2(aa.y) : 0.f);
            const float2 wb = f2(i10 ? ex2(ab.x) : 0.f, i11 ? ex2(ab.y) : 0.f);
            Wa = __fadd2_rn(Wa, wa);
            Wb = __fadd2_rn(Wb, wb);
            Na[0] = __ffma2_rn(wa, f2(a.z, a.z), Na[0]);
            Nb[0] = __ffma2_rn(wb, f2(a.z, a.z), Nb[0]);
            if (CC > 1) {
                Na[1] = __ffma2_rn(wa, f2(a.w, a.w), Na[1]);
                Nb[1] = __ffma2_rn(wb, f2(a.w, a.w), Nb[1]);
            }
            if (CC > 2) {
                const float2 bc = bcur;
                Na[2] = __ffma2_rn(wa, f2(bc.x, bc.x), Na[2]);
                Nb[2] = __ffma2_rn(wb, f2(bc.x, bc.x), Nb[2]);
                if (CC > 3) {
                    Na[3] = __ffma2_rn(wa, f2(bc.y, bc.y), Na[3]);
                    Nb[3] = __ffma2_rn(wb, f2(bc.y, bc.y), Nb[3]);
                }
            }
            if (kCount) {
                cnt00 += i00;
                cnt01 += i01;
                cnt10 += i10;
                cnt11 += i11;
            }
        }

        // ---- boundary-ambiguous points: f64 predicate (rare) ----
        for (int k0 = 0; any_flag && k0 < T; k0 += 32) {
            const int k = k0 + lane;
            bool ex = false;
            if (k < T) {
                const float my = S.A[k].y;
                ex = S.flag[k] && my >= band_lo && my <= band_hi;
            }
            unsigned bx = __ballot_sync(0xffffffffu, ex);
            while (bx) {
                const int kk = k0 + __ffs(bx) - 1;
                bx &= bx - 1u;
                const float4 a = S.A[kk];
                float cc[4] = {a.z, a.w, 0.f, 0.f};
                if (CC > 2) {
                    const float2 bc = S.Bc[kk];
                    cc[2] = bc.x;
                    cc[3] = bc.y;
                }
#pragma unroll
                for (int py = 0; py < 2; ++py) {
#pragma unroll
                    for (int px = 0; px < 2; ++px) {
                        const int qx = xa + px, qy = ya + py;
                        if (d2_ref(qx, qy, a.x, a.y) > p.r2_64) continue;
                        const float ddx = static_cast<float>(qx) - a.x;
                        const float ddy = static_cast<float>(qy) - a.y;
                        const float w = ex2(fmaf(ddx, ddx, ddy * ddy) * p.nk);
                        float2& Wr = py ? Wb : Wa;
                        float2* Nr = py ? Nb : Na;
                        if (px) Wr.y += w; else Wr.x += w;
#pragma unroll
                        for (int c = 0; c < CC; ++c) {
                            if (px) Nr[c].y = fmaf(w, cc[c], Nr[c].y);
                            else Nr[c].x = fmaf(w, cc[c], Nr[c].x);
                        }
                        if (kCount) {
                            if (py) { if (px) ++cnt11; else ++cnt10; }
                            else { if (px) ++cnt01; else ++cnt00; }
                        }
                    }
                }
            }
        }
        const bool last = S.done;
        __syncthreads();
        if (last) break;
    }

    // ---- fused normalisation + store (engine.cpp:74-100) ----
#pragma unroll
    for (int py = 0; py < 2; ++py) {
#pragma unroll
        for (int px = 0; px < 2; ++px) {
            const int qx = xa + px, qy = ya + py;
            if (qx >= p.W || qy >= p.H) continue;
            const float w = py ? (px ? Wb.y : Wb.x) : (px ? Wa.y : Wa.x);
            const size_t bp = (static_cast<size_t>(b) * p.H + qy) * p.W + qx;
            float* out = p.image + bp * p.C + ch0;
            if (w > 0.f) {
                const float inv = 1.0f / w;
#pragma unroll
                for (int c = 0; c < CC; ++c) {
                    if (c >= nch) continue;
                    const float num = py ? (px ? Nb[c].y : Nb[c].x) : (px ? Na[c].y : Na[c].x);
                    const float q0 = num * inv;
                    out[c] = fmaf(fmaf(-q0, w, num), inv, q0);
                }
                if (blockIdx.z == 0) {
                    p.wsum[bp] = w;
                    if (kCount) p.counts[bp] = py ? (px ? cnt11 : cnt10) : (px ? cnt01 : cnt00);
                }
            } else if (blockIdx.z == 0) {
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

template <int CC, bool kCount>
void launch_cc(gmi_ctx* ctx, const GatherParams& p, dim3 grid) {
    const int smem = static_cast<int>(sizeof(SmemGather<CC>));
    GMI_CUDA(cudaFuncSetAttribute(k_gather<CC, kCount>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_gather<CC, kCount><<<grid, kNT, smem, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

}  // namespace

namespace gmi_host {

// Returns false when the configuration needs the generic gather
// (f64 weight mode, C > 4, or a radius whose fine-column window exceeds the
// staging tables).
bool launch_gather_fast(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts) {
    if (c->wsum64 != nullptr) return false;
    const double need_cols = 2.0 * (kTW - 1 + 2.0 * c->cutoff + 0.05) + 4.0;
    if (need_cols > kNqMax) return false;
    GatherParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.sx = c->sx;
    p.sy = c->sy;
    p.sidx = c->sidx;
    p.scol = c->scol;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.rf = static_cast<float>(c->cutoff);
    p.r2f = static_cast<float>(p.r2_64);
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    p.image = image;
    p.wsum = c->wsum;
    p.counts = counts;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    const int cc = c->C <= 4 ? c->C : 4;
    const dim3 grid((c->W + kTW - 1) / kTW, ((c->H + kTH - 1) / kTH) * c->B, (c->C + cc - 1) / cc);
    GMI_CUDA(cudaMemsetAsync(c->special_count_d, 0, sizeof(int32_t), ctx->stream));
    const bool cnt = counts != nullptr;
    switch (cc) {
        case 1: cnt ? launch_cc<1, true>(ctx, p, grid) : launch_cc<1, false>(ctx, p, grid); break;
        case 2: cnt ? launch_cc<2, true>(ctx, p, grid) : launch_cc<2, false>(ctx, p, grid); break;
        case 3: cnt ? launch_cc<3, true>(ctx, p, grid) : launch_cc<3, false>(ctx, p, grid); break;
        default: cnt ? launch_cc<4, true>(ctx, p, grid) : launch_cc<4, false>(ctx, p, grid); break;
    }
    return true;
}

}  // namespace gmi_host
