// K4 — backward (engine.cpp:190-234 backward_rows, engine.cpp:238-309).
//
// Point-major and atomic-free: a CTA takes a block of reference cells, stages
// the per-pixel quantities of the pixels those points can reach —
//     u_c = upstream_c / W,   out_c
// (0 on fallback / special pixels) — in shared memory, and every thread owns
// whole points.  For its point a thread walks the exact disk row by row
// (closed ball d^2 <= r^2 as the reference decides it in f64, bin_grid.cpp:98),
// recomputing the Gaussian weight on the SFU instead of storing it, and
// accumulates, in registers,
//     d_col_c += w * u_c                       (= up_c * w/W, engine.cpp:222)
//     d_pos   += w * (sum_c u_c (c_c - out_c)) * (q - mu) / sigma^2
//                                   (= ratio * dot / sigma^2 * (q-mu), :223-230)
// then writes the point's gradients once.  Each point has exactly one owner,
// so the result is bit-deterministic with no atomics and no reduction pass.
//
// K5 — special pixels: NearestPoint fallbacks route upstream to the nearest
// colour (engine.cpp:200-211); pixels whose fp32 normaliser underflowed are
// differentiated in f64 over the reference neighbour set.
#include <algorithm>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

constexpr int kThreads = 256;
constexpr int kCG = 4;                 // channels per pass
constexpr int kSmemBudget = 64 * 1024;  // staged pixel bytes per CTA

struct BwdParams {
    const Geom* geom;
    const int32_t* bins;
    const int32_t* blk_off;  // [B+1] block offsets per image
    const int32_t* blk_dims; // [B][2] (blocks per row, cells per block side)
    const float* sx;
    const float* sy;
    const int32_t* sidx;
    const float* scol;      // [B][C][N]
    const float* wsum;      // [B][H][W]
    const float* image;     // [B][H][W][C]
    const float* upstream;  // [B][H][W][C]
    int B, N, C, W, H;
    int bw, bh;             // cells per block
    double r64, r2_64;
    float r2f, guard, nk, inv_s2;
    float* d_col;           // [B][N][C]
    float* d_pos;           // [B][N][2] or partial [G][B][N][2]
    int groups;
};

__device__ __forceinline__ bool in_ref(int x, int y, float mx, float my,
                                       double r2_64) {
    return d2_ref(static_cast<double>(x), static_cast<double>(y),
                  static_cast<double>(mx), static_cast<double>(my)) <= r2_64;
}

__global__ void __launch_bounds__(kThreads)
k_backward_points(BwdParams p) {
    extern __shared__ float s_pix[];  // [region_h][region_w][2*kCG]
    __shared__ int s_run[65];
    __shared__ float s_red[4][kThreads / 32];
    __shared__ int s_region[5];

    // ---- which image / block ----
    int b = 0;
    {
        int lo = 0, hi = p.B;  // blk_off[b] <= blockIdx.x < blk_off[b+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (p.blk_off[mid] <= static_cast<int>(blockIdx.x)) lo = mid;
            else hi = mid;
        }
        b = lo;
    }
    const Geom g = p.geom[b];
    const int local = blockIdx.x - p.blk_off[b];
    const int nbx = (g.n_cols + p.bw - 1) / p.bw;
    const int cx0 = (local % nbx) * p.bw, cy0 = (local / nbx) * p.bh;
    const int cx1 = min(cx0 + p.bw, g.n_cols), cy1 = min(cy0 + p.bh, g.n_rows);
    const int cg = blockIdx.y, ch0 = cg * kCG, nch = min(kCG, p.C - ch0);
    const int tid = threadIdx.x;
    const size_t base = static_cast<size_t>(b) * p.N;

    // ---- point runs (one per cell row of the block) ----
    const int nrun = cy1 - cy0;
    if (tid <= nrun) {
        // s_run[k] = start of run k; s_run[nrun] = total
        s_run[tid] = 0;
    }
    __syncthreads();
    if (tid == 0) {
        int tot = 0;
        for (int k = 0; k < nrun; ++k) {
            const int64_t r0 = g.bin_off + static_cast<int64_t>(cy0 + k) * g.n_cols;
            s_run[k] = tot;
            tot += p.bins[r0 + cx1] - p.bins[r0 + cx0];
        }
        s_run[nrun] = tot;
    }
    __syncthreads();
    const int total = s_run[nrun];
    if (total == 0) return;
    auto slot_of = [&](int k) -> int {  // concatenated index -> SoA slot
        int r = 0;
        while (s_run[r + 1] <= k) ++r;
        const int64_t r0 = g.bin_off + static_cast<int64_t>(cy0 + r) * g.n_cols;
        return p.bins[r0 + cx0] + (k - s_run[r]);
    };

    // ---- pixel region reached by the block's points ----
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int k = tid; k < total; k += kThreads) {
        const int s = slot_of(k);
        const float x = p.sx[base + s], y = p.sy[base + s];
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
    if ((tid & 31) == 0) {
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
        const int x0 = max(0, static_cast<int>(floorf(mnx - rr)));
        const int y0 = max(0, static_cast<int>(floorf(mny - rr)));
        const int x1 = min(p.W - 1, static_cast<int>(ceilf(mxx + rr)));
        const int y1 = min(p.H - 1, static_cast<int>(ceilf(mxy + rr)));
        s_region[0] = x0;
        s_region[1] = y0;
        s_region[2] = x1;
        s_region[3] = y1;
        const long area = (x1 >= x0 && y1 >= y0)
                              ? static_cast<long>(x1 - x0 + 1) * (y1 - y0 + 1)
                              : 0;
        s_region[4] = (area * (2 * kCG) * 4 <= kSmemBudget) ? 1 : 0;
    }
    __syncthreads();
    const int rx0 = s_region[0], ry0 = s_region[1], rx1 = s_region[2], ry1 = s_region[3];
    if (rx1 < rx0 || ry1 < ry0) {
        // no pixel in the frame is reachable: all gradients are zero
        for (int k = tid; k < total; k += kThreads) {
            const int i = p.sidx[base + slot_of(k)];
            for (int c = 0; c < nch; ++c) p.d_col[(base + i) * p.C + ch0 + c] = 0.f;
            float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
            dp[0] = 0.f;
            dp[1] = 0.f;
        }
        return;
    }
    const bool staged = s_region[4] != 0;
    const int rw = rx1 - rx0 + 1;
    const size_t img_base = static_cast<size_t>(b) * p.H * p.W;

    // per-pixel quantities for this channel group (engine.cpp:213-222):
    // q[c] = upstream_c / W and q[kCG + c] = out_c (0 on special pixels).
    // Staging out (not sum_c u_c out_c) lets the point loop form c_ic - out_c
    // exactly (Sterbenz) before weighting, which keeps d_positions accurate
    // where the reference's value is a cancellation to ~0 (isolated points).
    auto pixel_q = [&](int x, int y, float* q) {
        const size_t pix = img_base + static_cast<size_t>(y) * p.W + x;
        const float wv = p.wsum[pix];
#pragma unroll
        for (int c = 0; c < 2 * kCG; ++c) q[c] = 0.f;
        if (wv > 0.f) {
            const float inv = 1.0f / wv;
            const float* up = p.upstream + pix * p.C + ch0;
            const float* out = p.image + pix * p.C + ch0;
#pragma unroll
            for (int c = 0; c < kCG; ++c) {
                if (c < nch) {
                    q[c] = up[c] * inv;
                    q[kCG + c] = out[c];
                }
            }
        }
    };
    if (staged) {
        const int area = rw * (ry1 - ry0 + 1);
        for (int k = tid; k < area; k += kThreads) {
            float q[2 * kCG];
            pixel_q(rx0 + k % rw, ry0 + k / rw, q);
#pragma unroll
            for (int c = 0; c < 2 * kCG; ++c) s_pix[k * (2 * kCG) + c] = q[c];
        }
        __syncthreads();
    }

    // ---- per point ----
    for (int k = tid; k < total; k += kThreads) {
        const int s = slot_of(k);
        const float mx = p.sx[base + s], my = p.sy[base + s];
        const int i = p.sidx[base + s];
        float cc[kCG];
#pragma unroll
        for (int c = 0; c < kCG; ++c)
            cc[c] = c < nch ? p.scol[(static_cast<size_t>(b) * p.C + ch0 + c) * p.N + s] : 0.f;
        float dcol[kCG];
#pragma unroll
        for (int c = 0; c < kCG; ++c) dcol[c] = 0.f;
        float gx = 0.f, gy = 0.f;
        const float tx = truncf(mx);
        const float fmu = mx - tx;  // exact
        const int bx = static_cast<int>(tx);
        const int ya = max(ry0, static_cast<int>(floorf(my - static_cast<float>(p.r64))) - 1);
        const int yb = min(ry1, static_cast<int>(ceilf(my + static_cast<float>(p.r64))) + 1);
        for (int y = ya; y <= yb; ++y) {
            const double dy64 = __dsub_rn(static_cast<double>(y), static_cast<double>(my));
            const double h2 = __dsub_rn(p.r2_64, __dmul_rn(dy64, dy64));
            const float h2f = static_cast<float>(h2);
            if (h2f < -p.guard) continue;  // row entirely outside the ball
            const float sq = sqrtf(fmaxf(h2f, 0.f));
            const float al = fmu - sq, ar = fmu + sq;
            int xl = bx + static_cast<int>(ceilf(al));
            int xr = bx + static_cast<int>(floorf(ar));
            const float nl = rintf(al), nr = rintf(ar);
            const float el = fmaf(nl - fmu, nl - fmu, -h2f);
            const float er = fmaf(nr - fmu, nr - fmu, -h2f);
            if (fabsf(el) <= p.guard || fabsf(er) <= p.guard) {
                // boundary pixel within the guard band: decide in f64
                int a = xl - 2;
                while (a <= xl + 2 && !in_ref(a, y, mx, my, p.r2_64)) ++a;
                int z = xr + 2;
                while (z >= xr - 2 && !in_ref(z, y, mx, my, p.r2_64)) --z;
                xl = a;
                xr = z;
            }
            xl = max(xl, rx0);
            xr = min(xr, rx1);
            if (xl > xr) continue;
            const float dy = static_cast<float>(dy64);
            const float dy2 = dy * dy;
            float gyr = 0.f;
            float dx = static_cast<float>(xl - bx) - fmu;
            for (int x = xl; x <= xr; ++x, dx += 1.0f) {
                const float d2 = fmaf(dx, dx, dy2);
                const float w = ex2(d2 * p.nk);
                float q[2 * kCG];
                if (staged) {
                    const float* sp = s_pix + ((y - ry0) * rw + (x - rx0)) * (2 * kCG);
#pragma unroll
                    for (int c = 0; c < 2 * kCG; ++c) q[c] = sp[c];
                } else {
                    pixel_q(x, y, q);
                }
                // dot/W = sum_c u_c (c_ic - out_c)   (engine.cpp:219-221)
                float t = 0.f;
#pragma unroll
                for (int c = 0; c < kCG; ++c) t = fmaf(q[c], cc[c] - q[kCG + c], t);
                const float a = w * t;
#pragma unroll
                for (int c = 0; c < kCG; ++c) dcol[c] = fmaf(w, q[c], dcol[c]);
                gx = fmaf(a, dx, gx);
                gyr += a;
            }
            gy = fmaf(gyr, dy, gy);
        }
        for (int c = 0; c < nch; ++c) p.d_col[(base + i) * p.C + ch0 + c] = dcol[c];
        float* dp = p.d_pos + (static_cast<size_t>(cg) * p.B * p.N + base + i) * 2;
        dp[0] = gx * p.inv_s2;
        dp[1] = gy * p.inv_s2;
    }
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

// ---------------------------------------------------------------------------
struct SpecBwdParams {
    const Geom* geom;
    const int32_t* bins;
    const float* sx;
    const float* sy;
    const int32_t* sidx;
    const float* scol;
    const float* image;
    const float* upstream;
    const Special* special;
    const int32_t* special_count;
    int special_cap;
    int N, C, W, H;
    double r64, r2_64, sigma;
    int fallback;
    float* d_col;
    float* d_pos;
};

__global__ void k_special_backward(SpecBwdParams p) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = min(*p.special_count, p.special_cap);
    for (int si = warp; si < n; si += nwarps) {
        const Special sp = p.special[si];
        const size_t pixb = static_cast<size_t>(sp.b) * p.H * p.W + sp.pix;
        const float* up = p.upstream + pixb * p.C;
        const size_t base = static_cast<size_t>(sp.b) * p.N;
        if (sp.kind == 1) {
            // engine.cpp:200-211: colour-only routing to the nearest point
            if (p.fallback == GMI_FALLBACK_NEAREST && sp.nearest >= 0) {
                for (int c = lane; c < p.C; c += 32)
                    atomicAdd(p.d_col + (base + sp.nearest) * p.C + c, up[c]);
            }
            continue;
        }
        if (sp.kind != 2) continue;
        // f64 differentiation over the reference neighbour set
        const Geom g = p.geom[sp.b];
        const int pr = sp.pix / p.W, pc = sp.pix % p.W;
        const double qx = pc, qy = pr;
        const double inv2s2 = 1.0 / (2.0 * p.sigma * p.sigma);
        const double inv_s2 = 1.0 / (p.sigma * p.sigma);
        const int cx0 = cell_of(qx - p.r64, g.ox, g.cell, g.n_cols);
        const int cx1 = cell_of(qx + p.r64, g.ox, g.cell, g.n_cols);
        const int cy0 = cell_of(qy - p.r64, g.oy, g.cell, g.n_rows);
        const int cy1 = cell_of(qy + p.r64, g.oy, g.cell, g.n_rows);
        double W64 = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int cy = cy0; cy <= cy1; ++cy) {
                const int64_t r0 = g.bin_off + static_cast<int64_t>(cy) * g.n_cols;
                const int s = p.bins[r0 + cx0], e = p.bins[r0 + cx1 + 1];
                for (int k = s + lane; k < e; k += 32) {
                    const double mx = p.sx[base + k], my = p.sy[base + k];
                    const double d2 = d2_ref(qx, qy, mx, my);
                    if (!(d2 <= p.r2_64)) continue;
                    const double w = exp(-d2 * inv2s2);
                    if (pass == 0) {
                        W64 += w;
                        continue;
                    }
                    const double ratio = w / W64;
                    const int i = p.sidx[base + k];
                    double dot = 0.0;
                    for (int c = 0; c < p.C; ++c) {
                        const double u = up[c];
                        atomicAdd(p.d_col + (base + i) * p.C + c, static_cast<float>(u * ratio));
                        dot += u * (static_cast<double>(
                                        p.scol[(static_cast<size_t>(sp.b) * p.C + c) * p.N + k]) -
                                    static_cast<double>(p.image[pixb * p.C + c]));
                    }
                    const double coef = ratio * dot * inv_s2;
                    atomicAdd(p.d_pos + (base + i) * 2, static_cast<float>(coef * (qx - mx)));
                    atomicAdd(p.d_pos + (base + i) * 2 + 1, static_cast<float>(coef * (qy - my)));
                }
            }
            if (pass == 0)
                for (int o = 16; o > 0; o >>= 1) W64 += __shfl_xor_sync(0xffffffffu, W64, o);
        }
    }
}

}  // namespace

namespace gmi_host {

void launch_backward(gmi_ctx* ctx, const gmi_cache* c, const float* upstream,
                     float* d_colors, float* d_positions) {
    cudaStream_t st = ctx->stream;
    const int groups = (c->C + kCG - 1) / kCG;
    // cells per block side so that the staged pixel region fits the budget
    const double cell = c->cutoff;
    const double side_px = std::sqrt(static_cast<double>(kSmemBudget) / ((2 * kCG) * 4.0));
    int bs = static_cast<int>(std::floor((side_px - 2.0 * cell - 6.0) / cell));
    bs = std::max(1, std::min(bs, 64));
    std::vector<int32_t> off(c->B + 1, 0);
    for (int b = 0; b < c->B; ++b) {
        const auto& g = c->geom_h[b];
        const int nb = ((g.n_cols + bs - 1) / bs) * ((g.n_rows + bs - 1) / bs);
        off[b + 1] = off[b] + nb;
    }
    int32_t* d_off = static_cast<int32_t*>(dalloc(ctx, sizeof(int32_t) * (c->B + 1)));
    GMI_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * (c->B + 1),
                             cudaMemcpyHostToDevice, st));
    BwdParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.blk_off = d_off;
    p.sx = c->sx;
    p.sy = c->sy;
    p.sidx = c->sidx;
    p.scol = c->scol;
    p.wsum = c->wsum;
    p.image = c->image;
    p.upstream = upstream;
    p.B = c->B;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.bw = bs;
    p.bh = bs;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.r2f = static_cast<float>(p.r2_64);
    p.guard = 4e-6f * p.r2f + 1e-30f;
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    p.inv_s2 = static_cast<float>(1.0 / (c->sigma * c->sigma));
    p.d_col = d_colors;
    p.groups = groups;
    float* part = nullptr;
    const size_t n2 = static_cast<size_t>(c->B) * c->N * 2;
    if (groups > 1) {
        part = static_cast<float*>(dalloc(ctx, sizeof(float) * n2 * groups));
        p.d_pos = part;
    } else {
        p.d_pos = d_positions;
    }
    GMI_CUDA(cudaFuncSetAttribute(k_backward_points,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    if (off[c->B] > 0) {
        k_backward_points<<<dim3(off[c->B], groups), kThreads, kSmemBudget, st>>>(p);
        GMI_LAUNCHED(ctx);
    }
    if (groups > 1) {
        k_sum_groups<<<static_cast<unsigned>((n2 + 255) / 256), 256, 0, st>>>(part, d_positions, n2, groups);
        GMI_LAUNCHED(ctx);
        dfree(ctx, part);
    }
    dfree(ctx, d_off);
}

void launch_special_backward(gmi_ctx* ctx, const gmi_cache* c,
                             const float* upstream, float* d_colors,
                             float* d_positions) {
    SpecBwdParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.sx = c->sx;
    p.sy = c->sy;
    p.sidx = c->sidx;
    p.scol = c->scol;
    p.image = c->image;
    p.upstream = upstream;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.sigma = c->sigma;
    p.fallback = c->fallback;
    p.d_col = d_colors;
    p.d_pos = d_positions;
    k_special_backward<<<2 * ctx->num_sms, 256, 0, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

}  // namespace gmi_host
