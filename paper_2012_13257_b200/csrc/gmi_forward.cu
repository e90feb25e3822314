// K2 — forward gather (engine.cpp:44-103 forward_rows + query_radius +
// gaussian_weight) and K3 — special pixels (empty neighbourhood / weight
// underflow: engine.cpp:74-92, nearest_point bin_grid.cpp:114-164).
//
// One CTA per TWxTH output tile per image (per channel group).  The CTA
// stages the tile's candidate points (the reference cells overlapping the
// tile grown by the cutoff, engine.cpp:115 / bin_grid.cpp:88-91) from the
// bin-ordered SoA into shared memory, and every thread owns pixels whose
// numerator and normaliser live in registers.  Weights are exp2 on the SFU;
// normalisation and the store are fused.
//
// Inclusion is the reference's closed ball d^2 <= r^2 evaluated in f64
// (bin_grid.cpp:87,98).  The fp32 d^2 used in the loop differs from the
// reference's f64 value by < 1e-6 r^2; whenever |d2 - r2| is inside the
// guard band g the pair is re-decided with the exact f64 predicate, so the
// neighbour sets — and the per-pixel counts (pixel_start deltas) — equal the
// reference's bit for bit.
#include <algorithm>

#include "gmi_internal.cuh"

using namespace gmi_dev;

namespace {

constexpr int kTW = 32;       // tile width  (pixels)
constexpr int kTH = 8;        // tile height (pixels)
constexpr int kThreads = kTW * kTH;
constexpr int kCap = 1024;    // staged candidates per chunk
constexpr int kCG = 4;        // channels per pass (grid.z = channel groups)

struct FwdParams {
    const Geom* geom;
    const int32_t* bins;
    const float* sx;
    const float* sy;
    const float* scol;  // [B][C][N]
    int N, C, W, H;
    double r64, r2_64;   // cutoff, cutoff^2 (f64, as the reference)
    float r2f, guard, nk;  // fp32 r^2, guard band, -log2(e)/(2 sigma^2)
    double inv2s2;      // 1/(2 sigma^2) (f64 weight mode)
    float* image;       // [B][H][W][C]
    float* wsum;        // [B][H][W]
    double* wsum64;     // [B][H][W] (f64 weight mode only)
    double* image64;    // [B][H][W][C] (f64 weight mode only)
    int32_t* counts;    // [B][H][W] or null
    Special* special;
    int32_t* special_count;
    int special_cap;
};

// kF64: weights and sums in f64 (gaussian_weight, core.cpp:49-53, exactly as
// the reference evaluates it) — used when cutoff > 6 sigma, where the fp32
// exponent argument (up to (r/sigma)^2/2) would carry more than the 1e-5
// relative error budget and fp32 weights could underflow.
template <bool kCount, bool kF64>
__global__ void __launch_bounds__(kThreads)
k_forward_tile(FwdParams p) {
    __shared__ float s_x[kCap];
    __shared__ float s_y[kCap];
    __shared__ float s_c[kCG][kCap];
    __shared__ int s_scan[kThreads / 32];
    __shared__ int s_n;

    const int tiles_y = (p.H + kTH - 1) / kTH;
    const int b = blockIdx.y / tiles_y;
    const int ty0 = (blockIdx.y % tiles_y) * kTH;
    const int tx0 = blockIdx.x * kTW;
    const int cg = blockIdx.z;
    const int ch0 = cg * kCG;
    const int nch = min(kCG, p.C - ch0);
    const Geom g = p.geom[b];
    const int tid = threadIdx.x;
    const int px = tx0 + (tid % kTW), py = ty0 + (tid / kTW);
    const float fx = static_cast<float>(px), fy = static_cast<float>(py);

    // candidate cell rectangle (bin_grid.cpp:88-91 for the whole tile)
    const double xlo = static_cast<double>(tx0) - p.r64;
    const double xhi = static_cast<double>(tx0 + kTW - 1) + p.r64;
    const double ylo = static_cast<double>(ty0) - p.r64;
    const double yhi = static_cast<double>(ty0 + kTH - 1) + p.r64;
    const int cx0 = cell_of(xlo, g.ox, g.cell, g.n_cols);
    const int cx1 = cell_of(xhi, g.ox, g.cell, g.n_cols);
    const int cy0 = cell_of(ylo, g.oy, g.cell, g.n_rows);
    const int cy1 = cell_of(yhi, g.oy, g.cell, g.n_rows);
    const float fxlo = static_cast<float>(xlo) - 1e-3f, fxhi = static_cast<float>(xhi) + 1e-3f;
    const float fylo = static_cast<float>(ylo) - 1e-3f, fyhi = static_cast<float>(yhi) + 1e-3f;

    const size_t base = static_cast<size_t>(b) * p.N;
    const float* sx = p.sx + base;
    const float* sy = p.sy + base;
    const float* sc = p.scol + static_cast<size_t>(b) * p.C * p.N;

    float wsum = 0.f;
    float num[kCG];
    double wsum64 = 0.0;
    double num64[kF64 ? kCG : 1];
#pragma unroll
    for (int c = 0; c < kCG; ++c) num[c] = 0.f;
#pragma unroll
    for (int c = 0; c < (kF64 ? kCG : 1); ++c) num64[c] = 0.0;
    int cnt = 0;

    if (tid == 0) s_n = 0;
    __syncthreads();

    auto consume = [&](int n) {
        for (int k = 0; k < n; ++k) {
            const float mx = s_x[k], my = s_y[k];
            if constexpr (kF64) {
                const double d2 = d2_ref(static_cast<double>(px), static_cast<double>(py),
                                         static_cast<double>(mx), static_cast<double>(my));
                if (d2 <= p.r2_64) {
                    const double w = exp(-d2 * p.inv2s2);
                    wsum64 += w;
#pragma unroll
                    for (int c = 0; c < kCG; ++c) num64[c] += w * static_cast<double>(s_c[c][k]);
                    if (kCount) ++cnt;
                }
                continue;
            }
            const float dx = fx - mx, dy = fy - my;
            const float d2 = fmaf(dx, dx, dy * dy);
            const float e = d2 - p.r2f;
            bool in = e <= 0.f;
            if (fabsf(e) <= p.guard) {
                in = d2_ref(static_cast<double>(px), static_cast<double>(py),
                            static_cast<double>(mx), static_cast<double>(my)) <= p.r2_64;
            }
            if (in) {
                // e = nk dx^2 + nk dy^2, the same fp32 operations as the
                // fast gather and the backward (bit-identical weights)
                const float w = ex2(fmaf(dx * p.nk, dx, (dy * p.nk) * dy));
                wsum += w;
#pragma unroll
                for (int c = 0; c < kCG; ++c) num[c] = fmaf(w, s_c[c][k], num[c]);
                if (kCount) ++cnt;
            }
        }
    };

    for (int cy = cy0; cy <= cy1; ++cy) {
        const int rs = p.bins[g.bin_off + static_cast<int64_t>(cy) * g.n_cols + cx0];
        const int re = p.bins[g.bin_off + static_cast<int64_t>(cy) * g.n_cols + cx1 + 1];
        for (int j0 = rs; j0 < re; j0 += kThreads) {
            const int j = j0 + tid;
            float mx = 0.f, my = 0.f;
            int keep = 0;
            if (j < re) {
                mx = sx[j];
                my = sy[j];
                keep = (mx >= fxlo && mx <= fxhi && my >= fylo && my <= fyhi) ? 1 : 0;
            }
            // deterministic block compaction (order = bin order)
            const int lane = tid & 31, warp = tid >> 5;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_scan[warp] = __popc(bal);
            __syncthreads();
            int before = 0, total = 0;
            for (int w = 0; w < kThreads / 32; ++w) {
                const int v = s_scan[w];
                before += w < warp ? v : 0;
                total += v;
            }
            const int n0 = s_n;
            if (n0 + total > kCap) {  // flush the buffer first
                consume(n0);
                __syncthreads();
                if (tid == 0) s_n = 0;
                __syncthreads();
            }
            const int dst = (n0 + total > kCap ? 0 : n0) + before +
                            __popc(bal & ((1u << lane) - 1u));
            if (keep) {
                s_x[dst] = mx;
                s_y[dst] = my;
#pragma unroll
                for (int c = 0; c < kCG; ++c)
                    s_c[c][dst] = c < nch ? sc[static_cast<size_t>(ch0 + c) * p.N + j] : 0.f;
            }
            __syncthreads();
            if (tid == 0) s_n = (n0 + total > kCap ? 0 : n0) + total;
            __syncthreads();
        }
    }
    consume(s_n);

    if (px >= p.W || py >= p.H) return;
    const size_t pix = static_cast<size_t>(py) * p.W + px;
    const size_t bp = static_cast<size_t>(b) * p.H * p.W + pix;
    float* out = p.image + bp * p.C + ch0;
    if constexpr (kF64) {
        if (wsum64 > 0.0) {
            for (int c = 0; c < nch; ++c) {
                const double o64 = num64[c] / wsum64;
                out[c] = static_cast<float>(o64);
                if (p.image64) p.image64[bp * p.C + ch0 + c] = o64;
            }
            if (cg == 0) {
                p.wsum64[bp] = wsum64;
                p.wsum[bp] = 1.0f;
                if (kCount) p.counts[bp] = cnt;
            }
        } else if (cg == 0) {
            p.wsum64[bp] = 0.0;
            p.wsum[bp] = 0.f;
            if (kCount) p.counts[bp] = 0;
            const int slot = atomicAdd(p.special_count, 1);
            if (slot < p.special_cap) p.special[slot] = Special{b, static_cast<int32_t>(pix), -1, 1};
        }
        return;
    }
    if (wsum > 0.f) {
        const float inv = 1.0f / wsum;
        for (int c = 0; c < nch; ++c) {
            // num/W with one Newton step: faithful quotient (engine.cpp:97-99)
            const float q0 = num[c] * inv;
            out[c] = fmaf(fmaf(-q0, wsum, num[c]), inv, q0);
        }
        if (cg == 0) {
            p.wsum[bp] = wsum;
            if (kCount) p.counts[bp] = cnt;
        }
    } else if (cg == 0) {
        // empty neighbourhood (fp32 weights are >= e^-18 here, so W == 0
        // exactly when the reference's wsum <= 0, engine.cpp:74-76)
        p.wsum[bp] = 0.f;
        if (kCount) p.counts[bp] = 0;
        const int slot = atomicAdd(p.special_count, 1);
        if (slot < p.special_cap) p.special[slot] = Special{b, static_cast<int32_t>(pix), -1, 1};
    }
}

// ---------------------------------------------------------------------------
// K3: one warp per special pixel.
struct SpecParams {
    const Geom* geom;
    const int32_t* bins;
    const float* sx;
    const float* sy;
    const int32_t* sidx;
    const float* scol;   // [B][C][N]
    const float4* rec;   // fast layout [B][N][2] (sx/sy/sidx null)
    const float* col;    // original colours [B][N][C]
    const float* wsum;
    int N, C, W, H;
    double r64, r2_64, sigma;
    int fallback;
    float* image;
    int32_t* counts;
    Special* special;
    const int32_t* special_count;
    int special_cap;
    int overflow_scan;   // 1: list overflowed — scan wsum for specials
};

// position and original index of hot-layout slot k (either layout)
__device__ __forceinline__ void point_at(const SpecParams& p, size_t k, float& x, float& y, int& i) {
    if (p.rec) {
        const float4 ra = p.rec[k * 2];
        x = ra.x;
        y = ra.y;
        i = static_cast<int>(__float_as_uint(p.rec[k * 2 + 1].z) & 0x7fffffffu);
    } else {
        x = p.sx[k];
        y = p.sy[k];
        i = p.sidx[k] & 0x7fffffff;
    }
}

__device__ __forceinline__ void warp_argmin(double& d2, int& idx) {
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d2, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (od < d2 || (od == d2 && oi < idx)) {
            d2 = od;
            idx = oi;
        }
    }
}

// exact argmin over all points, ties to the smallest original index
// (nearest_point's contract, bin_grid.hpp:39-41)
__device__ int nearest_exact(const SpecParams& p, const Geom& g, int b,
                             double qx, double qy) {
    const int lane = threadIdx.x & 31;
    const size_t base = static_cast<size_t>(b) * p.N;
    double best = INFINITY;
    int bi = INT32_MAX;
    if (g.capped) {
        // clamped edge cells break ring pruning: brute force
        for (int k = lane; k < p.N; k += 32) {
            float px, py;
            int i;
            point_at(p, base + k, px, py, i);
            const double d2 = d2_ref(qx, qy, static_cast<double>(px), static_cast<double>(py));
            if (d2 < best || (d2 == best && i < bi)) {
                best = d2;
                bi = i;
            }
        }
        warp_argmin(best, bi);
        return bi;
    }
    // Chebyshev ring search with the (ring-1)*cell bound (bin_grid.cpp:127-163)
    const int qcx = cell_of_unclamped(qx, g.ox, g.cell);
    const int qcy = cell_of_unclamped(qy, g.oy, g.cell);
    const int cap_x = max(abs(qcx), abs(qcx - (g.n_cols - 1)));
    const int cap_y = max(abs(qcy), abs(qcy - (g.n_rows - 1)));
    const int ring_cap = max(cap_x, cap_y);
    // lane-parallel over the cells of a ring (8 R cells), each lane scanning
    // its cell's points in turn; the bound is checked between rings exactly
    // as the reference does, so the set of rings visited is the same
    auto scan_cell_serial = [&](int gx, int gy) {
        if (gx < 0 || gx >= g.n_cols || gy < 0 || gy >= g.n_rows) return;
        const int64_t bin = g.bin_off + static_cast<int64_t>(gy) * g.n_cols + gx;
        const int s = p.bins[bin], e = p.bins[bin + 1];
        for (int k = s; k < e; ++k) {
            float px, py;
            int i;
            point_at(p, base + k, px, py, i);
            const double d2 = d2_ref(qx, qy, static_cast<double>(px), static_cast<double>(py));
            if (d2 < best || (d2 == best && i < bi)) {
                best = d2;
                bi = i;
            }
        }
    };
    // rings 0..kR0 at once (a fallback pixel's nearest point is usually 1-2
    // cells away): one round of dependent loads instead of kR0 + 1; the
    // argmin over a superset of the rings the reference visits is the same
    // point, and the ring bound then resumes at ring kR0 + 1
    constexpr int kR0 = 2, kSide0 = 2 * kR0 + 1;
    for (int c = lane; c < kSide0 * kSide0; c += 32)
        scan_cell_serial(qcx - kR0 + c % kSide0, qcy - kR0 + c / kSide0);
    for (int ring = kR0 + 1; ring <= ring_cap; ++ring) {
        double wb = best;
        int wi = bi;
        warp_argmin(wb, wi);
        if (wi != INT32_MAX) {
            const double lb = (ring - 1) * g.cell;
            if (lb * lb > wb) break;
        }
        const int side = 2 * ring + 1;
        for (int c = lane; c < 8 * ring; c += 32) {
            int gx, gy;
            if (c < side) {
                gx = qcx - ring + c;
                gy = qcy - ring;
            } else if (c < 2 * side) {
                gx = qcx - ring + (c - side);
                gy = qcy + ring;
            } else if (c < 2 * side + side - 2) {
                gx = qcx - ring;
                gy = qcy - ring + 1 + (c - 2 * side);
            } else {
                gx = qcx + ring;
                gy = qcy - ring + 1 + (c - 2 * side - (side - 2));
            }
            scan_cell_serial(gx, gy);
        }
    }
    warp_argmin(best, bi);
    return bi;
}

// Fallback pixel (engine.cpp:76-92): NearestPoint copies the colour of the
// exact argmin (ties to the smallest index); Zero writes 0.
__device__ void special_pixel(const SpecParams& p, int b, int pix, int slot) {
    const int lane = threadIdx.x & 31;
    const Geom g = p.geom[b];
    const int pr = pix / p.W, pc = pix % p.W;
    const double qx = pc, qy = pr;
    const size_t base = static_cast<size_t>(b) * p.N;
    float* out = p.image + (static_cast<size_t>(b) * p.H * p.W + pix) * p.C;
    int nearest = -1;
    if (p.fallback == GMI_FALLBACK_NEAREST) nearest = nearest_exact(p, g, b, qx, qy);
    if (nearest == INT32_MAX) nearest = -1;  // no finite point (a validation error is pending)
    if (lane == 0) {
        for (int c = 0; c < p.C; ++c)
            out[c] = nearest >= 0 ? p.col[(base + nearest) * p.C + c] : 0.0f;
        p.special[slot].nearest = nearest;
    }
}

__global__ void k_special(SpecParams p) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = min(*p.special_count, p.special_cap);
    for (int s = warp; s < n; s += nwarps) {
        const Special sp = p.special[s];
        special_pixel(p, sp.b, sp.pix, s);
    }
}

}  // namespace

namespace gmi_host {

static FwdParams fwd_params(const gmi_cache* c, float* image, int32_t* counts) {
    FwdParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.sx = c->sx;
    p.sy = c->sy;
    p.scol = c->scol;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.r2f = static_cast<float>(p.r2_64);
    p.guard = 4e-6f * p.r2f + 1e-30f;
    p.nk = static_cast<float>(-1.4426950408889634 / (2.0 * c->sigma * c->sigma));
    p.inv2s2 = 1.0 / (2.0 * c->sigma * c->sigma);
    p.image = image;
    p.wsum = c->wsum;
    p.wsum64 = c->wsum64;
    p.image64 = c->image64;
    p.counts = counts;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    return p;
}

void launch_forward(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts) {
    // fast path (gmi_gather.cu) unless f64 weights / C > 4 / very wide radius
    if (launch_gather_fast(ctx, c, image, counts)) return;
    const FwdParams p = fwd_params(c, image, counts);
    const int tiles_x = (c->W + kTW - 1) / kTW;
    const int tiles_y = (c->H + kTH - 1) / kTH;
    const dim3 grid(tiles_x, tiles_y * c->B, (c->C + kCG - 1) / kCG);
    GMI_CUDA(cudaMemsetAsync(c->special_count_d, 0, sizeof(int32_t), ctx->stream));
    const bool f64 = c->wsum64 != nullptr;
    if (counts) {
        if (f64) k_forward_tile<true, true><<<grid, kThreads, 0, ctx->stream>>>(p);
        else k_forward_tile<true, false><<<grid, kThreads, 0, ctx->stream>>>(p);
    } else {
        if (f64) k_forward_tile<false, true><<<grid, kThreads, 0, ctx->stream>>>(p);
        else k_forward_tile<false, false><<<grid, kThreads, 0, ctx->stream>>>(p);
    }
    GMI_LAUNCHED(ctx);
}

void launch_special_forward(gmi_ctx* ctx, gmi_cache* c, float* image, int32_t* counts) {
    SpecParams p{};
    p.geom = c->geom_d;
    p.bins = c->bins;
    p.sx = c->sx;
    p.sy = c->sy;
    p.sidx = c->sidx;
    p.scol = c->scol;
    p.rec = c->rec;
    p.col = c->col;
    p.wsum = c->wsum;
    p.N = c->N;
    p.C = c->C;
    p.W = c->W;
    p.H = c->H;
    p.r64 = c->cutoff;
    p.r2_64 = c->cutoff * c->cutoff;
    p.sigma = c->sigma;
    p.fallback = c->fallback;
    p.image = image;
    p.counts = counts;
    p.special = c->special;
    p.special_count = c->special_count_d;
    p.special_cap = c->special_cap;
    // one warp per fallback pixel, up to 64 per SM in flight: the ring
    // search is a chain of dependent loads, hidden by many pixels at once
    k_special<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(p);
    GMI_LAUNCHED(ctx);
}

}  // namespace gmi_host
