// Shared device-side definitions for the B200 Gaussian-mixture interpolation
// path.  Everything that must agree bit-for-bit between kernels (cell
// assignment, fine x-columns, the inclusion predicate) lives here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>

#define GMI_HD __host__ __device__ __forceinline__

// Device-side bounds checks for a debug build (-DGMI_DEBUG_BOUNDS, built by
// tools/gpu_bounds.sh as a variant library): every shared / global index of
// the hot kernels' staging, lists and scatters is checked and a violation
// traps with its location.  Compiled out of the product build.
#ifdef GMI_DEBUG_BOUNDS
#include <cstdio>
#define GMI_CHECK(cond)                                                          \
    do {                                                                         \
        if (!(cond)) {                                                           \
            printf("GMI_CHECK failed %s:%d: %s (block %d,%d,%d thread %d)\n",     \
                   __FILE__, __LINE__, #cond, blockIdx.x, blockIdx.y, blockIdx.z, \
                   threadIdx.x);                                                 \
            __trap();                                                            \
        }                                                                        \
    } while (0)
#else
#define GMI_CHECK(cond) do { } while (0)
#endif

namespace gmi_dev {

// ----------------------------------------------------------------------------
// Reference arithmetic (bin_grid.cpp:14-36), f64, no contraction.
// ----------------------------------------------------------------------------

// (int)v as the reference's x86-64 build executes it (cvttsd2si): NaN and
// out-of-range values become INT_MIN.  The C++ cast is UB there; this pins
// the behaviour the reference binary actually has.
GMI_HD int x86_d2i(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(v);
}

GMI_HD int clamp_int(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// BinGrid::cell_of_x / cell_of_y (bin_grid.cpp:28-36):
//   clamp((int)floor((v - origin) / cell), 0, n - 1)
__device__ __forceinline__ int cell_of(double v, double origin, double cell,
                                       int n) {
    const double t = __ddiv_rn(__dsub_rn(v, origin), cell);
    return clamp_int(x86_d2i(floor(t)), 0, n - 1);
}

// cell_of with the division replaced by a multiply by the rounded
// reciprocal: q = d * (1/cell) is within ~2 ulp of fl(d / cell), so its floor
// is the reference's unless q lies within 1e-9 of an integer (|q| < 2^20
// here), in which case the exact division decides.  Bit-identical to cell_of.
__device__ __forceinline__ int cell_of_fast(double v, double origin, double cell,
                                            double inv_cell, int n) {
    const double d = __dsub_rn(v, origin);
    const double q = __dmul_rn(d, inv_cell);
    double f = floor(q);
    if (!(q - f > 1e-9 && f + 1.0 - q > 1e-9 && fabs(q) < 1048576.0))
        f = floor(__ddiv_rn(d, cell));
    return clamp_int(x86_d2i(f), 0, n - 1);
}

// Unclamped cell index (nearest_point's ring centre, bin_grid.cpp:131-132).
__device__ __forceinline__ int cell_of_unclamped(double v, double origin,
                                                 double cell) {
    return x86_d2i(floor(__ddiv_rn(__dsub_rn(v, origin), cell)));
}

// rsqrt.approx without the denormal-input fix-up (callers clamp the input
// to >= 1e-30, a normal number): the same MUFU.RSQ result as rsqrtf for every
// normal input, three instructions shorter.
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One 32-byte record as ONE 256-bit store (STG.E.ENL2.256): the sector is
// written whole, so scattered record writes never leave half-written sectors
// for the L2 to merge or read back.  p must be 32-byte aligned.
__device__ __forceinline__ void st_rec32(float4* p, const float4 a, const float4 b) {
    GMI_CHECK((reinterpret_cast<uintptr_t>(p) & 31) == 0);
#ifdef GMI_REC_STORE128
    p[0] = a;  // A/B: two 128-bit stores
    p[1] = b;
#else
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 :: "l"(p), "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                 : "memory");
#endif
}

// One 32-byte record as ONE 256-bit load (LDG.E.ENL2.256).
__device__ __forceinline__ void ld_rec32(const float4* p, float4& a, float4& b) {
    GMI_CHECK((reinterpret_cast<uintptr_t>(p) & 31) == 0);
    asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}

// Reference inclusion predicate (bin_grid.cpp:87,98; core.hpp:21-23):
//   (qx-mx)^2 + (qy-my)^2 <= r^2, f64, two roundings, no FMA.
__device__ __forceinline__ double d2_ref(double qx, double qy, double mx,
                                         double my) {
    const double dx = __dsub_rn(qx, mx);
    const double dy = __dsub_rn(qy, my);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// ----------------------------------------------------------------------------
// Exact inclusion with fp32 arithmetic.
//
// The reference includes point i in pixel q iff fl64(dx^2 + dy^2) <= r^2
// (bin_grid.cpp:98).  A point is SAFE when every integer pixel q has
// |d^2(q) - r^2| > kAmbRel * r^2.  For a safe point every fp32 evaluation of
// d^2 used by the kernels (relative error < 1e-6) takes the reference's
// decision, so the hot loops compare in fp32 with no guard band.  The few
// AMBIGUOUS points (about 1e-4 of random inputs; all of them for integer
// lattices at integer radii) are flagged once by K1 (bit 31 of the sorted
// index) and decided with the f64 predicate d2_ref everywhere.
//
// Only the integer nearest to each row's two boundary crossings mu_x +- s,
// s = sqrt(r^2 - dy^2), can be within the band: any other integer is >= 1/2
// away from both crossings, so |dx^2 - s^2| >= 1/4.
// ----------------------------------------------------------------------------
constexpr float kAmbRel = 8e-6f;
constexpr uint32_t kUnsafeBit = 0x80000000u;

__device__ __forceinline__ bool point_ambiguous(float mx, float my, double r64,
                                                double r2_64, float r2f) {
    if (!(fabsf(mx) < 1048576.f && fabsf(my) < 1048576.f)) return true;
    const float tau = kAmbRel * r2f;
    const float tx = truncf(mx);
    const float fmu = mx - tx;  // exact
    const float rf = static_cast<float>(r64);
    const int y0 = static_cast<int>(floorf(my - rf)) - 1;
    const int y1 = static_cast<int>(ceilf(my + rf)) + 1;
    for (int y = y0; y <= y1; ++y) {
        const double dy = __dsub_rn(static_cast<double>(y), static_cast<double>(my));
        const float h2f = static_cast<float>(__dsub_rn(r2_64, __dmul_rn(dy, dy)));
        if (h2f < -tau) continue;
        const float s = sqrtf(fmaxf(h2f, 0.f));
        const float nl = rintf(fmu - s), nr = rintf(fmu + s);
        const float el = fmaf(nl - fmu, nl - fmu, -h2f);
        const float er = fmaf(nr - fmu, nr - fmu, -h2f);
        if (fabsf(el) <= tau || fabsf(er) <= tau) return true;
    }
    return false;
}

// ----------------------------------------------------------------------------
// Per-image grid geometry (BinGrid fields, bin_grid.hpp:17-28) plus the
// hot-path extras.
// ----------------------------------------------------------------------------
struct Geom {
    double ox, oy;     // origin = (min - cell) (bin_grid.cpp:58)
    double cell;       // = cutoff_radius (engine.cpp:115)
    int n_cols, n_rows;
    int64_t bin_off;   // offset of this image's bin_start in the bin array
    int capped;        // 1 when an axis hit the cell cap (clamping active)
    float qx0;         // fine x-column anchor (float(ox))
    float qscale;      // fine x-columns per pixel
};

// Fine x-column of a position: monotone non-decreasing in x (fp32 subtract
// and multiply by a positive constant are monotone; floorf too).  Within a
// cell the hot layout is sorted by (fine column, original index), so the
// concatenation of the cells of one cell row is sorted by fine column.
__device__ __forceinline__ int fine_col(float x, float qx0, float qscale) {
    const float t = floorf((x - qx0) * qscale);
    // clamp into int range; NaN -> 0 (invalid inputs are rejected anyway)
    if (!(t > -1.0e9f)) return -1000000000;
    if (t > 1.0e9f) return 1000000000;
    return static_cast<int>(t);
}

// ----------------------------------------------------------------------------
// float <-> order-preserving uint for atomic min/max
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
GMI_HD float ord2f(uint32_t u) {
    const uint32_t v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
    return __uint_as_float(v);
#else
    float f;
    std::memcpy(&f, &v, 4);
    return f;
#endif
}

// exp2 on the SFU (MUFU.EX2), flush-to-zero.
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Validation issue key: (point index << 8) | (1 + ErrorCode).  atomicMin over
// keys selects the reference's first violated invariant (core.cpp:55-96):
// lowest point index first; within a point positions are checked before
// colours, colours in channel order.
constexpr unsigned long long kNoIssue = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ bool is_finite_f(float v) {
    return fabsf(v) <= 3.402823466e38f;  // false for inf and NaN
}

}  // namespace gmi_dev
