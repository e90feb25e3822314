// Shared device-side definitions for the B200 Gaussian-mixture interpolation
// path.  Everything that must agree bit-for-bit between kernels (cell
// assignment, fine x-columns, the inclusion predicate) lives here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>

#define GMI_HD __host__ __device__ __forceinline__

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

// Unclamped cell index (nearest_point's ring centre, bin_grid.cpp:131-132).
__device__ __forceinline__ int cell_of_unclamped(double v, double origin,
                                                 double cell) {
    return x86_d2i(floor(__ddiv_rn(__dsub_rn(v, origin), cell)));
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
