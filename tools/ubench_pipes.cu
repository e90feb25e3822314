// Pipe-throughput microbenchmarks on B200 (sm_100a): scalar FFMA, f32x2
// FFMA2/FADD2/FMUL2, MUFU.EX2, FSETP+FSEL, shared-memory loads and float
// atomics.  Each kernel runs many independent chains so latency is hidden;
// the result is lane-ops per SM per clock at the observed SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void k_ffma(float* out, float a, float b) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fmaf(v[k], a, b);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    float2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float2(threadIdx.x + k, k);
    const float2 A = make_float2(a, a), Bv = make_float2(b, b);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ffma2_rn(v[k], A, Bv);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    if (s == 12345.f) out[0] = s;
}

__global__ void k_fadd2(float* out, float a, float b) {
    float2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float2(threadIdx.x + k, k);
    const float2 A = make_float2(a, b);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __fadd2_rn(v[k], A);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    if (s == 12345.f) out[0] = s;
}

__global__ void k_mufu(float* out, float a, float b) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = -(threadIdx.x + k) * 1e-3f;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ex2(v[k]);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 12345.f) out[0] = s;
}

// 4 FFMA2 : 1 MUFU (does MUFU co-issue with the fma pipe?)
__global__ void k_mix(float* out, float a, float b) {
    float2 v[4];
    float m[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = make_float2(threadIdx.x + k, k);
        m[k] = -(threadIdx.x + k) * 1e-3f;
    }
    const float2 A = make_float2(a, a), Bv = make_float2(b, b);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = __ffma2_rn(v[k], A, Bv);
            m[k] = ex2(m[k]);
        }
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += v[k].x + v[k].y + m[k];
    if (s == 12345.f) out[0] = s;
}

// compare + select (the in-disk mask)
__global__ void k_sel(float* out, float a, float b) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = v[k] <= a ? v[k] : b;
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 12345.f) out[0] = s;
}

// LDS.128 with per-lane stride (stride 1 = conflict-free, 0 = broadcast)
__global__ void k_lds(float* out, int stride, int mask) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = (threadIdx.x & 31) * stride;
    for (int i = 0; i < ITERS; ++i) {
        const float4 t = s[(idx + i) & mask];
        acc.x += t.x;
        acc.y += t.y;
        acc.z += t.z;
        acc.w += t.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = 1;
}

// shared-memory float atomics, lanes hit distinct words (stride) in a 4K table
__global__ void k_atoms(float* out, int stride) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    int idx = (threadIdx.x * stride) & 4095;
    for (int i = 0; i < ITERS / 4; ++i) {
        atomicAdd(&s[(idx + i * 33) & 4095], 1.0f);
    }
    __syncthreads();
    if (s[threadIdx.x] == 12345.f) out[0] = 1;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread, int blocks, int threads) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double ops = ops_per_thread * blocks * threads;
    const double per_sm_clk = ops / (ms * 1e-3) / 148.0 / 1.965e9;
    printf("%-28s %8.3f ms  %8.1f lane-ops/SM/clk (at 1965 MHz)\n", name, ms, per_sm_clk);
}

int main() {
    float* out;
    cudaMalloc(&out, 16);
    const int B = 148 * 8, T = 256;
    run("FFMA (scalar)", [&] { k_ffma<<<B, T>>>(out, 0.999f, 0.001f); }, 8.0 * ITERS, B, T);
    run("FFMA2 (x2 ops)", [&] { k_ffma2<<<B, T>>>(out, 0.999f, 0.001f); }, 16.0 * ITERS, B, T);
    run("FADD2 (x2 ops)", [&] { k_fadd2<<<B, T>>>(out, 0.999f, 0.001f); }, 16.0 * ITERS, B, T);
    run("MUFU.EX2", [&] { k_mufu<<<B, T>>>(out, 0.f, 0.f); }, 8.0 * ITERS, B, T);
    run("mix 4 FFMA2 + 4 EX2 (ex2 ops)", [&] { k_mix<<<B, T>>>(out, 0.999f, 0.001f); }, 4.0 * ITERS, B, T);
    run("FSETP+FSEL", [&] { k_sel<<<B, T>>>(out, 100.f, 0.f); }, 8.0 * ITERS, B, T);
    run("LDS.128 broadcast", [&] { k_lds<<<B, T>>>(out, 0, 2047); }, 1.0 * ITERS, B, T);
    run("LDS.128 stride1", [&] { k_lds<<<B, T>>>(out, 1, 2047); }, 1.0 * ITERS, B, T);
    run("LDS.128 stride5", [&] { k_lds<<<B, T>>>(out, 5, 2047); }, 1.0 * ITERS, B, T);
    run("LDS.128 stride6", [&] { k_lds<<<B, T>>>(out, 6, 2047); }, 1.0 * ITERS, B, T);
    run("ATOMS.ADD.F32 stride1", [&] { k_atoms<<<B, T>>>(out, 1); }, ITERS / 4.0, B, T);
    run("ATOMS.ADD.F32 stride 7", [&] { k_atoms<<<B, T>>>(out, 7); }, ITERS / 4.0, B, T);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
