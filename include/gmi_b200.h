/*
 * gmi_b200.h — C-ABI of the B200-native Gaussian-mixture interpolation hot
 * path (arXiv 2012.13257).  Plain pointers and sizes only; no torch, no C++
 * types.  Implemented by libgmi_b200.so (paper_2012_13257_b200/csrc/).
 *
 * Every entry point replaces one interface of the reference
 * (/root/reference/proj) — cited beside it.  Semantics, argument meaning and
 * error codes follow the reference; the differences are the batch dimension
 * (B independent reference calls), fp32 storage
 * (the reference is f64; tolerance rel 1e-5 / abs 1e-6) and C >= 1 instead
 * of C in {1,3} (core.cpp:60-64).
 *
 * Layouts (per image identical to the reference, batch-major):
 *   positions  [B][N][2]   x,y interleaved        (core.hpp:67-79 PointSet)
 *   colors     [B][N][C]   point-major            (core.hpp:67-79)
 *   image      [B][H][W][C] row-major, channel-last (core.hpp:96-117)
 *   upstream   [B][H][W][C]
 *   d_colors   [B][N][C],  d_positions [B][N][2]  (core.hpp:121-131)
 * Pixel (row r, col c) is centred at (x=c, y=r) (core.hpp:25-30).
 *
 * Error convention: every int-returning call returns GMI_OK (0) or a
 * gmi_status; the reference's gmi::ErrorCode values map to 1 + code
 * (core.hpp:35-50); CUDA failures map to GMI_ERR_CUDA.  A thread-local
 * message is available from gmi_last_error().  No exception crosses the ABI.
 */
#ifndef GMI_B200_H
#define GMI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gmi_status {
    GMI_OK = 0,
    /* 1 + gmi::ErrorCode (core.hpp:35-50) */
    GMI_ERR_NON_FINITE_VALUE = 1,
    GMI_ERR_COLOR_OUT_OF_RANGE = 2,
    GMI_ERR_EMPTY_POINT_SET = 3,
    GMI_ERR_SHAPE_MISMATCH = 4,
    GMI_ERR_INVALID_CELL_SIZE = 5,
    GMI_ERR_CONFIG_INVALID = 6,
    GMI_ERR_CACHE_MISMATCH = 7,
    GMI_ERR_INVALID_DIMENSIONS = 8,
    GMI_ERR_INVALID_FACTOR = 9,
    GMI_ERR_INVALID_COUNT = 10,
    GMI_ERR_UNSUPPORTED_FORMAT = 11,
    GMI_ERR_CORRUPT_FILE = 12,
    GMI_ERR_EMPTY_LOG = 13,
    GMI_ERR_IO_ERROR = 14,
    /* B200-side failures (no reference equivalent) */
    GMI_ERR_CUDA = 100,
    GMI_ERR_INVALID_ARGUMENT = 101,
    GMI_ERR_OUT_OF_MEMORY = 102
} gmi_status;

/* Fallback policy for empty neighbourhoods (core.hpp:32-33 Fallback). */
enum { GMI_FALLBACK_NEAREST = 0, GMI_FALLBACK_ZERO = 1 };

/* Interpolation parameters (core.hpp:81-88 InterpConfig).  sigma and
 * cutoff_radius stay double so r^2 and the bin geometry are computed exactly
 * as the reference computes them.  cutoff_radius <= 0 is rejected
 * (ConfigInvalid); use gmi_default_cutoff() for make_config's 3*sigma
 * (core.hpp:90-94). */
typedef struct gmi_config {
    double sigma;
    double cutoff_radius;
    int32_t fallback; /* GMI_FALLBACK_* */
    int32_t width;    /* CoordinateFrame (core.hpp:25-30) */
    int32_t height;
} gmi_config;

/* Context flags. */
enum {
    /* Report validation errors asynchronously: forward/backward return as
     * soon as the work is queued and a later gmi_ctx_synchronize() returns
     * the first error.  This includes the host-buffer calls
     * (gmi_forward_host / gmi_backward_host): their host outputs are
     * complete, and their host inputs may be reused, after
     * gmi_ctx_synchronize() — so a backward's upload overlaps the preceding
     * forward's download.  Default (0): every call synchronises and returns
     * the reference's error synchronously.  The pending error is the first
     * failing call's first failing image (smallest index there); it stays
     * pending until gmi_ctx_synchronize() reports and clears it. */
    GMI_CTX_ASYNC_ERRORS = 1u << 0,
    /* Reserved, ignored: every path (forward, backward, fallback routing) is
     * bit-deterministic run to run; there is no faster non-deterministic
     * mode. */
    GMI_CTX_NONDETERMINISTIC = 1u << 1,
    /* Reference-grade precision: weights, sums and the normalised image of
     * the gradient in f64 (the path cutoff > 6 sigma always takes), for
     * inputs where the fp32 hot path's d_positions / d_colors can exceed the
     * 1e-6 absolute floor — isolated points at sigma < 1, disks of thousands
     * of pixels, > ~10^4 contributors per pixel.  Slower
     * (generic kernels); the image itself is returned in fp32. */
    GMI_CTX_PRECISE = 1u << 2,
    /* Test hook, the analogue of the reference's inject_fault
     * (validate.cpp:207-209): every backward adds 1e-3 to d_colors[0] of its
     * first image on the device, so a parity harness can prove it detects a
     * corrupted GPU output.  Never set in production. */
    GMI_CTX_INJECT_FAULT = 1u << 3
};

typedef struct gmi_ctx gmi_ctx;     /* one device + one stream */
typedef struct gmi_cache gmi_cache; /* ForwardCache (engine.hpp:20-41) */

/* ---- context ------------------------------------------------------------ */
int gmi_ctx_create(int device, gmi_ctx** out);
/* Drops the caller's handle.  Caches made on the ctx keep it alive (its
 * stream and device state) until the last of them is freed. */
int gmi_ctx_destroy(gmi_ctx* ctx);
/* Use an external cudaStream_t (passed as void*); NULL = the ctx's own. */
int gmi_ctx_set_stream(gmi_ctx* ctx, void* cuda_stream);
void* gmi_ctx_stream(const gmi_ctx* ctx);
int gmi_ctx_set_flags(gmi_ctx* ctx, uint32_t flags);
/* Waits for queued work; returns the first pending asynchronous error. */
int gmi_ctx_synchronize(gmi_ctx* ctx);
/* Makes the ctx stream wait (on the device, no host block) for the copies
 * queued by asynchronous host-buffer calls, e.g. before recording an event
 * that must cover their downloads. */
int gmi_ctx_join_host_copies(gmi_ctx* ctx);
/* Number of kernels this ctx has launched (for bench gpu_launches). */
uint64_t gmi_ctx_launch_count(const gmi_ctx* ctx);

/* Per-phase device time (CUDA events on the ctx stream), for measurement:
 *   0 BIN       K1 binning (bbox, count, scan, scatter, cell sort + SoA)
 *   1 GATHER    K2 forward gather
 *   2 SPECIAL_F K3 fallback / exact pixels (forward)
 *   3 POINTS    K4 point-major backward
 *   4 SPECIAL_B K5 fallback routing / exact pixels (backward)
 * gmi_ctx_phase_times synchronises the stream, folds the recorded events into
 * ms[GMI_NUM_PHASES] / calls[GMI_NUM_PHASES] (accumulated since the last
 * reset) and optionally resets them. */
#define GMI_NUM_PHASES 5
int gmi_ctx_set_profiling(gmi_ctx* ctx, int on);
int gmi_ctx_phase_times(gmi_ctx* ctx, double* ms, uint64_t* calls, int reset);

/* ---- helpers ------------------------------------------------------------- */
const char* gmi_last_error(void);
const char* gmi_error_name(int code); /* error_code_name (core.cpp:7-25) */
const char* gmi_version(void);
/* make_config's default cutoff (core.hpp:90-94): 3*sigma. */
double gmi_default_cutoff(double sigma);
/* gaussian_weight (core.cpp:49-53), host f64. */
double gmi_gaussian_weight(double qx, double qy, double mux, double muy,
                           double sigma);

/* ---- forward: gmi::forward (engine.hpp:48-55, engine.cpp:107-176) --------
 * Device pointers.  Writes image[B][H][W][C] and returns a cache that owns
 * the per-pixel normalizer W, fallback flags / nearest indices and the
 * binned point layout; it records (does not copy) `positions`, `colors` and
 * `image`, which must stay valid and unmodified until gmi_backward() has
 * been queued or the cache is freed — the reference keeps the same data
 * inside ForwardCache (cache.output, engine.cpp:174).  num_workers of the
 * reference has no equivalent (output is worker-independent there too). */
int gmi_forward(gmi_ctx* ctx, const float* positions, const float* colors,
                int32_t batch, int32_t num_points, int32_t channels,
                const gmi_config* cfg, float* image, gmi_cache** cache_out);

/* ---- backward: gmi::backward (engine.hpp:57-64, engine.cpp:238-309) ------
 * Gradients of sum(upstream * forward_output) w.r.t. colours and positions.
 * Throws (returns) CacheMismatch under the reference's exact == checks on
 * N, C, W, H, sigma, cutoff and fallback (engine.cpp:243-250). */
int gmi_backward(gmi_ctx* ctx, const float* positions, const float* colors,
                 int32_t batch, int32_t num_points, int32_t channels,
                 const gmi_config* cfg, const gmi_cache* cache,
                 const float* upstream, float* d_colors, float* d_positions);

/* Host-buffer variants (the reference's value-semantics API shape): inputs
 * and outputs are host pointers (pinned or pageable); the H2D and D2H copies
 * run on the ctx stream inside the call.  The cache keeps device copies. */
int gmi_forward_host(gmi_ctx* ctx, const float* positions, const float* colors,
                     int32_t batch, int32_t num_points, int32_t channels,
                     const gmi_config* cfg, float* image, gmi_cache** cache_out);
int gmi_backward_host(gmi_ctx* ctx, const float* positions,
                      const float* colors, int32_t batch, int32_t num_points,
                      int32_t channels, const gmi_config* cfg,
                      const gmi_cache* cache, const float* upstream,
                      float* d_colors, float* d_positions);

/* ---- ForwardCache accessors (engine.hpp:20-41, bindings.cpp:133-139) ---- */
void gmi_cache_free(gmi_cache* cache);
/* ForwardCache::fallback_count (engine.cpp:27-33), per image; out[batch]. */
int gmi_cache_fallback_count(const gmi_cache* cache, int64_t* out);
int gmi_cache_shape(const gmi_cache* cache, int32_t* batch, int32_t* num_points,
                    int32_t* channels, int32_t* width, int32_t* height);
/* Copies per-pixel cache arrays to HOST buffers (any may be NULL):
 * normalizer[B][H][W] (fp32 W = sum of weights, 0 on fallback pixels),
 * fallback_flag[B][H][W] (uint8), nearest_index[B][H][W] (int32, -1 when not
 * a NearestPoint fallback pixel) — engine.hpp:32-34. */
int gmi_cache_copy_pixels(const gmi_cache* cache, float* normalizer,
                          uint8_t* fallback_flag, int32_t* nearest_index);
/* Per-pixel contribution counts (pixel_start deltas, engine.hpp:29-31),
 * computed by the same gather kernel instantiated with counting on;
 * counts[B][H][W] int32 on the HOST.  Test/parity use. */
int gmi_forward_counts(gmi_ctx* ctx, const gmi_cache* cache, int32_t* counts);

/* ---- spatial bin grid: build_bin_grid (bin_grid.hpp:17-31,
 * bin_grid.cpp:38-82) --------------------------------------------------------
 * Bit-exact reproduction of the reference BinGrid for each image (f64 cell
 * arithmetic, 2048-cells-per-axis cap, stable ascending point_index within
 * each bin).  Device input positions[B][N][2]; HOST outputs:
 *   origin[B][2] (double), n_cols[B], n_rows[B]  — first call with
 *   bin_start == NULL to size; then bin_start[sum(n_cols*n_rows + 1)]
 *   (concatenated per image) and point_index[B][N]. */
int gmi_bin_grid(gmi_ctx* ctx, const float* positions, int32_t batch,
                 int32_t num_points, double cell_size, double* origin,
                 int32_t* n_cols, int32_t* n_rows, int32_t* bin_start,
                 int32_t* point_index);
/* Same with HOST input positions (copied to the device inside the call). */
int gmi_bin_grid_host(gmi_ctx* ctx, const float* positions, int32_t batch,
                      int32_t num_points, double cell_size, double* origin,
                      int32_t* n_cols, int32_t* n_rows, int32_t* bin_start,
                      int32_t* point_index);

/* ---- point optimisation: optimize_points (optimize.hpp:43-46,
 * optimize.cpp:47-98) -------------------------------------------------------
 * `steps` rounds of: forward -> L1 loss against target (l1_loss_and_grad,
 * optimize.cpp:12-28: loss = mean |pred - target|, upstream = sign/(H*W*C))
 * -> backward -> descent (positions -= lr * d_positions; colours clamped to
 * [0,1] after colours -= lr * d_colors), the bin grid rebuilt on the device in
 * every forward.  positions[B][N][2] / colors[B][N][C] are updated in place
 * (DEVICE buffers); target[B][H][W][C] on the device; loss_curve, if not NULL,
 * receives B x (steps + 1) losses on the HOST (step 0 = the initial points).
 * flags: GMI_OPT_POSITIONS | GMI_OPT_COLORS.  steps >= 1 and a finite
 * learning_rate >= 0, else ConfigInvalid (optimize.cpp:32-44). */
enum { GMI_OPT_POSITIONS = 1, GMI_OPT_COLORS = 2 };
int gmi_optimize_points(gmi_ctx* ctx, float* positions, float* colors, int32_t batch,
                        int32_t num_points, int32_t channels, const gmi_config* cfg,
                        const float* target, int32_t steps, double learning_rate,
                        uint32_t flags, double* loss_curve);
/* Same with HOST buffers (copied in and back inside the call). */
int gmi_optimize_points_host(gmi_ctx* ctx, float* positions, float* colors, int32_t batch,
                             int32_t num_points, int32_t channels, const gmi_config* cfg,
                             const float* target, int32_t steps, double learning_rate,
                             uint32_t flags, double* loss_curve);

/* ---- device memory for callers without a framework (the zero-copy Python
 * path): cudaMalloc / cudaFree on the ctx's device, and a copy
 * ordered on the ctx stream (kind: 0 host->device, 1 device->host,
 * 2 device->device; host memory may be pageable; returns after the copy). */
int gmi_device_alloc(gmi_ctx* ctx, size_t bytes, void** out);
int gmi_device_free(gmi_ctx* ctx, void* ptr);
int gmi_memcpy(gmi_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind);

/* ---- run_benchmark's GMM branch (benchmark.cpp:88-107) for one image ------
 * image: HOST H x W x C.  Known points at the block centres of `lowres`
 * (HOST lh x lw x C, lh = ceil(H/factor), lw = ceil(W/factor);
 * point_set_from_lowres, benchmark.cpp:24-39) or, lowres == NULL, of the
 * block means of `image` computed on the device (block_mean_downsample,
 * imaging.cpp:306-350).  One forward per sigma over the full W x H frame
 * (make_config: cutoff 3 sigma, NearestPoint), L1 against `image` (l1_metric,
 * imaging.cpp:376-386): l1[k] and ms[k] (device time of that forward; ms may
 * be NULL) per sigma; *best = the first sigma with the smallest L1
 * (benchmark.cpp:101-106); best_image (HOST H x W x C, may be NULL) receives
 * that forward's output.  sigmas == NULL: auto_sigma_candidates(factor) =
 * {0.4, 0.5, 0.6} * factor (benchmark.cpp:48-50), n_sigma must be 3.
 * factor < 1: GMI_ERR_INVALID_FACTOR (benchmark.cpp:62-68). */
int gmi_gmm_benchmark_host(gmi_ctx* ctx, const float* image, int32_t width, int32_t height,
                           int32_t channels, int32_t factor, const float* lowres,
                           const double* sigmas, int32_t n_sigma, double* l1, double* ms,
                           int32_t* best, float* best_image);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GMI_B200_H */
