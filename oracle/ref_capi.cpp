// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference implementation, compiled
// from the reference's own sources where they lie
// (/root/reference/proj/src/{core,bin_grid,engine,oracle,validate,optimize,
// imaging,resample,benchmark}.cpp) by
// oracle/Makefile into oracle/_ref/libgmi_ref.so.  It lets the Python test
// harness and bench.py's cpu_baseline / --impl reference legs call the
// reference's C++ API (gmi::forward / gmi::backward / gmi::build_bin_grid /
// gmi::oracle_forward ...) through ctypes.  Nothing here re-implements the
// algorithm: every call forwards to the reference function cited beside it.
//
// Error convention: return 0 on success, 1 + (int)gmi::ErrorCode on a
// gmi::Error (core.hpp:35-50), 100 on any other exception; the message is
// copied into a thread-local buffer readable through ref_last_error().

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gmi/benchmark.hpp"
#include "gmi/bin_grid.hpp"
#include "gmi/engine.hpp"
#include "gmi/imaging.hpp"
#include "gmi/optimize.hpp"
#include "gmi/oracle.hpp"
#include "gmi/rng.hpp"
#include "gmi/validate.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return 0;
    } catch (const gmi::Error& e) {
        g_last_error = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 100;
    }
}

gmi::PointSet make_points(const double* pos, const double* col, int n,
                          int channels) {
    gmi::PointSet ps;
    ps.channels = channels;
    ps.positions.resize(n);
    for (int i = 0; i < n; ++i) {
        ps.positions[i] = {pos[2 * i], pos[2 * i + 1]};
    }
    ps.colors.assign(col, col + static_cast<std::size_t>(n) * channels);
    return ps;
}

gmi::InterpConfig make_cfg(double sigma, double cutoff, int fallback,
                           int width, int height) {
    gmi::InterpConfig cfg;
    cfg.sigma = sigma;
    cfg.cutoff_radius = cutoff;
    cfg.fallback = fallback == 0 ? gmi::Fallback::NearestPoint
                                 : gmi::Fallback::Zero;
    cfg.frame = {width, height};
    return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

// gmi::gaussian_weight (core.cpp:49-53)
double ref_gaussian_weight(double qx, double qy, double mx, double my,
                           double sigma) {
    return gmi::gaussian_weight({qx, qy}, {mx, my}, sigma);
}

// gmi::build_bin_grid (bin_grid.cpp:38-82).  Returns an opaque handle.
int ref_bin_grid_new(const double* pos, const double* col, int n, int channels,
                     double cell, void** out) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        *out = new gmi::BinGrid(gmi::build_bin_grid(ps, cell));
    });
}

void ref_bin_grid_info(const void* h, double* origin, int* n_cols,
                       int* n_rows) {
    const auto* g = static_cast<const gmi::BinGrid*>(h);
    origin[0] = g->origin.x;
    origin[1] = g->origin.y;
    *n_cols = g->n_cols;
    *n_rows = g->n_rows;
}

void ref_bin_grid_copy(const void* h, int* bin_start, int* point_index) {
    const auto* g = static_cast<const gmi::BinGrid*>(h);
    std::memcpy(bin_start, g->bin_start.data(),
                g->bin_start.size() * sizeof(int));
    std::memcpy(point_index, g->point_index.data(),
                g->point_index.size() * sizeof(int));
}

void ref_bin_grid_free(void* h) { delete static_cast<gmi::BinGrid*>(h); }

// gmi::query_radius (bin_grid.cpp:84-105); out must hold n ints.
int ref_query_radius(const double* pos, const double* col, int n, int channels,
                     double cell, double qx, double qy, double radius,
                     int* out, int* count) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        const gmi::BinGrid g = gmi::build_bin_grid(ps, cell);
        const std::vector<int> hits = gmi::query_radius(g, ps, {qx, qy}, radius);
        std::memcpy(out, hits.data(), hits.size() * sizeof(int));
        *count = static_cast<int>(hits.size());
    });
}

// gmi::nearest_point (bin_grid.cpp:114-164) for a batch of queries.
int ref_nearest_point(const double* pos, const double* col, int n,
                      int channels, double cell, const double* q, int nq,
                      int* out) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        const gmi::BinGrid g = gmi::build_bin_grid(ps, cell);
        for (int k = 0; k < nq; ++k) {
            out[k] = gmi::nearest_point(g, ps, {q[2 * k], q[2 * k + 1]});
        }
    });
}

// gmi::forward (engine.cpp:107-176).  image: H*W*C doubles.  The returned
// handle owns the ForwardCache (engine.hpp:20-41).
int ref_forward(const double* pos, const double* col, int n, int channels,
                int width, int height, double sigma, double cutoff,
                int fallback, int workers, double* image, void** cache_out) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        const gmi::InterpConfig cfg =
            make_cfg(sigma, cutoff, fallback, width, height);
        gmi::ForwardResult r = gmi::forward(ps, cfg, cfg.frame, workers);
        std::memcpy(image, r.image.data.data(),
                    r.image.data.size() * sizeof(double));
        *cache_out = new gmi::ForwardCache(std::move(r.cache));
    });
}

void ref_cache_info(const void* h, std::int64_t* num_pairs,
                    int* fallback_count) {
    const auto* c = static_cast<const gmi::ForwardCache*>(h);
    *num_pairs = static_cast<std::int64_t>(c->contrib_point.size());
    *fallback_count = c->fallback_count();
}

// Any pointer may be null to skip that array.
void ref_cache_copy(const void* h, std::int64_t* pixel_start,
                    int* contrib_point, double* contrib_weight,
                    double* normalizer, std::uint8_t* fallback_flag,
                    int* nearest_index) {
    const auto* c = static_cast<const gmi::ForwardCache*>(h);
    auto cp = [](auto* dst, const auto& v) {
        if (dst != nullptr && !v.empty()) {
            std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
        }
    };
    cp(pixel_start, c->pixel_start);
    cp(contrib_point, c->contrib_point);
    cp(contrib_weight, c->contrib_weight);
    cp(normalizer, c->normalizer);
    cp(fallback_flag, c->fallback_flag);
    cp(nearest_index, c->nearest_index);
}

void ref_cache_free(void* h) { delete static_cast<gmi::ForwardCache*>(h); }

// gmi::backward (engine.cpp:238-309).  upstream: H*W*C doubles.
int ref_backward(const double* pos, const double* col, int n, int channels,
                 const void* cache, const double* upstream, double sigma,
                 double cutoff, int fallback, int workers, double* d_colors,
                 double* d_positions) {
    return guarded([&] {
        const auto* c = static_cast<const gmi::ForwardCache*>(cache);
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        const gmi::InterpConfig cfg =
            make_cfg(sigma, cutoff, fallback, c->width, c->height);
        gmi::ImageBuffer up;
        up.height = c->height;
        up.width = c->width;
        up.channels = channels;
        up.data.assign(upstream, upstream + static_cast<std::size_t>(c->height) *
                                                c->width * channels);
        const gmi::GradientSet g = gmi::backward(ps, cfg, *c, up, workers);
        std::memcpy(d_colors, g.d_colors.data(),
                    g.d_colors.size() * sizeof(double));
        for (int i = 0; i < n; ++i) {
            d_positions[2 * i] = g.d_positions[i].x;
            d_positions[2 * i + 1] = g.d_positions[i].y;
        }
    });
}

// gmi::oracle_forward (oracle.cpp:36-45): untruncated O(N*HW) sum.
int ref_oracle_forward(const double* pos, const double* col, int n,
                       int channels, int width, int height, double sigma,
                       double* image) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        const gmi::ImageBuffer img =
            gmi::oracle_forward(ps, sigma, {width, height});
        std::memcpy(image, img.data.data(), img.data.size() * sizeof(double));
    });
}

// gmi::oracle_gradients_fd (oracle.cpp:59-111).
int ref_oracle_gradients_fd(const double* pos, const double* col, int n,
                            int channels, int width, int height, double sigma,
                            const double* upstream, double step,
                            double* d_colors, double* d_positions) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        gmi::ImageBuffer up;
        up.height = height;
        up.width = width;
        up.channels = channels;
        up.data.assign(upstream,
                       upstream + static_cast<std::size_t>(height) * width *
                                      channels);
        const gmi::GradientSet g =
            gmi::oracle_gradients_fd(ps, sigma, {width, height}, up, step);
        std::memcpy(d_colors, g.d_colors.data(),
                    g.d_colors.size() * sizeof(double));
        for (int i = 0; i < n; ++i) {
            d_positions[2 * i] = g.d_positions[i].x;
            d_positions[2 * i + 1] = g.d_positions[i].y;
        }
    });
}

// gmi::random_instance (validate.cpp:12-35): sizes first (positions/colors
// null), then fill.
int ref_random_instance(std::uint64_t seed, int grid_max, int points_max,
                        int* n, int* channels, int* width, int* height,
                        double* sigma, double* pos, double* col) {
    return guarded([&] {
        const gmi::RandomInstance inst =
            gmi::random_instance(seed, grid_max, points_max);
        *n = inst.points.size();
        *channels = inst.points.channels;
        *width = inst.frame.width;
        *height = inst.frame.height;
        *sigma = inst.sigma;
        if (pos != nullptr) {
            for (int i = 0; i < *n; ++i) {
                pos[2 * i] = inst.points.positions[i].x;
                pos[2 * i + 1] = inst.points.positions[i].y;
            }
        }
        if (col != nullptr) {
            std::memcpy(col, inst.points.colors.data(),
                        inst.points.colors.size() * sizeof(double));
        }
    });
}

// gmi::Rng (rng.hpp:12-59): first k outputs of next_u64 for a seed.
void ref_rng_u64(std::uint64_t seed, int k, std::uint64_t* out) {
    gmi::Rng rng(seed);
    for (int i = 0; i < k; ++i) {
        out[i] = rng.next_u64();
    }
}

// gmi::optimize_points (optimize.cpp:47-98): `steps` rounds of forward -> L1
// loss (l1_loss_and_grad, optimize.cpp:12-28) -> backward -> descent, the bin
// grid rebuilt inside every forward.  Final positions / colours and the loss
// curve (steps + 1 entries) are copied out.
int ref_optimize_points(const double* pos, const double* col, int n, int channels,
                        const double* target, int width, int height, double sigma,
                        double cutoff, int fallback, int steps, double lr, int opt_pos,
                        int opt_col, double* out_pos, double* out_col, double* loss_curve) {
    return guarded([&] {
        const gmi::PointSet ps = make_points(pos, col, n, channels);
        gmi::ImageBuffer tgt = gmi::ImageBuffer::zeros(height, width, channels);
        tgt.data.assign(target, target + static_cast<std::size_t>(height) * width * channels);
        gmi::OptimConfig oc;
        oc.steps = steps;
        oc.learning_rate = lr;
        oc.optimize_positions = opt_pos != 0;
        oc.optimize_colors = opt_col != 0;
        oc.log_every = steps > 0 ? steps : 1;
        const gmi::OptimResult r =
            gmi::optimize_points(ps, tgt, make_cfg(sigma, cutoff, fallback, width, height), oc, 1);
        for (int i = 0; i < n; ++i) {
            out_pos[2 * i] = r.points.positions[i].x;
            out_pos[2 * i + 1] = r.points.positions[i].y;
        }
        std::memcpy(out_col, r.points.colors.data(), sizeof(double) * r.points.colors.size());
        std::memcpy(loss_curve, r.loss_curve.data(), sizeof(double) * r.loss_curve.size());
    });
}

// gmi::run_benchmark (benchmark.cpp:53-120) restricted to the "gmm" method
// for one image and one factor: the row's l1, sigma_used and wall_time_ms.
// sigma <= 0: the auto sweep (auto_sigma_candidates, benchmark.cpp:48-50).
// box != 0: BoxAverage downsampling, else Bicubic (benchmark.cpp:73-80).
int ref_run_benchmark_gmm(const double* image, int width, int height, int channels, int factor,
                          double sigma, int box, double* l1, double* sigma_used, double* ms) {
    return guarded([&] {
        gmi::ImageBuffer img = gmi::ImageBuffer::zeros(height, width, channels);
        img.data.assign(image, image + static_cast<std::size_t>(height) * width * channels);
        gmi::BenchmarkOptions opt;
        opt.factors = {factor};
        opt.methods = {"gmm"};
        if (sigma > 0.0) opt.sigma = sigma;
        opt.downsample = box ? gmi::DownsampleMode::BoxAverage : gmi::DownsampleMode::Bicubic;
        const std::vector<gmi::BenchmarkRow> rows = gmi::run_benchmark({{"img", img}}, opt);
        *l1 = rows.at(0).l1;
        *sigma_used = rows.at(0).sigma_used.value_or(0.0);
        *ms = rows.at(0).wall_time_ms;
    });
}

// gmi::block_mean_downsample (imaging.cpp:343-350) and gmi::l1_metric
// (imaging.cpp:376-386).
int ref_block_mean_downsample(const double* image, int width, int height, int channels,
                              int factor, double* out) {
    return guarded([&] {
        gmi::ImageBuffer img = gmi::ImageBuffer::zeros(height, width, channels);
        img.data.assign(image, image + static_cast<std::size_t>(height) * width * channels);
        const gmi::ImageBuffer low = gmi::block_mean_downsample(img, factor);
        std::memcpy(out, low.data.data(), sizeof(double) * low.data.size());
    });
}

// Point-set and image files (imaging.cpp:235-304, 433-494).
int ref_save_point_set(const double* pos, const double* col, int n, int channels, const char* path) {
    return guarded([&] { gmi::save_point_set(make_points(pos, col, n, channels), path); });
}

// Loads into caller buffers of capacity cap points (n/channels always set).
int ref_load_point_set(const char* path, int cap, int* n, int* channels, double* pos, double* col) {
    return guarded([&] {
        const gmi::PointSet ps = gmi::load_point_set(path);
        *n = ps.size();
        *channels = ps.channels;
        if (ps.size() <= cap) {
            for (int i = 0; i < ps.size(); ++i) {
                pos[2 * i] = ps.positions[i].x;
                pos[2 * i + 1] = ps.positions[i].y;
            }
            std::memcpy(col, ps.colors.data(), sizeof(double) * ps.colors.size());
        }
    });
}

int ref_save_image(const double* img, int height, int width, int channels, const char* path) {
    return guarded([&] {
        gmi::ImageBuffer b = gmi::ImageBuffer::zeros(height, width, channels);
        b.data.assign(img, img + static_cast<std::size_t>(height) * width * channels);
        gmi::save_image(b, path);
    });
}

int ref_load_image(const char* path, long cap, int* height, int* width, int* channels, double* out) {
    return guarded([&] {
        const gmi::ImageBuffer b = gmi::load_image(path);
        *height = b.height;
        *width = b.width;
        *channels = b.channels;
        if (static_cast<long>(b.data.size()) <= cap)
            std::memcpy(out, b.data.data(), sizeof(double) * b.data.size());
    });
}

}  // extern "C"
