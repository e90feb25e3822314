// The reference's C++ API (include/gmi_b200/gmi.hpp) layered on the C-ABI:
// f64 value types in, fp32 device path, f64 value types out; gmi::Error with
// the reference's ErrorCode on every validation failure.
#include "gmi_b200/gmi.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "gmi_b200.h"

namespace gmi {

namespace {

thread_local int t_device = 0;
thread_local Fp32Inputs t_fp32 = Fp32Inputs::Allow;
thread_local bool t_precise = false;

struct CtxDeleter {
    void operator()(gmi_ctx* c) const { gmi_ctx_destroy(c); }
};

gmi_ctx* thread_ctx() {
    thread_local std::unique_ptr<gmi_ctx, CtxDeleter> ctx;
    thread_local int ctx_device = -1;
    if (!ctx || ctx_device != t_device) {
        gmi_ctx* c = nullptr;
        const int rc = gmi_ctx_create(t_device, &c);
        if (rc != GMI_OK) throw DeviceError(rc, gmi_last_error());
        ctx.reset(c);
        ctx_device = t_device;
    }
    gmi_ctx_set_flags(ctx.get(), t_precise ? GMI_CTX_PRECISE : 0u);
    return ctx.get();
}

[[noreturn]] void raise(int rc) {
    const std::string msg = gmi_last_error();
    if (rc >= 1 && rc <= 14) throw Error(static_cast<ErrorCode>(rc - 1), msg);
    throw DeviceError(rc, msg);
}

void check(int rc) {
    if (rc != GMI_OK) raise(rc);
}

gmi_config to_cfg(const InterpConfig& cfg, const CoordinateFrame& frame) {
    gmi_config c{};
    c.sigma = cfg.sigma;
    c.cutoff_radius = cfg.cutoff_radius;
    c.fallback = cfg.fallback == Fallback::NearestPoint ? GMI_FALLBACK_NEAREST : GMI_FALLBACK_ZERO;
    c.width = frame.width;
    c.height = frame.height;
    return c;
}

bool inexact(double v) {
    // NaN / inf go to the device's own validation (the reference's codes)
    return std::isfinite(v) && static_cast<double>(static_cast<float>(v)) != v;
}

// Rounds the f64 inputs to the device's fp32; returns how many changed value
// (Fp32Inputs::Reject: throws on the first).
std::int64_t to_f32(const PointSet& ps, std::vector<float>& pos, std::vector<float>& col) {
    std::int64_t rounded = 0;
    auto reject = [&](const char* what, std::size_t i, double v) {
        if (t_fp32 == Fp32Inputs::Reject) {
            char buf[160];
            std::snprintf(buf, sizeof(buf), "%s %.17g at index %zu is not representable in fp32",
                          what, v, i);
            throw DeviceError(GMI_ERR_INVALID_ARGUMENT, buf);
        }
        ++rounded;
    };
    pos.resize(static_cast<std::size_t>(ps.size()) * 2);
    for (int i = 0; i < ps.size(); ++i) {
        const Vec2 p = ps.positions[i];
        if (inexact(p.x)) reject("position x", i, p.x);
        if (inexact(p.y)) reject("position y", i, p.y);
        pos[2 * i] = static_cast<float>(p.x);
        pos[2 * i + 1] = static_cast<float>(p.y);
    }
    col.resize(ps.colors.size());
    for (std::size_t k = 0; k < ps.colors.size(); ++k) {
        if (inexact(ps.colors[k])) reject("color", k / std::max(ps.channels, 1), ps.colors[k]);
        col[k] = static_cast<float>(ps.colors[k]);
    }
    return rounded;
}

// core.cpp:55-66 shape checks (C relaxed to >= 1); value checks run on the
// device and come back with the reference's codes.
void check_shape(const PointSet& ps) {
    if (ps.positions.empty()) throw Error(ErrorCode::EmptyPointSet, "point set is empty");
    if (ps.channels < 1)
        throw Error(ErrorCode::ShapeMismatch, "channels must be >= 1, got " + std::to_string(ps.channels));
    const std::size_t expected = ps.positions.size() * static_cast<std::size_t>(ps.channels);
    if (ps.colors.size() != expected)
        throw Error(ErrorCode::ShapeMismatch, "colors holds " + std::to_string(ps.colors.size()) +
                                                  " values, expected " + std::to_string(expected));
}

}  // namespace

const char* error_code_name(ErrorCode code) { return gmi_error_name(static_cast<int>(code) + 1); }

void set_device(int device) { t_device = device; }

void set_fp32_inputs(Fp32Inputs policy) { t_fp32 = policy; }

void set_precise(bool on) { t_precise = on; }

std::int64_t count_inexact_fp32(const PointSet& ps) {
    std::int64_t n = 0;
    for (const Vec2& p : ps.positions) n += inexact(p.x) + inexact(p.y);
    for (double c : ps.colors) n += inexact(c);
    return n;
}

// core.cpp:55-96 (C >= 1)
std::optional<ValidationIssue> validate_point_set(const PointSet& ps) {
    if (ps.positions.empty()) return ValidationIssue{ErrorCode::EmptyPointSet, -1, "point set is empty"};
    if (ps.channels < 1)
        return ValidationIssue{ErrorCode::ShapeMismatch, -1,
                               "channels must be >= 1, got " + std::to_string(ps.channels)};
    const std::size_t expected = ps.positions.size() * static_cast<std::size_t>(ps.channels);
    if (ps.colors.size() != expected)
        return ValidationIssue{ErrorCode::ShapeMismatch, -1,
                               "colors holds " + std::to_string(ps.colors.size()) +
                                   " values, expected " + std::to_string(expected)};
    for (int i = 0; i < ps.size(); ++i) {
        const Vec2 p = ps.positions[i];
        if (!std::isfinite(p.x) || !std::isfinite(p.y))
            return ValidationIssue{ErrorCode::NonFiniteValue, i,
                                   "non-finite position at index " + std::to_string(i)};
        for (int ch = 0; ch < ps.channels; ++ch) {
            const double c = ps.color(i, ch);
            if (!std::isfinite(c))
                return ValidationIssue{ErrorCode::NonFiniteValue, i,
                                       "non-finite color at index " + std::to_string(i)};
            if (c < 0.0 || c > 1.0)
                return ValidationIssue{ErrorCode::ColorOutOfRange, i,
                                       "color " + std::to_string(c) + " out of [0,1] at index " +
                                           std::to_string(i)};
        }
    }
    return std::nullopt;
}

void require_valid(const PointSet& ps) {
    if (auto issue = validate_point_set(ps)) throw Error(issue->code, issue->message);
}

// core.cpp:104-113
void require_valid(const InterpConfig& cfg) {
    if (!std::isfinite(cfg.sigma) || cfg.sigma <= 0.0)
        throw Error(ErrorCode::ConfigInvalid, "sigma must be positive and finite");
    if (!std::isfinite(cfg.cutoff_radius) || cfg.cutoff_radius <= 0.0)
        throw Error(ErrorCode::ConfigInvalid, "cutoff_radius must be positive and finite");
}

// core.cpp:115-120
void require_frame(const CoordinateFrame& frame) {
    if (frame.width < 1 || frame.height < 1)
        throw Error(ErrorCode::InvalidDimensions, "frame dimensions must be at least 1x1");
}

ImageBuffer ImageBuffer::zeros(int height, int width, int channels) {
    if (height < 1 || width < 1 || channels < 1)
        throw Error(ErrorCode::InvalidDimensions, "image dimensions must be positive");
    ImageBuffer img;
    img.height = height;
    img.width = width;
    img.channels = channels;
    img.data.assign(static_cast<std::size_t>(height) * width * channels, 0.0);
    return img;
}

GradientSet GradientSet::zeros(int num_points, int channels) {
    GradientSet g;
    g.channels = channels;
    g.d_colors.assign(static_cast<std::size_t>(num_points) * channels, 0.0);
    g.d_positions.assign(static_cast<std::size_t>(num_points), Vec2{});
    return g;
}

double gaussian_weight(const Vec2& q, const Vec2& mu, double sigma) {
    return gmi_gaussian_weight(q.x, q.y, mu.x, mu.y, sigma);
}

int ForwardCache::fallback_count() const {
    int n = 0;
    for (std::uint8_t f : fallback_flag) n += f;
    return n;
}

std::vector<std::int32_t> ForwardCache::contribution_counts() const {
    std::vector<std::int32_t> counts(static_cast<std::size_t>(num_pixels()));
    if (device) check(gmi_forward_counts(thread_ctx(), device.get(), counts.data()));
    return counts;
}

ForwardResult forward(const PointSet& ps, const InterpConfig& cfg,
                      const CoordinateFrame& out_frame, int /*num_workers*/) {
    check_shape(ps);
    const gmi_config c = to_cfg(cfg, out_frame);
    std::vector<float> pos, col;
    const std::int64_t rounded = to_f32(ps, pos, col);
    std::vector<float> img(static_cast<std::size_t>(std::max(out_frame.width, 0)) *
                           std::max(out_frame.height, 0) * ps.channels);
    gmi_cache* h = nullptr;
    check(gmi_forward_host(thread_ctx(), pos.data(), col.data(), 1, ps.size(), ps.channels, &c,
                           img.data(), &h));
    ForwardResult r;
    r.image = ImageBuffer::zeros(out_frame.height, out_frame.width, ps.channels);
    for (std::size_t k = 0; k < img.size(); ++k) r.image.data[k] = img[k];
    ForwardCache& fc = r.cache;
    fc.device = std::shared_ptr<gmi_cache>(h, [](gmi_cache* p) { gmi_cache_free(p); });
    fc.width = out_frame.width;
    fc.height = out_frame.height;
    fc.channels = ps.channels;
    fc.num_points = ps.size();
    fc.sigma = cfg.sigma;
    fc.cutoff_radius = cfg.cutoff_radius;
    fc.fallback = cfg.fallback;
    fc.inexact_inputs = rounded;
    const std::size_t hw = static_cast<std::size_t>(fc.num_pixels());
    std::vector<float> norm(hw);
    fc.fallback_flag.resize(hw);
    fc.nearest_index.resize(hw);
    check(gmi_cache_copy_pixels(h, norm.data(), fc.fallback_flag.data(), fc.nearest_index.data()));
    fc.normalizer.assign(norm.begin(), norm.end());
    fc.output = r.image.data;
    return r;
}

ForwardResult forward(const PointSet& ps, const InterpConfig& cfg, int num_workers) {
    return forward(ps, cfg, cfg.frame, num_workers);
}

GradientSet backward(const PointSet& ps, const InterpConfig& cfg, const ForwardCache& cache,
                     const ImageBuffer& upstream, int /*num_workers*/) {
    check_shape(ps);
    // engine.cpp:243-250: exact == checks
    if (cache.num_points != ps.size() || cache.channels != ps.channels ||
        cache.width != upstream.width || cache.height != upstream.height ||
        cache.channels != upstream.channels || cache.sigma != cfg.sigma ||
        cache.cutoff_radius != cfg.cutoff_radius || cache.fallback != cfg.fallback ||
        !cache.device)
        throw Error(ErrorCode::CacheMismatch, "forward cache does not match the given inputs");
    const gmi_config c = to_cfg(cfg, {cache.width, cache.height});
    std::vector<float> pos, col;
    to_f32(ps, pos, col);
    std::vector<float> up(upstream.data.begin(), upstream.data.end());
    std::vector<float> dc(static_cast<std::size_t>(ps.size()) * ps.channels);
    std::vector<float> dp(static_cast<std::size_t>(ps.size()) * 2);
    check(gmi_backward_host(thread_ctx(), pos.data(), col.data(), 1, ps.size(), ps.channels, &c,
                            cache.device.get(), up.data(), dc.data(), dp.data()));
    GradientSet g = GradientSet::zeros(ps.size(), ps.channels);
    for (std::size_t k = 0; k < dc.size(); ++k) g.d_colors[k] = dc[k];
    for (int i = 0; i < ps.size(); ++i) g.d_positions[i] = {dp[2 * i], dp[2 * i + 1]};
    return g;
}

BinGrid build_bin_grid(const PointSet& ps, double cell_size) {
    check_shape(ps);
    std::vector<float> pos, col;
    to_f32(ps, pos, col);
    double origin[2];
    int32_t nc = 0, nr = 0;
    gmi_ctx* ctx = thread_ctx();
    check(gmi_bin_grid_host(ctx, pos.data(), 1, ps.size(), cell_size, origin, &nc, &nr, nullptr,
                            nullptr));
    BinGrid g;
    g.cell_size = cell_size;
    g.origin = {origin[0], origin[1]};
    g.n_cols = nc;
    g.n_rows = nr;
    g.bin_start.resize(static_cast<std::size_t>(nc) * nr + 1);
    g.point_index.resize(ps.size());
    check(gmi_bin_grid_host(ctx, pos.data(), 1, ps.size(), cell_size, origin, &nc, &nr,
                            g.bin_start.data(), g.point_index.data()));
    return g;
}

}  // namespace gmi
