// gmi_b200/gmi.hpp — the reference's C++ API (namespace gmi) re-implemented on
// the B200 C-ABI (include/gmi_b200.h).  Source-compatible with
// /root/reference/proj/include/gmi/{core,engine,bin_grid}.hpp for the hot path:
// callers such as cmd_forward (tools/gmi_main.cpp:61-74), optimize_points
// (src/optimize.cpp:60-79) and the pybind module (python/bindings.cpp:147-184)
// compile against it unchanged and link libgmi_b200_cxx.so instead of
// engine.cpp/bin_grid.cpp.
//
// Differences (documented in INTEGRATION.md): the device path computes in fp32
// (inputs are rounded to float; results within rel 1e-5 / abs 1e-6 of the
// reference, binning / neighbour sets / fallback choices exact for
// fp32-representable inputs); C >= 1 channels (reference: 1 or 3);
// ForwardCache keeps W, the fallback data and a device-resident copy of the
// inputs instead of the per-pixel contribution CSR (weights are recomputed).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

struct gmi_cache;
struct gmi_ctx;

namespace gmi {

struct Vec2 {
    double x = 0.0;
    double y = 0.0;
};

inline Vec2 operator+(Vec2 a, Vec2 b) { return {a.x + b.x, a.y + b.y}; }
inline Vec2 operator-(Vec2 a, Vec2 b) { return {a.x - b.x, a.y - b.y}; }
inline Vec2 operator*(double s, Vec2 v) { return {s * v.x, s * v.y}; }
inline double squared_norm(Vec2 v) { return v.x * v.x + v.y * v.y; }

struct CoordinateFrame {  // core.hpp:25-30
    int width = 0;
    int height = 0;
};

enum class Fallback { NearestPoint, Zero };  // core.hpp:32-33

enum class ErrorCode {  // core.hpp:35-50 (same order and values)
    NonFiniteValue,
    ColorOutOfRange,
    EmptyPointSet,
    ShapeMismatch,
    InvalidCellSize,
    ConfigInvalid,
    CacheMismatch,
    InvalidDimensions,
    InvalidFactor,
    InvalidCount,
    UnsupportedFormat,
    CorruptFile,
    EmptyLog,
    IoError,
};

const char* error_code_name(ErrorCode code);

class Error : public std::runtime_error {  // core.hpp:54-62
public:
    Error(ErrorCode code, const std::string& message)
        : std::runtime_error(message), code_(code) {}
    ErrorCode code() const { return code_; }

private:
    ErrorCode code_;
};

// Failure of the device path itself (no reference equivalent).
class DeviceError : public std::runtime_error {
public:
    DeviceError(int status, const std::string& message)
        : std::runtime_error(message), status_(status) {}
    int status() const { return status_; }

private:
    int status_;
};

struct PointSet {  // core.hpp:64-79
    std::vector<Vec2> positions;
    std::vector<double> colors;
    int channels = 1;

    int size() const { return static_cast<int>(positions.size()); }
    double color(int i, int ch) const {
        return colors[static_cast<std::size_t>(i) * channels + ch];
    }
    double& color(int i, int ch) {
        return colors[static_cast<std::size_t>(i) * channels + ch];
    }
};

struct InterpConfig {  // core.hpp:81-88
    double sigma = 1.0;
    double cutoff_radius = 3.0;
    Fallback fallback = Fallback::NearestPoint;
    CoordinateFrame frame;
};

inline InterpConfig make_config(double sigma, CoordinateFrame frame,
                                Fallback fallback = Fallback::NearestPoint) {
    return InterpConfig{sigma, 3.0 * sigma, fallback, frame};  // core.hpp:90-94
}

struct ImageBuffer {  // core.hpp:96-117
    int height = 0;
    int width = 0;
    int channels = 0;
    std::vector<double> data;

    static ImageBuffer zeros(int height, int width, int channels);
    std::size_t index(int r, int c, int ch) const {
        return (static_cast<std::size_t>(r) * width + c) * channels + ch;
    }
    double at(int r, int c, int ch) const { return data[index(r, c, ch)]; }
    double& at(int r, int c, int ch) { return data[index(r, c, ch)]; }
    CoordinateFrame frame() const { return {width, height}; }
    bool same_shape(const ImageBuffer& o) const {
        return height == o.height && width == o.width && channels == o.channels;
    }
};

struct GradientSet {  // core.hpp:119-131
    std::vector<double> d_colors;
    std::vector<Vec2> d_positions;
    int channels = 1;

    static GradientSet zeros(int num_points, int channels);
    double d_color(int i, int ch) const {
        return d_colors[static_cast<std::size_t>(i) * channels + ch];
    }
};

double gaussian_weight(const Vec2& q, const Vec2& mu, double sigma);  // core.cpp:49-53

struct ValidationIssue {  // core.hpp:138-142
    ErrorCode code;
    int index;  // offending point, -1 when not point-specific
    std::string message;
};

// core.hpp:144-149 (core.cpp:55-120), with C >= 1 channels accepted (the
// device path's contract) instead of C in {1, 3}
std::optional<ValidationIssue> validate_point_set(const PointSet& ps);
void require_valid(const PointSet& ps);  // throws Error on violation
void require_valid(const InterpConfig& cfg);
void require_frame(const CoordinateFrame& frame);

// The device path computes on fp32 inputs.  Positions / colours that are not
// exactly representable in fp32 are rounded to nearest (the reference would
// see the unrounded f64 values).  Allow (default) rounds and records the
// number of rounded values in ForwardCache::inexact_inputs; Reject throws
// DeviceError(GMI_ERR_INVALID_ARGUMENT) naming the first such value, for
// callers that need the reference's bit-exact binning / neighbour decisions.
enum class Fp32Inputs { Allow, Reject };
void set_fp32_inputs(Fp32Inputs policy);  // this thread's calls
// Number of positions + colours of `ps` that fp32 cannot hold exactly.
std::int64_t count_inexact_fp32(const PointSet& ps);

// ForwardCache (engine.hpp:20-41): metadata + per-pixel normaliser, fallback
// flags and nearest indices, output copy; the device state (binned points,
// W) backs backward().
struct ForwardCache {
    int width = 0;
    int height = 0;
    int channels = 0;
    int num_points = 0;
    double sigma = 0.0;
    double cutoff_radius = 0.0;
    Fallback fallback = Fallback::NearestPoint;

    std::vector<double> normalizer;
    std::vector<std::uint8_t> fallback_flag;
    std::vector<int> nearest_index;
    std::vector<double> output;

    std::int64_t num_pixels() const { return static_cast<std::int64_t>(width) * height; }
    int fallback_count() const;
    // pixel_start deltas (engine.hpp:29-31), recomputed on the device
    std::vector<std::int32_t> contribution_counts() const;
    // positions + colours rounded to fp32 by this forward (Fp32Inputs)
    std::int64_t inexact_inputs = 0;

    std::shared_ptr<gmi_cache> device;  // owned device state
};

struct ForwardResult {  // engine.hpp:43-46
    ImageBuffer image;
    ForwardCache cache;
};

// engine.hpp:48-55 — num_workers is accepted for source compatibility
ForwardResult forward(const PointSet& ps, const InterpConfig& cfg,
                      const CoordinateFrame& out_frame, int num_workers = 1);
ForwardResult forward(const PointSet& ps, const InterpConfig& cfg, int num_workers = 1);

// engine.hpp:57-64
GradientSet backward(const PointSet& ps, const InterpConfig& cfg, const ForwardCache& cache,
                     const ImageBuffer& upstream, int num_workers = 1);

// bin_grid.hpp:17-31 — bit-exact build_bin_grid on the GPU
struct BinGrid {
    double cell_size = 1.0;
    Vec2 origin;
    int n_cols = 1;
    int n_rows = 1;
    std::vector<int> bin_start;
    std::vector<int> point_index;
    int num_cells() const { return n_cols * n_rows; }
};
BinGrid build_bin_grid(const PointSet& ps, double cell_size);

// Device selection for this thread's calls (default: device 0).
void set_device(int device);

// This thread's calls in reference-grade precision (GMI_CTX_PRECISE: f64
// weights, sums and image on the device; slower).  Default off: the fp32 hot
// path, within rel 1e-5 / abs 1e-6 of the reference on the BASELINE configs.
void set_precise(bool on);

}  // namespace gmi
