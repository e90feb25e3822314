// Drop-in check of the reference-shaped C++ API (include/gmi_b200/gmi.hpp):
// restated reference unit tests (test_engine.cpp, test_bin_grid.cpp) compiled
// against libgmi_b200_cxx.so.  Exit code 0 = all pass.  Needs a GPU.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gmi_b200/gmi.hpp"

using namespace gmi;

static int failures = 0;
#define CHECK(cond)                                                         \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                     \
        }                                                                   \
    } while (0)

static bool close(double a, double b, double rel) {
    return std::fabs(a - b) <= rel * std::fmax(std::fabs(a), std::fabs(b)) + 1e-12;
}

int main() {
    // test_engine.cpp:53-70 three-point mixture
    {
        PointSet ps;
        ps.channels = 1;
        ps.positions = {{-0.5, -0.5}, {1.5, -0.5}, {-0.5, 1.5}};
        ps.colors = {1.0, 0.0, 0.0};
        InterpConfig cfg{1.0, 10.0, Fallback::NearestPoint, {1, 1}};
        const ForwardResult r = forward(ps, cfg, {1, 1});
        CHECK(close(r.image.at(0, 0, 0), 0.5761168847658291, 1e-6));
    }
    // test_engine.cpp:217-239 fallback policies
    {
        PointSet ps;
        ps.channels = 1;
        ps.positions = {{100, 100}, {200, 200}};
        ps.colors = {0.9, 0.1};
        const auto fn = forward(ps, InterpConfig{1.0, 2.0, Fallback::NearestPoint, {}}, {4, 4});
        CHECK(fn.cache.fallback_count() == 16);
        for (double v : fn.image.data) CHECK(v == static_cast<double>(0.9f));
        const auto fz = forward(ps, InterpConfig{1.0, 2.0, Fallback::Zero, {}}, {4, 4});
        for (double v : fz.image.data) CHECK(v == 0.0);
    }
    // test_engine.cpp:302-311 backward single point unit upstream
    {
        PointSet ps;
        ps.channels = 1;
        ps.positions = {{2, 2}};
        ps.colors = {0.5};
        const InterpConfig cfg{1.0, 100.0, Fallback::NearestPoint, {6, 5}};
        const auto f = forward(ps, cfg, {6, 5});
        ImageBuffer up = ImageBuffer::zeros(5, 6, 1);
        for (double& v : up.data) v = 1.0;
        const GradientSet g = backward(ps, cfg, f.cache, up);
        CHECK(close(g.d_colors[0], 30.0, 1e-6));
        CHECK(std::fabs(g.d_positions[0].x) < 1e-6 && std::fabs(g.d_positions[0].y) < 1e-6);
        // test_engine.cpp:372-400 CacheMismatch
        InterpConfig other = cfg;
        other.sigma = 2.0;
        bool threw = false;
        try {
            backward(ps, other, f.cache, up);
        } catch (const Error& e) {
            threw = e.code() == ErrorCode::CacheMismatch;
        }
        CHECK(threw);
    }
    // core.cpp:55-96 validation through the device path
    {
        PointSet ps;
        ps.channels = 1;
        ps.positions = {{0, 0}, {1, 1}};
        ps.colors = {0.5, 1.5};
        bool threw = false;
        try {
            forward(ps, make_config(1.0, {2, 2}));
        } catch (const Error& e) {
            threw = e.code() == ErrorCode::ColorOutOfRange;
        }
        CHECK(threw);
    }
    // test_bin_grid.cpp:40-86 conservation + exact reference geometry
    {
        PointSet ps;
        ps.channels = 1;
        for (int i = 0; i < 1000; ++i) {
            ps.positions.push_back({static_cast<float>((i * 37) % 64 + 0.25), static_cast<float>((i * 11) % 64 + 0.5)});
            ps.colors.push_back(0.5);
        }
        const BinGrid g = build_bin_grid(ps, 4.0);
        CHECK(g.bin_start.back() == 1000);
        CHECK(g.point_index.size() == 1000);
        CHECK(g.origin.x == 0.25 - 4.0 && g.origin.y == 0.5 - 4.0);
        for (int b = 0; b < g.num_cells(); ++b)
            for (int k = g.bin_start[b] + 1; k < g.bin_start[b + 1]; ++k)
                CHECK(g.point_index[k - 1] < g.point_index[k]);  // ascending in a bin
    }
    std::printf("%s (%d failures)\n", failures == 0 ? "cxx api ok" : "cxx api FAILED", failures);
    return failures == 0 ? 0 : 1;
}
