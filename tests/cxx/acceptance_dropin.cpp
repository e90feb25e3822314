// Drop-in proof on the reference's own callers (VERDICT r1 "what's missing"
// 5): this driver and the UNMODIFIED reference sources oracle.cpp,
// validate.cpp, optimize.cpp and imaging.cpp are compiled against
// include/gmi_dropin (gmi/core.hpp, gmi/engine.hpp -> gmi_b200/gmi.hpp) and
// linked with libgmi_b200_cxx.so — the reference's engine.cpp / bin_grid.cpp
// / core.cpp are NOT linked, so every forward()/backward() below, including
// the ones inside the reference's optimize_points, runs on the B200 path.
//
// The acceptance criteria of /root/reference/proj/tests/acceptance.cpp that
// exercise the hot path (1, 3, 4, 5; lines 68-232), with the reference's
// seeds (0xACCE2026, 0xBEEF2026, 0xD00D2026) and instance families, at the
// device path's fp32 tolerance |a-b| <= 1e-6 + 1e-5 max(|a|,|b|) instead of
// the f64 engine's 1e-12.  Instances are rounded to fp32 first (both sides
// then see identical inputs; gmi::count_inexact_fp32 == 0 is asserted).
// Criterion 4's ForwardCache CSR is not kept by the device path (weights are
// recomputed), so partition of unity is checked through the backward: a unit
// upstream gives sum_i d_colors[i, ch] = sum_pixels sum_i w_i/W = H*W.
//
// Exit code 0 = every criterion passed.  Needs a GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gmi/engine.hpp"
#include "gmi/optimize.hpp"
#include "gmi/oracle.hpp"
#include "gmi/rng.hpp"
#include "gmi/validate.hpp"

using namespace gmi;

namespace {

constexpr std::uint64_t kForwardSeed = 0xACCE2026ULL;      // acceptance.cpp:45
constexpr std::uint64_t kGradientSeed = 0xBEEF2026ULL;     // acceptance.cpp:46
constexpr std::uint64_t kDeterminismSeed = 0xD00D2026ULL;  // acceptance.cpp:47
constexpr double kRel = 1e-5, kAbs = 1e-6;                 // north-star tolerance

double excess(double a, double b) {
    return std::fabs(a - b) / (kAbs + kRel * std::max(std::fabs(a), std::fabs(b)));
}

void round_fp32(RandomInstance& inst) {
    for (Vec2& p : inst.points.positions) {
        p.x = static_cast<float>(p.x);
        p.y = static_cast<float>(p.y);
    }
    for (double& c : inst.points.colors) c = static_cast<float>(c);
}

std::vector<RandomInstance> forward_family() {  // acceptance.cpp:59-66
    std::vector<RandomInstance> out;
    Rng master(kForwardSeed);
    for (int k = 0; k < 100; ++k) {
        out.push_back(random_instance(master.next_u64(), 16, 50));
        round_fp32(out.back());
    }
    return out;
}

struct Result {
    int id;
    bool passed;
    std::string detail;
};

// acceptance.cpp:68-86: untruncated forward == oracle
Result criterion_1() {
    double worst = 0.0;
    bool exact_inputs = true;
    for (const RandomInstance& inst : forward_family()) {
        exact_inputs &= count_inexact_fp32(inst.points) == 0;
        const InterpConfig cfg{inst.sigma, untruncated_radius(inst), Fallback::NearestPoint,
                               inst.frame};
        const ForwardResult fwd = forward(inst.points, cfg, inst.frame);
        const ImageBuffer ref = oracle_forward(inst.points, inst.sigma, inst.frame);
        for (std::size_t k = 0; k < ref.data.size(); ++k)
            worst = std::max(worst, excess(fwd.image.data[k], ref.data[k]));
        exact_inputs &= fwd.cache.inexact_inputs == 0;
    }
    char buf[160];
    std::snprintf(buf, sizeof(buf), "worst %.3f x tolerance over 100 instances (oracle_forward)", worst);
    return {1, worst <= 1.0 && exact_inputs, buf};
}

// acceptance.cpp:122-148: analytic gradients vs central finite differences
Result criterion_3() {
    bool passed = true;
    double worst_ref = 0.0;
    Rng master(kGradientSeed);
    for (int k = 0; k < 100; ++k) {
        RandomInstance inst = random_instance(master.next_u64(), 8, 20);
        round_fp32(inst);
        Rng aux(inst.seed ^ 0xABCDEFULL);
        ImageBuffer upstream = random_upstream(aux, inst.frame, inst.points.channels);
        for (double& u : upstream.data) u = static_cast<float>(u);
        const InterpConfig cfg{inst.sigma, untruncated_radius(inst), Fallback::NearestPoint,
                               inst.frame};
        const ForwardResult fwd = forward(inst.points, cfg, inst.frame);
        const GradientSet analytic = backward(inst.points, cfg, fwd.cache, upstream);
        const GradientSet fd = oracle_gradients_fd(inst.points, inst.sigma, inst.frame, upstream, 1e-5);
        // the reference's comparator (validate.cpp:72-94) at the north-star
        // tolerance; its worst relative error is reported beside it
        const GradientCheck check = compare_gradients(analytic, fd, kRel, kAbs);
        passed = passed && check.passed;
        worst_ref = std::max(worst_ref, check.worst_rel);
    }
    char buf[160];
    std::snprintf(buf, sizeof(buf), "worst rel err %.3e over 100 instances (compare_gradients %g / %g)",
                  worst_ref, kRel, kAbs);
    return {3, passed, buf};
}

// acceptance.cpp:150-197: partition of unity and constant-colour invariance
Result criterion_4() {
    double worst_unity = 0.0, worst_const = 0.0;
    for (const RandomInstance& inst : forward_family()) {
        const InterpConfig cfg = make_config(inst.sigma, inst.frame);
        const ForwardResult fwd = forward(inst.points, cfg, inst.frame);
        ImageBuffer ones = ImageBuffer::zeros(inst.frame.height, inst.frame.width,
                                              inst.points.channels);
        std::fill(ones.data.begin(), ones.data.end(), 1.0);
        const GradientSet g = backward(inst.points, cfg, fwd.cache, ones);
        const double hw = static_cast<double>(fwd.cache.num_pixels());
        for (int ch = 0; ch < inst.points.channels; ++ch) {
            double s = 0.0;
            for (int i = 0; i < inst.points.size(); ++i) s += g.d_color(i, ch);
            worst_unity = std::max(worst_unity, std::fabs(s - hw) / hw);
        }
        PointSet constant = inst.points;
        const double kappa = 0.4375;
        for (double& c : constant.colors) c = kappa;
        const ForwardResult flat = forward(constant, cfg, inst.frame);
        for (std::int64_t pix = 0; pix < flat.cache.num_pixels(); ++pix) {
            for (int ch = 0; ch < constant.channels; ++ch)
                worst_const = std::max(worst_const,
                                       std::fabs(flat.image.data[pix * constant.channels + ch] - kappa));
        }
    }
    char buf[160];
    std::snprintf(buf, sizeof(buf), "worst |sum w/W - 1| %.3e, worst constant deviation %.3e",
                  worst_unity, worst_const);
    return {4, worst_unity <= kRel && worst_const <= kAbs, buf};
}

// acceptance.cpp:199-232: bit-identical results with 1/2/4/8 workers (and
// across repeated calls on the device)
Result criterion_5() {
    bool passed = true;
    Rng master(kDeterminismSeed);
    for (int k = 0; k < 20; ++k) {
        RandomInstance inst = random_instance(master.next_u64(), 16, 50);
        round_fp32(inst);
        Rng aux(inst.seed ^ 0x777ULL);
        const ImageBuffer upstream = random_upstream(aux, inst.frame, inst.points.channels);
        const InterpConfig cfg = make_config(inst.sigma, inst.frame);
        const ForwardResult base = forward(inst.points, cfg, inst.frame, 1);
        const GradientSet base_grad = backward(inst.points, cfg, base.cache, upstream, 1);
        for (int workers : {2, 4, 8}) {
            const ForwardResult fwd = forward(inst.points, cfg, inst.frame, workers);
            const GradientSet grad = backward(inst.points, cfg, fwd.cache, upstream, workers);
            passed = passed && fwd.image.data == base.image.data &&
                     grad.d_colors == base_grad.d_colors;
            for (std::size_t i = 0; i < grad.d_positions.size(); ++i)
                passed = passed && grad.d_positions[i].x == base_grad.d_positions[i].x &&
                         grad.d_positions[i].y == base_grad.d_positions[i].y;
        }
    }
    return {5, passed, "20 instances, forward + backward"};
}

// The reference's own optimize_points (optimize.cpp:47-98, compiled
// unmodified) driving the B200 forward/backward: the loss must fall.
Result optimize_caller() {
    Rng rng(424242u);  // acceptance.cpp:49 kOptimSeed
    const int w = 24, h = 20;
    ImageBuffer target = ImageBuffer::zeros(h, w, 1);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) target.at(r, c, 0) = (c > w / 2) ? 0.9 : 0.1;
    PointSet ps;
    ps.channels = 1;
    for (int i = 0; i < 80; ++i) {
        ps.positions.push_back({static_cast<float>(rng.uniform(-0.5, w - 0.5)),
                                static_cast<float>(rng.uniform(-0.5, h - 0.5))});
        ps.colors.push_back(static_cast<float>(rng.next_double()));
    }
    OptimConfig oc;
    oc.steps = 40;
    oc.learning_rate = 0.5;
    oc.optimize_positions = true;
    oc.optimize_colors = true;
    const OptimResult r = optimize_points(ps, target, make_config(1.0, {w, h}), oc);
    const double first = r.loss_curve.front(), last = r.loss_curve.back();
    char buf[160];
    std::snprintf(buf, sizeof(buf), "optimize_points (reference loop): L1 %.5f -> %.5f in %d steps",
                  first, last, oc.steps);
    return {8, std::isfinite(last) && last < first, buf};
}

}  // namespace

int main() {
    std::vector<Result> results;
    for (auto fn : {criterion_1, criterion_3, criterion_4, criterion_5, optimize_caller}) {
        const auto t0 = std::chrono::steady_clock::now();
        Result r = fn();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("[%s] %s %d: %s (%.2f s)\n", r.passed ? "PASS" : "FAIL",
                    r.id == 8 ? "caller" : "criterion", r.id, r.detail.c_str(), s);
        results.push_back(r);
    }
    int failures = 0;
    for (const Result& r : results) failures += r.passed ? 0 : 1;
    std::printf("%d/%zu passed\n", static_cast<int>(results.size()) - failures, results.size());
    return failures == 0 ? 0 : 1;
}
