// carve/bench.hpp — drop-in for the reference's fixture and timers
// (/root/reference/proj/include/carve/bench.hpp:67-201). make_test_image is
// the host generator (byte-identical to the reference's); the timers measure
// host PixelGrid in -> host PixelGrid out through the B200 engine, min over reps.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>

#include "carve/carver.hpp"

namespace carve {

inline PixelGrid make_test_image(int width, int height) {
    PixelGrid img(width, height);
    detail::check(carve_make_test_image(width, height, 0, img.bytes()));
    return img;
}

/// make_test_image with the C5 batch variant seed (variant 0 = reference fixture).
inline PixelGrid make_test_image_variant(int width, int height, uint32_t variant) {
    PixelGrid img(width, height);
    detail::check(carve_make_test_image(width, height, variant, img.bytes()));
    return img;
}

struct TimedResult {
    double wall_time_s = 0.0;  // minimum over repetitions
    int repetitions = 1;
};

/// bench.hpp:140-174 — energy outside the timed region, find_seam timed.
inline TimedResult time_single_seam(const PixelGrid& grid, const CarveConfig& cfg, int reps) {
    if (reps < 1) fail(Errc::usage_error, "reps must be >= 1");
    detail::check_config(cfg);
    const EnergyMap e = energy_e1(grid);
    double best = std::numeric_limits<double>::infinity();
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        volatile int sink = find_seam(e, cfg.solver, cfg.solver_opts).back();
        (void)sink;
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    return {std::max(best, 1e-9), reps};
}

/// bench.hpp:177-201 — carve_to_width(grid, round(scale*width)) end to end.
inline TimedResult time_full_carve(const PixelGrid& grid, double scale, const CarveConfig& cfg, int reps) {
    if (reps < 1) fail(Errc::usage_error, "reps must be >= 1");
    if (!(scale > 0.0) || scale > 1.0) fail(Errc::usage_error, "scale must be in (0, 1]");
    const int target = int(std::lround(scale * grid.width));
    double best = std::numeric_limits<double>::infinity();
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        auto res = carve_to_width(grid, target, cfg);
        volatile int sink = res.first.width;
        (void)sink;
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    return {std::max(best, 1e-9), reps};
}

} // namespace carve
