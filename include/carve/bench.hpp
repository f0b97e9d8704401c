// carve/bench.hpp — drop-in for the reference's fixture and timers
// (/root/reference/proj/include/carve/bench.hpp:22-59, 67-94, 140-201).
// make_test_image is the host generator (byte-identical to the reference's);
// the timers return the reference's BenchRecord and measure what it measures:
// time_single_seam the solver call alone (energy / forward costs computed once
// outside the timed region, then uploaded per call like any host EnergyMap),
// time_full_carve carve_to_width host PixelGrid in -> host PixelGrid out through
// the B200 engine; minimum over reps. The suite/CSV/plot helpers of the
// reference bench (run_suite, fit_scaling, emit_csv) are not on the hot path.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <ctime>
#include <limits>
#include <optional>
#include <string>

#include "carve/carver.hpp"

namespace carve {

enum class Phase { single_seam, full_carve };

inline const char* to_string(Phase p) { return p == Phase::single_seam ? "single_seam" : "full_carve"; }

inline std::optional<Phase> parse_phase(const std::string& name) {
    if (name == "single_seam") return Phase::single_seam;
    if (name == "full_carve") return Phase::full_carve;
    return std::nullopt;
}

/// bench.hpp:32-43 — one timed measurement.
struct BenchRecord {
    SolverKind solver = SolverKind::Dynamic;
    std::string energy_fn = "e1";
    int n = 0;                    // image height (square side for the reference suite)
    Phase phase = Phase::single_seam;
    std::optional<double> scale;  // full_carve only
    double wall_time_s = 0.0;     // minimum over repetitions
    int repetitions = 1;
    std::string timestamp_utc;    // RFC 3339, second precision

    friend bool operator==(const BenchRecord&, const BenchRecord&) = default;
};

inline std::string now_rfc3339() {
    const std::time_t t = std::chrono::system_clock::to_time_t(std::chrono::system_clock::now());
    std::tm tm{};
    gmtime_r(&t, &tm);
    char buf[32];
    std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", &tm);
    return buf;
}

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

namespace detail {
inline double clamp_time(double s) { return std::max(s, 1e-9); }  // monotonic clock floor (bench.hpp:134)
inline double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace detail

/// bench.hpp:140-174 — only the solver call is timed; the energy map (or, with
/// cfg.forward, the forward costs) is computed once outside the timed region.
inline BenchRecord time_single_seam(const PixelGrid& grid, const CarveConfig& cfg, int reps) {
    if (reps < 1) fail(Errc::usage_error, "reps must be >= 1");
    detail::check_config(cfg);

    BenchRecord rec;
    rec.solver = cfg.solver;
    rec.energy_fn = to_string(cfg.energy_fn);
    rec.n = grid.height;
    rec.phase = Phase::single_seam;
    rec.repetitions = reps;
    rec.timestamp_utc = now_rfc3339();

    const LumaGrid gray = to_grayscale(grid);
    double best = std::numeric_limits<double>::infinity();
    if (cfg.forward) {
        const ForwardCosts costs = forward_costs(gray);
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            volatile double sink = dp_seam_forward(gray, costs).table.m.back();
            (void)sink;
            best = std::min(best, detail::seconds_since(t0));
        }
    } else {
        const EnergyMap energy = compute_energy(gray, cfg.energy_fn);
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            Seam seam = find_seam(energy, cfg.solver, cfg.solver_opts);
            best = std::min(best, detail::seconds_since(t0));
            volatile int sink = seam.back();
            (void)sink;
        }
    }
    rec.wall_time_s = detail::clamp_time(best);
    return rec;
}

/// bench.hpp:177-201 — carve_to_width(grid, round(scale*width)) end to end.
inline BenchRecord time_full_carve(const PixelGrid& grid, double scale, const CarveConfig& cfg, int reps) {
    if (reps < 1) fail(Errc::usage_error, "reps must be >= 1");
    if (!(scale > 0.0) || scale > 1.0) fail(Errc::usage_error, "scale must be in (0, 1]");

    BenchRecord rec;
    rec.solver = cfg.solver;
    rec.energy_fn = to_string(cfg.energy_fn);
    rec.n = grid.height;
    rec.phase = Phase::full_carve;
    rec.scale = scale;
    rec.repetitions = reps;
    rec.timestamp_utc = now_rfc3339();

    const int target = int(std::lround(scale * grid.width));
    double best = std::numeric_limits<double>::infinity();
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        auto [carved, report] = carve_to_width(grid, target, cfg);
        best = std::min(best, detail::seconds_since(t0));
        volatile int sink = carved.width;
        (void)sink;
    }
    rec.wall_time_s = detail::clamp_time(best);
    return rec;
}

} // namespace carve
