// carve/solvers.hpp — drop-in for the reference solver layer
// (/root/reference/proj/include/carve/solvers.hpp). dp_seam, parallel_dp_seam
// and find_seam(Dynamic | ParallelDynamic) run the B200 DP kernel (K2+K3) and
// return the reference's exact table and seam; brute force and greedy (the
// paper-comparison backends) fail with usage_error.
#pragma once

#include <cstdlib>
#include <optional>
#include <string>
#include <vector>

#include "carve/energy.hpp"
#include "carve/error.hpp"

namespace carve {

using Seam = std::vector<int>;

enum class SolverKind { BruteForce, Greedy, Dynamic, ParallelDynamic };

inline const char* to_string(SolverKind k) {
    static const char* names[] = {"bruteforce", "greedy", "dp", "pardp"};
    return names[int(k)];
}

inline std::optional<SolverKind> parse_solver(const std::string& name) {
    for (auto k : {SolverKind::BruteForce, SolverKind::Greedy, SolverKind::Dynamic, SolverKind::ParallelDynamic})
        if (name == to_string(k)) return k;
    return std::nullopt;
}

struct CostTable {
    int width = 0;
    int height = 0;
    std::vector<double> m;
    std::vector<int> b;

    CostTable() = default;
    CostTable(int w, int h) : width(w), height(h), m(size_t(w) * h), b(size_t(w) * h) {}
    double cost(int row, int col) const { return m[size_t(row) * width + col]; }
    int back(int row, int col) const { return b[size_t(row) * width + col]; }
    friend bool operator==(const CostTable&, const CostTable&) = default;
};

struct SeamResult {
    Seam seam;
    CostTable table;
};

inline constexpr int kDefaultBruteCap = 16;

struct SolverOptions {
    int brute_cap = kDefaultBruteCap;
    unsigned workers = 0;  // accepted; never changes output
};

inline void validate_seam(const Seam& seam, int width, int height) {
    detail::check(carve_cuda_validate_seam(seam.data(), int(seam.size()), width, height));
}

inline double seam_cost(const EnergyMap& energy, const Seam& seam) {
    validate_seam(seam, energy.width, energy.height);
    double total = 0.0;
    for (int i = 0; i < energy.height; ++i) total += energy.at(i, seam[i]);
    return total;
}

/// Accumulated-cost table plus backtracking on the B200; bit-identical to the reference.
inline SeamResult dp_seam(const EnergyMap& energy) {
    if (energy.width < 1 || energy.height < 1) fail(Errc::empty_image, "image is empty");
    SeamResult r{Seam(size_t(energy.height)), CostTable(energy.width, energy.height)};
    detail::check(carve_cuda_dp_seam(energy.values.data(), energy.width, energy.height, r.table.m.data(),
                                     r.table.b.data(), r.seam.data()));
    return r;
}

/// Same table as dp_seam for every worker count (the worker knob is a no-op).
inline SeamResult parallel_dp_seam(const EnergyMap& energy, unsigned workers = 0) {
    (void)workers;
    return dp_seam(energy);
}

/// solvers.hpp:294-326 forward-energy DP on the B200 over the caller's three
/// cost planes (any finite values; `gray` only supplies the dimensions, as in
/// the reference). Non-finite costs throw usage_error: the device scan assumes
/// finite candidates where the reference starts from best = +inf.
inline SeamResult dp_seam_forward(const LumaGrid& gray, const ForwardCosts& costs) {
    if (gray.width < 1 || gray.height < 1) fail(Errc::empty_image, "image is empty");
    if (gray.width != costs.width || gray.height != costs.height)
        fail(Errc::dimension_mismatch, "forward costs do not match image dimensions");
    SeamResult r{Seam(size_t(gray.height)), CostTable(gray.width, gray.height)};
    detail::check(carve_cuda_dp_seam_forward_costs(costs.cost_left.data(), costs.cost_up.data(),
                                                   costs.cost_right.data(), gray.width, gray.height,
                                                   r.table.m.data(), r.table.b.data(), r.seam.data()));
    return r;
}

inline Seam brute_force_seam(const EnergyMap&, int = kDefaultBruteCap) { detail::unsupported("solver bruteforce"); }
inline Seam greedy_seam(const EnergyMap&) { detail::unsupported("solver greedy"); }

inline Seam find_seam(const EnergyMap& energy, SolverKind kind, const SolverOptions& opts = {}) {
    (void)opts;
    if (kind != SolverKind::Dynamic && kind != SolverKind::ParallelDynamic)
        detail::unsupported(std::string("solver ") + to_string(kind));
    if (energy.width < 1 || energy.height < 1) fail(Errc::empty_image, "image is empty");
    Seam seam(size_t(energy.height));
    detail::check(carve_cuda_dp_seam(energy.values.data(), energy.width, energy.height, nullptr, nullptr, seam.data()));
    return seam;
}

} // namespace carve
