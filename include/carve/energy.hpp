// carve/energy.hpp — drop-in for the reference energy layer
// (/root/reference/proj/include/carve/energy.hpp). Only the gradient-magnitude
// energy e1 is on the B200 path; the other energy functions, forward costs and
// masks keep their declarations and fail with usage_error (no CPU fallback).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "carve/error.hpp"
#include "carve/raster.hpp"

namespace carve {

struct EnergyMap {
    int width = 0;
    int height = 0;
    std::vector<double> values;

    double& at(int row, int col) { return values[size_t(row) * width + col]; }
    double at(int row, int col) const { return values[size_t(row) * width + col]; }
};

struct RemovalMask {
    int width = 0;
    int height = 0;
    std::vector<std::uint8_t> flags;
    bool marked(int row, int col) const { return flags[size_t(row) * width + col] != 0; }
    void set(int row, int col, bool v) { flags[size_t(row) * width + col] = v ? 1 : 0; }
    size_t marked_count() const {
        size_t n = 0;
        for (auto f : flags) n += f != 0;
        return n;
    }
};

struct ForwardCosts {
    int width = 0;
    int height = 0;
    std::vector<double> cost_left, cost_up, cost_right;

    double left(int row, int col) const { return cost_left[size_t(row) * width + col]; }
    double up(int row, int col) const { return cost_up[size_t(row) * width + col]; }
    double right(int row, int col) const { return cost_right[size_t(row) * width + col]; }
};

enum class EnergyFn { e1, e2, hog, entropy };

inline const char* to_string(EnergyFn fn) {
    static const char* names[] = {"e1", "e2", "hog", "entropy"};
    return names[int(fn)];
}

/// e = |gx| + |gy| over clamped central differences, FP64, on the device.
inline EnergyMap energy_e1(const LumaGrid& gray) {
    EnergyMap out{gray.width, gray.height, std::vector<double>(gray.values.size())};
    detail::check(carve_cuda_energy_e1_luma(gray.values.data(), gray.width, gray.height, out.values.data()));
    return out;
}

/// energy_e1(to_grayscale(img)) fused on the device (one upload, no luma plane).
inline EnergyMap energy_e1(const PixelGrid& img) {
    EnergyMap out{img.width, img.height, std::vector<double>(img.pixels.size())};
    detail::check(carve_cuda_energy_e1_rgb(img.bytes(), img.width, img.height, out.values.data()));
    return out;
}

inline EnergyMap energy_e2(const LumaGrid&) { detail::unsupported("energy e2"); }
inline EnergyMap energy_hog(const LumaGrid&) { detail::unsupported("energy hog"); }
inline EnergyMap energy_entropy(const LumaGrid&) { detail::unsupported("energy entropy"); }

inline EnergyMap compute_energy(const LumaGrid& gray, EnergyFn fn) {
    if (fn != EnergyFn::e1) detail::unsupported(std::string("energy ") + to_string(fn));
    return energy_e1(gray);
}

/// energy.hpp:196-216 forward transition costs, on the device.
inline ForwardCosts forward_costs(const LumaGrid& gray) {
    ForwardCosts fc;
    fc.width = gray.width;
    fc.height = gray.height;
    const size_t n = gray.values.size();
    fc.cost_left.resize(n);
    fc.cost_up.resize(n);
    fc.cost_right.resize(n);
    detail::check(carve_cuda_forward_costs(gray.values.data(), gray.width, gray.height, fc.cost_left.data(),
                                           fc.cost_up.data(), fc.cost_right.data()));
    return fc;
}
/// energy.hpp:220-241 on the device: masked cells -> -1000*(h*m + 1).
inline EnergyMap apply_mask(const EnergyMap& energy, const RemovalMask& mask) {
    if (energy.width != mask.width || energy.height != mask.height)
        fail(Errc::dimension_mismatch, "mask dimensions do not match energy map");
    EnergyMap out{energy.width, energy.height, std::vector<double>(energy.values.size())};
    detail::check(carve_cuda_apply_mask(energy.values.data(), energy.width, energy.height, mask.flags.data(),
                                        out.values.data()));
    return out;
}

/// energy.hpp:244-253: FP64 luma >= 128 marks a pixel (on the device).
inline RemovalMask mask_from_image(const PixelGrid& img) {
    RemovalMask mask;
    mask.width = img.width;
    mask.height = img.height;
    mask.flags.resize(img.pixels.size());
    detail::check(carve_cuda_mask_from_rgb(img.bytes(), img.width, img.height, mask.flags.data()));
    return mask;
}

/// energy.hpp:285-299: min-max normalisation to 8-bit gray (constant maps -> 0), the
/// `carve energy` export. Host arithmetic in the reference's operation order.
inline std::vector<std::uint8_t> normalize_to_gray(const EnergyMap& energy) {
    double lo = energy.values.empty() ? 0.0 : energy.values[0];
    double hi = lo;
    for (double v : energy.values) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
    }
    std::vector<std::uint8_t> out(energy.values.size(), 0);
    const double span = hi - lo;
    if (span > 0.0)
        for (size_t i = 0; i < out.size(); ++i)
            out[i] = std::uint8_t(std::lround((energy.values[i] - lo) / span * 255.0));
    return out;
}

inline RemovalMask transpose(const RemovalMask& mask) {
    RemovalMask out;
    out.width = mask.height;
    out.height = mask.width;
    out.flags.resize(mask.flags.size());
    for (int i = 0; i < mask.height; ++i)
        for (int j = 0; j < mask.width; ++j)
            out.flags[size_t(j) * out.width + i] = mask.flags[size_t(i) * mask.width + j];
    return out;
}

struct MaskBounds {
    int top = 0, left = 0, bottom = -1, right = -1;  // inclusive; empty when bottom < top
    int width() const { return right - left + 1; }
    int height() const { return bottom - top + 1; }
};

inline MaskBounds mask_bounds(const RemovalMask& mask) {
    MaskBounds b{mask.height, mask.width, -1, -1};
    for (int i = 0; i < mask.height; ++i)
        for (int j = 0; j < mask.width; ++j)
            if (mask.marked(i, j)) {
                b.top = std::min(b.top, i);
                b.left = std::min(b.left, j);
                b.bottom = std::max(b.bottom, i);
                b.right = std::max(b.right, j);
            }
    return b;
}

} // namespace carve
