// carve/carver.hpp — drop-in for the reference pipelines
// (/root/reference/proj/include/carve/carver.hpp). remove_seam(PixelGrid),
// carve_to_width and carve_to_height run entirely on the B200: the whole seam
// loop (energy, DP, backtrack, removal) stays on the device and the report's
// per-seam timings come from device %globaltimer stamps.
#pragma once

#include <algorithm>
#include <chrono>
#include <utility>
#include <vector>

#include "carve/energy.hpp"
#include "carve/error.hpp"
#include "carve/raster.hpp"
#include "carve/solvers.hpp"

namespace carve {

struct CarveConfig {
    SolverKind solver = SolverKind::ParallelDynamic;
    EnergyFn energy_fn = EnergyFn::e1;
    bool forward = false;
    bool recompute = true;  // false: e1 once, then carved alongside (carver.hpp:176-188)
    SolverOptions solver_opts{};
};

struct SeamTiming {
    double energy_s = 0.0;
    double solve_s = 0.0;
    double remove_s = 0.0;
};

struct CarveReport {
    int seam_count = 0;
    std::vector<SeamTiming> per_seam;
    std::vector<Seam> seams;  // coordinates of the image each seam was taken from
    double total_s = 0.0;
};

namespace detail {

inline void check_config(const CarveConfig& cfg) {
    const bool dp = cfg.solver == SolverKind::Dynamic || cfg.solver == SolverKind::ParallelDynamic;
    if (cfg.forward && !dp) fail(Errc::usage_error, "forward energy requires the dp or pardp solver");
    if (!dp) unsupported(std::string("solver ") + to_string(cfg.solver));
    // forward mode solves on forward costs; energy_fn only matters for the backward form
    if (!cfg.forward && cfg.energy_fn != EnergyFn::e1) unsupported(std::string("energy ") + to_string(cfg.energy_fn));
}

inline carve_cuda_config abi_config(const CarveConfig& cfg) {
    return carve_cuda_config{cfg.forward ? 1 : 0, cfg.recompute ? 1 : 0};
}

// one device-resident carve: width phase then height phase (run_resize order)
inline std::pair<PixelGrid, CarveReport> carve_device(const PixelGrid& grid, int tw, int th,
                                                      const CarveConfig& cfg = {}) {
    const auto t0 = std::chrono::steady_clock::now();
    const int vs = grid.width - tw, hs = grid.height - th;
    PixelGrid out(tw, th);
    std::vector<int32_t> flat(size_t(vs) * grid.height + size_t(hs) * tw);
    std::vector<carve_seam_timing> tim(size_t(vs + hs));
    const carve_cuda_config c = abi_config(cfg);
    check(carve_cuda_carve_cfg(grid.bytes(), grid.width, grid.height, tw, th, &c, out.bytes(), flat.data(),
                               tim.data()));
    CarveReport rep;
    rep.seam_count = vs + hs;
    size_t off = 0;
    for (int k = 0; k < vs + hs; ++k) {
        const size_t len = k < vs ? size_t(grid.height) : size_t(tw);
        rep.seams.emplace_back(flat.begin() + off, flat.begin() + off + len);
        off += len;
        rep.per_seam.push_back({tim[k].energy_s, tim[k].solve_s, tim[k].remove_s});
    }
    rep.total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(out), std::move(rep)};
}

/// carver.hpp:57-67: column deletion on a row-major scalar grid (row i loses
/// column seam[i]); on the device. Like the reference it does not require a
/// connected seam; columns outside [0, width) throw invalid_seam.
inline std::vector<double> drop_columns(const std::vector<double>& values, int width, int height,
                                        const Seam& seam) {
    std::vector<double> out(size_t(std::max(width - 1, 0)) * height);
    check(carve_cuda_remove_seam_f64(values.data(), width, height, seam.data(), int(seam.size()), out.data()));
    return out;
}

/// carver.hpp:118-132: per-row duplication without the seam-connectivity
/// requirement (replayed recorded seams may jump more than one column).
inline PixelGrid insert_columns(const PixelGrid& grid, const std::vector<int>& cols) {
    PixelGrid out(grid.width + 1, grid.height);
    check(carve_cuda_insert_columns_rgb(grid.bytes(), grid.width, grid.height, cols.data(), int(cols.size()),
                                        out.bytes()));
    return out;
}

} // namespace detail

inline PixelGrid remove_seam(const PixelGrid& grid, const Seam& seam) {
    validate_seam(seam, grid.width, grid.height);
    if (grid.width < 2) fail(Errc::width_too_small, "cannot remove a seam from a 1-pixel-wide image");
    PixelGrid out(grid.width - 1, grid.height);
    detail::check(carve_cuda_remove_seam_rgb(grid.bytes(), grid.width, grid.height, seam.data(), int(seam.size()),
                                             out.bytes()));
    return out;
}

/// carver.hpp:84-98: the LumaGrid and EnergyMap overloads (detail::drop_columns).
inline LumaGrid remove_seam(const LumaGrid& gray, const Seam& seam) {
    LumaGrid out;
    out.width = gray.width - 1;
    out.height = gray.height;
    out.values = detail::drop_columns(gray.values, gray.width, gray.height, seam);
    return out;
}

inline EnergyMap remove_seam(const EnergyMap& energy, const Seam& seam) {
    EnergyMap out;
    out.width = energy.width - 1;
    out.height = energy.height;
    out.values = detail::drop_columns(energy.values, energy.width, energy.height, seam);
    return out;
}

/// carver.hpp:100-112: the RemovalMask overload.
inline RemovalMask remove_seam(const RemovalMask& mask, const Seam& seam) {
    RemovalMask out;
    out.width = mask.width - 1;
    out.height = mask.height;
    out.flags.resize(size_t(std::max(out.width, 0)) * out.height);
    detail::check(carve_cuda_remove_seam_u8(mask.flags.data(), mask.width, mask.height, seam.data(),
                                            int(seam.size()), out.flags.data()));
    return out;
}

inline std::pair<PixelGrid, CarveReport> carve_to_width(const PixelGrid& grid, int target_width,
                                                        const CarveConfig& cfg = {}) {
    if (target_width < 1 || target_width > grid.width)
        fail(Errc::invalid_target, "target width must be in [1, width]");
    detail::check_config(cfg);
    return detail::carve_device(grid, target_width, grid.height, cfg);
}

inline std::pair<PixelGrid, CarveReport> carve_to_height(const PixelGrid& grid, int target_height,
                                                         const CarveConfig& cfg = {}) {
    if (target_height < 1 || target_height > grid.height)
        fail(Errc::invalid_target, "target height must be in [1, height]");
    detail::check_config(cfg);
    return detail::carve_device(grid, grid.width, target_height, cfg);
}

/// Batch entry point (no reference equivalent): same-size images sharded by
/// image over `devices` (empty = all visible GPUs), no inter-GPU traffic.
inline std::vector<PixelGrid> carve_batch(const std::vector<PixelGrid>& imgs, int target_width, int target_height,
                                          const std::vector<int>& devices = {}) {
    if (imgs.empty()) fail(Errc::empty_input, "empty batch");
    std::vector<PixelGrid> outs(imgs.size(), PixelGrid(target_width, target_height));
    std::vector<const uint8_t*> in(imgs.size());
    std::vector<uint8_t*> out(imgs.size());
    for (size_t k = 0; k < imgs.size(); ++k) {
        if (imgs[k].width != imgs[0].width || imgs[k].height != imgs[0].height)
            fail(Errc::dimension_mismatch, "batch images must share one size");
        in[k] = imgs[k].bytes();
        out[k] = outs[k].bytes();
    }
    detail::check(carve_cuda_carve_batch(in.data(), int(imgs.size()), imgs[0].width, imgs[0].height, target_width,
                                         target_height, out.data(), devices.empty() ? nullptr : devices.data(),
                                         int(devices.size())));
    return outs;
}

/// carver.hpp:137-140: one pixel per row right of the seam, the rounded mean of
/// its left and right neighbours (duplicating at the right border).
inline PixelGrid insert_seam(const PixelGrid& grid, const Seam& seam) {
    validate_seam(seam, grid.width, grid.height);
    PixelGrid out(grid.width + 1, grid.height);
    detail::check(carve_cuda_insert_seam_rgb(grid.bytes(), grid.width, grid.height, seam.data(), int(seam.size()),
                                             out.bytes()));
    return out;
}

/// carver.hpp:226-262: the removal loop on the device; seams reported in
/// original-image coordinates.
inline std::pair<std::vector<Seam>, CarveReport> record_seams(const PixelGrid& grid, int count,
                                                              const CarveConfig& cfg = {}) {
    if (count < 0 || count > grid.width - 1) fail(Errc::invalid_target, "cannot record more seams than width-1");
    detail::check_config(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<int32_t> flat(size_t(count) * grid.height);
    std::vector<carve_seam_timing> tim(size_t(std::max(count, 1)));
    const carve_cuda_config c = detail::abi_config(cfg);
    detail::check(
        carve_cuda_record_seams(grid.bytes(), grid.width, grid.height, count, &c, flat.data(), tim.data()));
    std::vector<Seam> seams;
    CarveReport rep;
    for (int t = 0; t < count; ++t) {
        seams.emplace_back(flat.begin() + size_t(t) * grid.height, flat.begin() + size_t(t + 1) * grid.height);
        rep.per_seam.push_back({tim[t].energy_s, tim[t].solve_s, tim[t].remove_s});
    }
    rep.seam_count = count;
    rep.seams = seams;
    rep.total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(seams), std::move(rep)};
}

/// carver.hpp:266-285: record target_width - width seams, then insert them
/// (one device expansion pass, identical to the reference's ordered replay).
inline std::pair<PixelGrid, CarveReport> enlarge_to_width(const PixelGrid& grid, int target_width,
                                                          const CarveConfig& cfg = {}) {
    const int k = target_width - grid.width;
    if (k < 0) fail(Errc::invalid_target, "enlargement target is below the current width");
    if (target_width > 2 * grid.width - 1)
        fail(Errc::target_too_large, "single-pass enlargement is limited to 2*width-1");
    detail::check_config(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    PixelGrid out(target_width, grid.height);
    std::vector<int32_t> flat(std::max<size_t>(size_t(k) * grid.height, 1));
    const carve_cuda_config c = detail::abi_config(cfg);
    std::vector<carve_seam_timing> tim(size_t(std::max(k, 1)));
    detail::check(carve_cuda_enlarge_timed(grid.bytes(), grid.width, grid.height, target_width, grid.height, &c,
                                           out.bytes(), flat.data(), tim.data()));
    CarveReport rep;  // record_seams' report (carver.hpp:275)
    for (int t = 0; t < k; ++t) {
        rep.seams.emplace_back(flat.begin() + size_t(t) * grid.height, flat.begin() + size_t(t + 1) * grid.height);
        rep.per_seam.push_back({tim[t].energy_s, tim[t].solve_s, tim[t].remove_s});
    }
    rep.seam_count = k;
    rep.total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(out), std::move(rep)};
}

namespace detail {

// the device removal loop (carver.hpp:289-340): orientation 0 = by mask_bounds, 1 = vertical
inline std::pair<PixelGrid, CarveReport> remove_object_device(const PixelGrid& grid, const RemovalMask& mask,
                                                              const CarveConfig& cfg, bool restore, int orientation) {
    if (grid.width != mask.width || grid.height != mask.height)
        fail(Errc::dimension_mismatch, "mask dimensions do not match image");
    const auto t0 = std::chrono::steady_clock::now();
    const carve_cuda_config c = abi_config(cfg);
    std::vector<uint8_t> buf(grid.pixels.size() * 3);
    std::vector<int32_t> flat(std::max<size_t>(grid.pixels.size(), 1));
    std::vector<carve_seam_timing> tim(std::max<size_t>(size_t(std::max(grid.width, grid.height)), 1));
    int ow = 0, oh = 0, ns = 0;
    check(carve_cuda_remove_object_ex(grid.bytes(), grid.width, grid.height, mask.flags.data(), &c, restore ? 1 : 0,
                                      orientation, buf.data(), &ow, &oh, flat.data(), &ns, tim.data()));
    PixelGrid out(ow, oh);
    std::copy(buf.begin(), buf.begin() + size_t(ow) * oh * 3, out.bytes());
    CarveReport rep;
    rep.seam_count = ns;
    const MaskBounds b = mask_bounds(mask);
    const size_t len = size_t(orientation == 1 || b.width() <= b.height() ? grid.height : grid.width);
    for (int t = 0; t < ns; ++t) {
        rep.seams.emplace_back(flat.begin() + size_t(t) * len, flat.begin() + size_t(t + 1) * len);
        rep.per_seam.push_back({tim[t].energy_s, tim[t].solve_s, tim[t].remove_s});
    }
    rep.total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(out), std::move(rep)};
}

/// carver.hpp:289-321: the removal loop along columns (then the restoring
/// enlargement), on the device; an empty mask carves nothing.
inline std::pair<PixelGrid, CarveReport> remove_object_vertical(const PixelGrid& grid, const RemovalMask& mask,
                                                                const CarveConfig& cfg, bool restore) {
    return remove_object_device(grid, mask, cfg, restore, 1);
}

} // namespace detail

/// carver.hpp:327-340: the whole removal loop (mask-biased e1, DP, removal of
/// image and mask) and the restoring enlargement run on the device; the report's
/// per-seam energy / solve / remove laps come from device timestamps.
inline std::pair<PixelGrid, CarveReport> remove_object(const PixelGrid& grid, const RemovalMask& mask,
                                                       const CarveConfig& cfg = {}, bool restore = true) {
    detail::check_config(cfg);
    return detail::remove_object_device(grid, mask, cfg, restore, 0);
}

} // namespace carve
