// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference headers, compiled in place
// from /root/reference/proj/include by oracle/Makefile into oracle/_ref/.
// The reference is placed in namespace carve_ref so it can never collide with
// the product's own `carve::` drop-in headers.
//
// Build flags follow the reference's own Release default
// (/root/reference/proj/CMakeLists.txt:8-10): -O3, default x86-64 target,
// no -march (FMA contraction would change FP64 luma bits).
//
// Status codes: 0 = ok, 1 + Errc on carve::Error, 100 on any other exception.

#define carve carve_ref
#include "carve/bench.hpp"
#include "carve/carver.hpp"
#include "carve/energy.hpp"
#include "carve/raster.hpp"
#include "carve/solvers.hpp"
#undef carve

#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const carve_ref::Error& e) {
        g_err = e.what();
        return 1 + int(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

carve_ref::PixelGrid grid_from(const std::uint8_t* rgb, int w, int h) {
    carve_ref::PixelGrid g(w, h);
    std::memcpy(g.pixels.data(), rgb, size_t(w) * h * 3);
    return g;
}

void grid_to(const carve_ref::PixelGrid& g, std::uint8_t* out) {
    std::memcpy(out, g.pixels.data(), g.pixels.size() * 3);
}

carve_ref::EnergyMap map_from(const double* e, int w, int h) {
    carve_ref::EnergyMap m;
    m.width = w;
    m.height = h;
    m.values.assign(e, e + size_t(w) * h);
    return m;
}

carve_ref::CarveConfig config_for(int solver, unsigned workers) {
    carve_ref::CarveConfig cfg;
    cfg.solver = solver == 0 ? carve_ref::SolverKind::Dynamic : carve_ref::SolverKind::ParallelDynamic;
    cfg.solver_opts.workers = workers;
    return cfg;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

unsigned ref_hardware_concurrency(void) { return std::thread::hardware_concurrency(); }

// bench.hpp:67-94
int ref_make_test_image(int w, int h, std::uint8_t* out) {
    return guarded([&] { grid_to(carve_ref::make_test_image(w, h), out); });
}

// raster.hpp:61-71
int ref_to_grayscale(const std::uint8_t* rgb, int w, int h, double* out) {
    return guarded([&] {
        auto l = carve_ref::to_grayscale(grid_from(rgb, w, h));
        std::memcpy(out, l.values.data(), l.values.size() * sizeof(double));
    });
}

// energy.hpp:89-98 on an arbitrary luma plane
int ref_energy_e1_luma(const double* luma, int w, int h, double* out) {
    return guarded([&] {
        carve_ref::LumaGrid g;
        g.width = w;
        g.height = h;
        g.values.assign(luma, luma + size_t(w) * h);
        auto e = carve_ref::energy_e1(g);
        std::memcpy(out, e.values.data(), e.values.size() * sizeof(double));
    });
}

// energy_e1(to_grayscale(img)) — the composition solve_step uses (carver.hpp:161-162)
int ref_energy_e1_rgb(const std::uint8_t* rgb, int w, int h, double* out) {
    return guarded([&] {
        auto e = carve_ref::compute_energy(carve_ref::to_grayscale(grid_from(rgb, w, h)), carve_ref::EnergyFn::e1);
        std::memcpy(out, e.values.data(), e.values.size() * sizeof(double));
    });
}

// solvers.hpp:263-289 (solver 0, dp_seam) / :331-347 (solver 1, parallel_dp_seam)
int ref_dp_seam(const double* e, int w, int h, int solver, unsigned workers, double* m_out, int* b_out,
                int* seam_out) {
    return guarded([&] {
        auto m = map_from(e, w, h);
        auto r = solver == 0 ? carve_ref::dp_seam(m) : carve_ref::parallel_dp_seam(m, workers);
        if (m_out) std::memcpy(m_out, r.table.m.data(), r.table.m.size() * sizeof(double));
        if (b_out) std::memcpy(b_out, r.table.b.data(), r.table.b.size() * sizeof(int));
        std::memcpy(seam_out, r.seam.data(), r.seam.size() * sizeof(int));
    });
}

// solvers.hpp:69-78
int ref_validate_seam(const int* seam, int n, int w, int h) {
    return guarded([&] { carve_ref::validate_seam(carve_ref::Seam(seam, seam + n), w, h); });
}

// carver.hpp:71-82
int ref_remove_seam(const std::uint8_t* rgb, int w, int h, const int* seam, int n, std::uint8_t* out) {
    return guarded([&] {
        auto g = carve_ref::remove_seam(grid_from(rgb, w, h), carve_ref::Seam(seam, seam + n));
        grid_to(g, out);
    });
}

// raster.hpp:73-79
int ref_transpose(const std::uint8_t* rgb, int w, int h, std::uint8_t* out) {
    return guarded([&] { grid_to(carve_ref::transpose(grid_from(rgb, w, h)), out); });
}

// run_resize semantics (cli.hpp:242-259): carve_to_width then carve_to_height.
// seams_out (nullable) receives every seam, concatenated in removal order.
// times_out (nullable) receives {width-phase total_s, height-phase total_s}.
int ref_carve(const std::uint8_t* rgb, int w, int h, int target_w, int target_h, int solver, unsigned workers,
              std::uint8_t* out, int* seams_out, double* times_out) {
    return guarded([&] {
        auto cfg = config_for(solver, workers);
        carve_ref::PixelGrid img = grid_from(rgb, w, h);
        size_t off = 0;
        double tw = 0.0, th = 0.0;
        if (target_w < 1 || target_w > img.width)
            carve_ref::fail(carve_ref::Errc::invalid_target, "target width must be in [1, width]");
        if (target_w < img.width) {
            auto [carved, report] = carve_ref::carve_to_width(img, target_w, cfg);
            img = std::move(carved);
            tw = report.total_s;
            if (seams_out)
                for (auto& s : report.seams) {
                    std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
                    off += s.size();
                }
        }
        if (target_h != img.height) {
            auto [carved, report] = carve_ref::carve_to_height(img, target_h, cfg);
            img = std::move(carved);
            th = report.total_s;
            if (seams_out)
                for (auto& s : report.seams) {
                    std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
                    off += s.size();
                }
        }
        grid_to(img, out);
        if (times_out) {
            times_out[0] = tw;
            times_out[1] = th;
        }
    });
}

// energy.hpp:196-216 forward_costs on an arbitrary LumaGrid
int ref_forward_costs(const double* luma, int w, int h, double* left, double* up, double* right) {
    return guarded([&] {
        carve_ref::LumaGrid g;
        g.width = w;
        g.height = h;
        g.values.assign(luma, luma + size_t(w) * h);
        auto fc = carve_ref::forward_costs(g);
        std::memcpy(left, fc.cost_left.data(), fc.cost_left.size() * 8);
        std::memcpy(up, fc.cost_up.data(), fc.cost_up.size() * 8);
        std::memcpy(right, fc.cost_right.data(), fc.cost_right.size() * 8);
    });
}

// solvers.hpp:294-326 dp_seam_forward(gray, forward_costs(gray))
int ref_dp_seam_forward(const double* luma, int w, int h, double* m_out, int* b_out, int* seam_out) {
    return guarded([&] {
        carve_ref::LumaGrid g;
        g.width = w;
        g.height = h;
        g.values.assign(luma, luma + size_t(w) * h);
        auto r = carve_ref::dp_seam_forward(g, carve_ref::forward_costs(g));
        std::memcpy(m_out, r.table.m.data(), r.table.m.size() * 8);
        std::memcpy(b_out, r.table.b.data(), r.table.b.size() * 4);
        std::memcpy(seam_out, r.seam.data(), r.seam.size() * 4);
    });
}

// solvers.hpp:294-326 dp_seam_forward(gray, costs) with arbitrary caller costs
// (gray only supplies the dimensions there)
int ref_dp_seam_forward_costs(const double* left, const double* up, const double* right, int w, int h,
                              double* m_out, int* b_out, int* seam_out) {
    return guarded([&] {
        carve_ref::LumaGrid g;
        g.width = w;
        g.height = h;
        g.values.assign(size_t(w) * h, 0.0);
        carve_ref::ForwardCosts fc;
        fc.width = w;
        fc.height = h;
        const size_t n = size_t(w) * h;
        fc.cost_left.assign(left, left + n);
        fc.cost_up.assign(up, up + n);
        fc.cost_right.assign(right, right + n);
        auto r = carve_ref::dp_seam_forward(g, fc);
        std::memcpy(m_out, r.table.m.data(), r.table.m.size() * 8);
        std::memcpy(b_out, r.table.b.data(), r.table.b.size() * 4);
        std::memcpy(seam_out, r.seam.data(), r.seam.size() * 4);
    });
}

// carver.hpp:84-112 remove_seam(LumaGrid) (kind 0) / remove_seam(EnergyMap) (kind 1)
int ref_remove_seam_f64(const double* in, int w, int h, const int* seam, int n, int kind, double* out) {
    return guarded([&] {
        const carve_ref::Seam s(seam, seam + n);
        std::vector<double> v;
        if (kind == 0) {
            carve_ref::LumaGrid g;
            g.width = w;
            g.height = h;
            g.values.assign(in, in + size_t(w) * h);
            v = carve_ref::remove_seam(g, s).values;
        } else {
            v = carve_ref::remove_seam(map_from(in, w, h), s).values;
        }
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

// carver.hpp:100-112 remove_seam(RemovalMask)
int ref_remove_seam_u8(const std::uint8_t* in, int w, int h, const int* seam, int n, std::uint8_t* out) {
    return guarded([&] {
        carve_ref::RemovalMask m;
        m.width = w;
        m.height = h;
        m.flags.assign(in, in + size_t(w) * h);
        auto r = carve_ref::remove_seam(m, carve_ref::Seam(seam, seam + n));
        std::memcpy(out, r.flags.data(), r.flags.size());
    });
}

// bench.hpp:140-174 time_single_seam / :177-201 time_full_carve: the BenchRecord
// fields (solver, n, phase, scale, repetitions) of one call, for the drop-in's
// BenchRecord test. out: [solver, n, phase, has_scale, repetitions], scale_out
int ref_bench_record(const std::uint8_t* rgb, int w, int h, int full, double scale, int forward, int reps,
                     int* out, double* scale_out) {
    return guarded([&] {
        carve_ref::CarveConfig cfg;
        cfg.forward = forward != 0;
        const auto img = grid_from(rgb, w, h);
        const carve_ref::BenchRecord r = full ? carve_ref::time_full_carve(img, scale, cfg, reps)
                                              : carve_ref::time_single_seam(img, cfg, reps);
        out[0] = int(r.solver);
        out[1] = r.n;
        out[2] = int(r.phase);
        out[3] = r.scale.has_value() ? 1 : 0;
        out[4] = r.repetitions;
        *scale_out = r.scale.value_or(0.0);
    });
}

// run_resize (cli.hpp:242-259) with CarveConfig::forward / ::recompute
// (carver.hpp:15-24, 153-188); seams_out as ref_carve.
int ref_carve_cfg(const std::uint8_t* rgb, int w, int h, int target_w, int target_h, int forward, int recompute,
                  std::uint8_t* out, int* seams_out) {
    return guarded([&] {
        carve_ref::CarveConfig cfg;
        cfg.forward = forward != 0;
        cfg.recompute = recompute != 0;
        carve_ref::PixelGrid img = grid_from(rgb, w, h);
        size_t off = 0;
        auto log = [&](const carve_ref::CarveReport& r) {
            if (seams_out)
                for (auto& s : r.seams) {
                    std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
                    off += s.size();
                }
        };
        if (target_w < 1 || target_w > img.width)
            carve_ref::fail(carve_ref::Errc::invalid_target, "target width must be in [1, width]");
        if (target_w < img.width) {
            auto [carved, report] = carve_ref::carve_to_width(img, target_w, cfg);
            img = std::move(carved);
            log(report);
        }
        if (target_h != img.height) {
            auto [carved, report] = carve_ref::carve_to_height(img, target_h, cfg);
            img = std::move(carved);
            log(report);
        }
        grid_to(img, out);
    });
}

// energy.hpp:220-241 apply_mask
int ref_apply_mask(const double* e, int w, int h, const std::uint8_t* mask, double* out) {
    return guarded([&] {
        carve_ref::RemovalMask m{w, h, std::vector<std::uint8_t>(mask, mask + size_t(w) * h)};
        auto r = carve_ref::apply_mask(map_from(e, w, h), m);
        std::memcpy(out, r.values.data(), r.values.size() * 8);
    });
}

// energy.hpp:244-253 mask_from_image
int ref_mask_from_image(const std::uint8_t* rgb, int w, int h, std::uint8_t* flags) {
    return guarded([&] {
        auto m = carve_ref::mask_from_image(grid_from(rgb, w, h));
        std::memcpy(flags, m.flags.data(), m.flags.size());
    });
}

// carver.hpp:327-340 remove_object (cfg.forward as given, restore flag). out:
// the result (caller buffer of w*h*3 bytes), out_dims = {width, height};
// seams_out (w*h ints) the report's seams concatenated, nseams their count.
int ref_remove_object(const std::uint8_t* rgb, int w, int h, const std::uint8_t* mask, int forward, int restore,
                      std::uint8_t* out, int* out_dims, int* seams_out, int* nseams) {
    return guarded([&] {
        carve_ref::CarveConfig cfg;
        cfg.forward = forward != 0;
        carve_ref::RemovalMask m{w, h, std::vector<std::uint8_t>(mask, mask + size_t(w) * h)};
        auto [res, report] = carve_ref::remove_object(grid_from(rgb, w, h), m, cfg, restore != 0);
        grid_to(res, out);
        out_dims[0] = res.width;
        out_dims[1] = res.height;
        size_t off = 0;
        for (auto& s : report.seams) {
            std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
            off += s.size();
        }
        *nseams = report.seam_count;
    });
}

// carver.hpp:289-321 detail::remove_object_vertical (no orientation choice, no
// empty-mask check)
int ref_remove_object_vertical(const std::uint8_t* rgb, int w, int h, const std::uint8_t* mask, int restore,
                               std::uint8_t* out, int* out_dims, int* seams_out, int* nseams) {
    return guarded([&] {
        carve_ref::CarveConfig cfg;
        carve_ref::RemovalMask m{w, h, std::vector<std::uint8_t>(mask, mask + size_t(w) * h)};
        auto [res, report] = carve_ref::detail::remove_object_vertical(grid_from(rgb, w, h), m, cfg, restore != 0);
        grid_to(res, out);
        out_dims[0] = res.width;
        out_dims[1] = res.height;
        size_t off = 0;
        for (auto& s : report.seams) {
            std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
            off += s.size();
        }
        *nseams = report.seam_count;
    });
}

// carver.hpp:117-140 insert_seam (validate_seam + insert_columns)
int ref_insert_seam(const std::uint8_t* rgb, int w, int h, const int* seam, int n, std::uint8_t* out) {
    return guarded([&] { grid_to(carve_ref::insert_seam(grid_from(rgb, w, h), carve_ref::Seam(seam, seam + n)), out); });
}

// carver.hpp:226-262 record_seams, default config: `count` seams in original
// coordinates, concatenated (count * h ints).
int ref_record_seams(const std::uint8_t* rgb, int w, int h, int count, int* seams_out) {
    return guarded([&] {
        auto [seams, report] = carve_ref::record_seams(grid_from(rgb, w, h), count, carve_ref::CarveConfig{});
        size_t off = 0;
        for (auto& s : seams) {
            std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
            off += s.size();
        }
    });
}

// run_enlarge semantics (cli.hpp:262-277): enlarge_to_width (carver.hpp:266-285)
// on the width, then on the transpose for the height. seams_out (nullable)
// receives the recorded seams of both phases (original coordinates of the grid
// each phase started from), concatenated.
int ref_enlarge(const std::uint8_t* rgb, int w, int h, int target_w, int target_h, std::uint8_t* out,
                int* seams_out) {
    return guarded([&] {
        carve_ref::PixelGrid img = grid_from(rgb, w, h);
        size_t off = 0;
        auto log = [&](const carve_ref::CarveReport& r) {
            if (seams_out)
                for (auto& s : r.seams) {
                    std::memcpy(seams_out + off, s.data(), s.size() * sizeof(int));
                    off += s.size();
                }
        };
        if (target_w != img.width) {
            auto [wider, report] = carve_ref::enlarge_to_width(img, target_w);
            img = std::move(wider);
            log(report);
        }
        if (target_h != img.height) {
            auto [taller, report] = carve_ref::enlarge_to_width(carve_ref::transpose(img), target_h);
            img = carve_ref::transpose(taller);
            log(report);
        }
        grid_to(img, out);
    });
}

// Batch driver for the C5 CPU baseline: the reference has no batch API but its
// pipelines are reentrant, so `threads` host threads each run
// carve_to_width over a static, strided share of the images.
int ref_carve_batch(const std::uint8_t* const* in, int n, int w, int h, int target_w, int solver, unsigned workers,
                    unsigned threads, std::uint8_t* const* out) {
    std::vector<int> status(threads ? threads : 1, 0);
    if (threads == 0) threads = 1;
    auto worker = [&](unsigned t) {
        status[t] = guarded([&] {
            auto cfg = config_for(solver, workers);
            for (int k = int(t); k < n; k += int(threads)) {
                auto [carved, report] = carve_ref::carve_to_width(grid_from(in[k], w, h), target_w, cfg);
                grid_to(carved, out[k]);
            }
        });
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (auto& th : pool) th.join();
    for (int s : status)
        if (s) return s;
    return 0;
}

} // extern "C"
