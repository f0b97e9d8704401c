// C++ drop-in parity driver: exercises the include/carve/*.hpp API the way the
// reference's own tests do (test_solvers.cpp:152-174, test_carver.cpp:34-210)
// and prints FNV-1a-64 hashes of the configs for tests/test_cpp_dropin.py.
//   carve_parity selftest            -> reference unit-test pins, exit 0/1
//   carve_parity hash W H TW TH      -> "<input hash> <output hash> <seams hash>"
//   carve_parity convert IN OUT      -> load_image + save_image (PNG / PPM codecs, host only)
#include <cstdio>
#include <cstring>
#include <string>

#include "carve/carve.hpp"

using namespace carve;

static uint64_t fnv(const void* p, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t k = 0; k < n; ++k) {
        h ^= static_cast<const uint8_t*>(p)[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

static int failures = 0;
#define EXPECT(c)                                                      \
    do {                                                               \
        if (!(c)) {                                                    \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                \
        }                                                              \
    } while (0)

template <class F>
static Errc thrown(F&& f) {
    try {
        f();
    } catch (const Error& e) {
        return e.code();
    }
    return Errc(-1);
}

static int selftest() {
    // dp_seam worked example (test_solvers.cpp:156-174)
    EnergyMap m{3, 3, {1, 2, 3, 4, 1, 6, 7, 8, 1}};
    auto [seam, table] = dp_seam(m);
    const double want[9] = {1, 2, 3, 5, 2, 8, 9, 10, 3};
    for (int k = 0; k < 9; ++k) EXPECT(table.m[k] == want[k]);
    EXPECT((seam == Seam{0, 1, 2}));
    EXPECT((dp_seam(EnergyMap{4, 1, {8, 2, 6, 2}}).seam == Seam{1}));
    EXPECT(parallel_dp_seam(m, 8).table == table);
    // energy_e1 pins (test_energy.cpp:33-64)
    LumaGrid g{3, 1, {0, 100, 0}};
    auto e = energy_e1(g);
    EXPECT(e.values[0] == 100.0 && e.values[1] == 0.0 && e.values[2] == 100.0);
    // remove_seam (test_carver.cpp:35-73)
    PixelGrid p(2, 1);
    p.at(0, 0) = Rgb{1, 1, 1};
    p.at(0, 1) = Rgb{2, 2, 2};
    EXPECT((remove_seam(p, {0}).at(0, 0) == Rgb{2, 2, 2}));
    EXPECT(thrown([] { remove_seam(PixelGrid(1, 2), {0, 0}); }) == Errc::width_too_small);
    EXPECT(thrown([] { remove_seam(PixelGrid(3, 2), {0, 2}); }) == Errc::invalid_seam);
    // zero-energy column carved exactly (test_carver.cpp:117-128)
    PixelGrid cols(4, 4);
    const uint8_t vals[4] = {10, 50, 10, 90};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) cols.at(i, j) = Rgb{vals[j], vals[j], vals[j]};
    auto [out, rep] = carve_to_width(cols, 3);
    EXPECT(rep.seam_count == 1 && (rep.seams[0] == Seam{1, 1, 1, 1}));
    EXPECT(out.width == 3 && out.at(2, 1).r == 10 && out.at(2, 2).r == 90);
    // report invariants (test_carver.cpp:129-142)
    auto img = make_test_image(24, 16);
    auto [o2, r2] = carve_to_width(img, 10);
    EXPECT(o2.width == 10 && r2.seam_count == 14 && r2.per_seam.size() == 14);
    double sum = 0;
    for (auto& t : r2.per_seam) sum += t.energy_s + t.solve_s + t.remove_s;
    EXPECT(r2.total_s >= sum);
    EXPECT(thrown([&] { carve_to_width(img, 0); }) == Errc::invalid_target);
    EXPECT(thrown([&] { carve_to_width(img, 25); }) == Errc::invalid_target);
    CarveConfig bad;
    bad.solver = SolverKind::Greedy;
    bad.forward = true;
    EXPECT(thrown([&] { carve_to_width(img, 2, bad); }) == Errc::usage_error);
    // transpose sandwich (test_carver.cpp:202-210)
    auto t = make_test_image(10, 8);
    EXPECT(carve_to_height(t, 5).first == transpose(carve_to_width(transpose(t), 5).first));
    EXPECT(transpose(transpose(t)) == t);
    // insert_seam (test_carver.cpp:76-92)
    PixelGrid one(1, 1, Rgb{9, 8, 7});
    auto ins = insert_seam(one, {0});
    EXPECT(ins.width == 2 && (ins.at(0, 0) == Rgb{9, 8, 7}) && (ins.at(0, 1) == Rgb{9, 8, 7}));
    PixelGrid two(2, 1);
    two.at(0, 0) = Rgb{0, 0, 0};
    two.at(0, 1) = Rgb{100, 100, 100};
    EXPECT((insert_seam(two, {0}).at(0, 1) == Rgb{50, 50, 50}));
    // enlarge_to_width (test_carver.cpp:214-253)
    PixelGrid pair(2, 1);
    pair.at(0, 0) = Rgb{10, 20, 30};
    pair.at(0, 1) = Rgb{30, 40, 50};
    auto [wide, wrep] = enlarge_to_width(pair, 3);
    EXPECT(wide.width == 3 && wrep.seam_count == 1 && (wrep.seams[0] == Seam{0}));
    EXPECT((wide.at(0, 1) == Rgb{20, 30, 40}) && (wide.at(0, 2) == Rgb{30, 40, 50}));
    auto six = make_test_image(6, 4);
    EXPECT(thrown([&] { enlarge_to_width(six, 5); }) == Errc::invalid_target);
    EXPECT(thrown([&] { enlarge_to_width(six, 12); }) == Errc::target_too_large);
    EXPECT(enlarge_to_width(six, 11).first.width == 11);
    // record_seams (test_carver.cpp:257-275)
    auto [rec, rrep] = record_seams(make_test_image(15, 9), 6);
    EXPECT(rec.size() == 6 && rrep.seam_count == 6 && rrep.per_seam.size() == 6);
    for (int i = 0; i < 9; ++i)
        for (size_t a = 0; a < rec.size(); ++a)
            for (size_t b = a + 1; b < rec.size(); ++b) EXPECT(rec[a][i] != rec[b][i]);
    EXPECT(thrown([] { record_seams(PixelGrid(4, 4), 4); }) == Errc::invalid_target);
    // apply_mask / remove_object (test_energy.cpp:209-216, test_carver.cpp:279-287, :335-344)
    EnergyMap unit{3, 3, std::vector<double>(9, 1.0)};
    for (double v : apply_mask(unit, RemovalMask{3, 3, std::vector<uint8_t>(9, 1)}).values) EXPECT(v == -4000.0);
    PixelGrid gc(5, 5);
    const uint8_t gv[5] = {50, 120, 60, 70, 80};
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) gc.at(i, j) = Rgb{gv[j], gv[j], gv[j]};
    RemovalMask col{5, 5, std::vector<uint8_t>(25, 0)};
    for (int i = 0; i < 5; ++i) col.set(i, 1, true);
    auto [ro, rrep2] = remove_object(gc, col);
    EXPECT(rrep2.seam_count == 1 && (rrep2.seams[0] == Seam{1, 1, 1, 1, 1}) && ro.width == 5 && ro.height == 5);
    EXPECT(thrown([] { remove_object(PixelGrid(4, 4), RemovalMask{4, 4, std::vector<uint8_t>(16, 0)}); }) ==
           Errc::empty_mask);
    EXPECT(thrown([] { remove_object(PixelGrid(4, 4), RemovalMask{3, 4, std::vector<uint8_t>(12, 1)}); }) ==
           Errc::dimension_mismatch);
    // remove_seam overloads on scalar grids (carver.hpp:84-112; test_carver.cpp:55-73)
    LumaGrid lg{3, 2, {1, 2, 3, 4, 5, 6}};
    auto lr = remove_seam(lg, {1, 0});
    EXPECT(lr.width == 2 && (lr.values == std::vector<double>{1, 3, 5, 6}));
    EnergyMap em{3, 2, {1, 2, 3, 4, 5, 6}};
    auto er = remove_seam(em, {2, 2});
    EXPECT(er.width == 2 && (er.values == std::vector<double>{1, 2, 4, 5}));
    RemovalMask rm{3, 2, {1, 0, 1, 0, 1, 0}};
    auto mr = remove_seam(rm, {0, 2});  // not connected: allowed, like the reference
    EXPECT(mr.width == 2 && (mr.flags == std::vector<uint8_t>{0, 1, 0, 1}));
    EXPECT((detail::drop_columns({1, 2, 3}, 3, 1, {1}) == std::vector<double>{1, 3}));
    EXPECT(thrown([] { remove_seam(EnergyMap{2, 1, {1, 2}}, {2}); }) == Errc::invalid_seam);
    // detail::insert_columns: per-row columns may jump (carver.hpp:116-132)
    PixelGrid jump(3, 2);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) jump.at(i, j) = Rgb{uint8_t(10 * j), uint8_t(10 * j), uint8_t(10 * j)};
    auto ic = detail::insert_columns(jump, {0, 2});
    EXPECT(ic.width == 4 && (ic.at(0, 1) == Rgb{5, 5, 5}) && (ic.at(1, 3) == Rgb{20, 20, 20}));
    // dp_seam_forward with caller costs (solvers.hpp:294-326): gray only gives the size
    LumaGrid g0{2, 2, {0, 0, 0, 0}};
    ForwardCosts fc{2, 2, {5, 5, 0, 9}, {1, 2, 9, 9}, {9, 9, 9, 9}};
    auto fr = dp_seam_forward(g0, fc);
    EXPECT((fr.table.m == std::vector<double>{1, 2, 10, 10}) && (fr.seam == Seam{0, 0}) && fr.table.b[3] == 0);
    // forward + recompute=false is a supported configuration (carver.hpp:175-184)
    CarveConfig fnr;
    fnr.forward = true;
    fnr.recompute = false;
    EXPECT(carve_to_width(make_test_image(20, 12), 15, fnr).first.width == 15);
    // BenchRecord timers (bench.hpp:32-59, 140-201)
    auto bimg = make_test_image(40, 30);
    CarveConfig dpcfg;
    dpcfg.solver = SolverKind::Dynamic;
    BenchRecord full = time_full_carve(bimg, 0.5, dpcfg, 2);
    EXPECT(full.phase == Phase::full_carve && full.n == 30 && full.scale && *full.scale == 0.5);
    EXPECT(full.repetitions == 2 && full.wall_time_s > 0.0 && full.solver == SolverKind::Dynamic);
    EXPECT(full.energy_fn == "e1" && full.timestamp_utc.size() == 20 && full.timestamp_utc.back() == 'Z');
    CarveConfig fwd;
    fwd.forward = true;
    BenchRecord single = time_single_seam(bimg, fwd, 1);
    EXPECT(single.phase == Phase::single_seam && !single.scale && single.solver == SolverKind::ParallelDynamic);
    EXPECT(thrown([&] { time_full_carve(bimg, 1.5, dpcfg, 1); }) == Errc::usage_error);
    EXPECT(thrown([&] { time_single_seam(bimg, dpcfg, 0); }) == Errc::usage_error);
    EXPECT(parse_phase("full_carve") == Phase::full_carve && !parse_phase("x"));
    BenchRecord copy = full;
    EXPECT(copy == full);
    std::printf(failures ? "selftest FAILED (%d)\n" : "selftest ok\n", failures);
    return failures ? 1 : 0;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::string(argv[1]) == "selftest") return selftest();
        if (argc == 4 && std::string(argv[1]) == "convert") {  // host-only image IO (PNG/PPM), no GPU
            save_image(load_image(argv[2]), argv[3]);
            return 0;
        }
        if (argc == 6 && std::string(argv[1]) == "hash") {
            const int w = std::atoi(argv[2]), h = std::atoi(argv[3]), tw = std::atoi(argv[4]), th = std::atoi(argv[5]);
            auto img = make_test_image(w, h);
            auto [out, rep] = ::carve::detail::carve_device(img, tw, th);
            uint64_t hs = 0xcbf29ce484222325ull;
            std::string all;
            for (auto& s : rep.seams) all.append(reinterpret_cast<const char*>(s.data()), s.size() * sizeof(int));
            hs = fnv(all.data(), all.size());
            std::printf("%016llx %016llx %016llx\n", (unsigned long long)fnv(img.bytes(), img.pixels.size() * 3),
                        (unsigned long long)fnv(out.bytes(), out.pixels.size() * 3), (unsigned long long)hs);
            return 0;
        }
        std::fprintf(stderr, "usage: carve_parity selftest | hash W H TW TH\n");
        return 1;
    } catch (const Error& e) {
        std::fprintf(stderr, "carve_parity: %s\n", e.what());
        return 2;
    }
}
