// carve/cli.hpp — drop-in for the reference CLI's `resize`, `enlarge` and
// `seams` paths (/root/reference/proj/include/carve/cli.hpp:146-309, 368-379)
// without CLI11:
//   carve resize  --input X --output Y [--scale S | --width W] [--height H]
//                 [--solver dp|pardp] [--energy e1] [--forward]
//   carve enlarge --input X --output Y [--scale S | --width W] [--height H] [solver flags]
//   carve seams   --input X --output Y --count N [solver flags]
//   carve remove-object --input X --mask M --output Y [--no-restore] [solver flags]
//   carve energy  --input X --output Y.png --energy e1|e2|hog|entropy
// Exit codes as the reference: 0 success, 1 usage error, 2 runtime error.
// CARVE_WORKERS is validated like the reference (cli.hpp:109-126) but never
// changes output. Other subcommands report usage_error (not on the B200 path).
#pragma once

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <string>
#include <vector>

#include "carve/carve.hpp"

namespace carve::cli {

struct ResizeCmd {
    std::string input, output;
    std::optional<double> scale;
    std::optional<int> width, height;
    std::string solver = "pardp", energy = "e1";
    bool forward = false;
    int count = 0;  // seams --count
    std::string mask;        // remove-object --mask (cli.hpp:41-45, 177-182)
    bool no_restore = false;  // remove-object --no-restore
};
using EnlargeCmd = ResizeCmd;  // same options (cli.hpp:34-39, 167-175)
struct SeamsCmd : ResizeCmd {};  // --input --output --count + solver flags (cli.hpp:52-56, 189-193)

namespace detail {

inline double parse_double(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const double d = std::strtod(v.c_str(), &end);
    if (end == v.c_str() || *end) fail(Errc::usage_error, flag + ": not a number: " + v);
    return d;
}

inline int parse_positive(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const long n = std::strtol(v.c_str(), &end, 10);
    if (end == v.c_str() || *end || n < 1 || n > 1 << 30) fail(Errc::usage_error, flag + ": not a positive integer: " + v);
    return int(n);
}

inline void check_env_workers() {
    if (const char* s = std::getenv("CARVE_WORKERS")) {
        char* end = nullptr;
        const long v = std::strtol(s, &end, 10);
        if (end == s || *end != '\0' || v < 0) fail(Errc::usage_error, "CARVE_WORKERS must be a nonnegative integer");
    }
}

} // namespace detail

inline ResizeCmd parse_resize(const std::vector<std::string>& a) {
    ResizeCmd c;
    for (size_t k = 1; k < a.size(); ++k) {
        const std::string& f = a[k];
        auto val = [&]() -> const std::string& {
            if (k + 1 >= a.size()) fail(Errc::usage_error, f + " needs a value");
            return a[++k];
        };
        if (f == "--input") c.input = val();
        else if (f == "--output") c.output = val();
        else if (f == "--scale") {
            c.scale = detail::parse_double(f, val());
            if (!(*c.scale > 0.0 && *c.scale <= 2.0)) fail(Errc::usage_error, "scale must be in (0, 2]");
        } else if (f == "--width") c.width = detail::parse_positive(f, val());
        else if (f == "--height") c.height = detail::parse_positive(f, val());
        else if (f == "--solver") {
            c.solver = val();
            if (!parse_solver(c.solver)) fail(Errc::usage_error, "--solver: unknown backend " + c.solver);
        } else if (f == "--energy") {
            c.energy = val();
            if (c.energy != "e1" && c.energy != "e2" && c.energy != "hog" && c.energy != "entropy")
                fail(Errc::usage_error, "--energy: unknown function " + c.energy);
        } else if (f == "--forward") c.forward = true;
        else if (f == "--count" && a[0] == "seams") c.count = detail::parse_positive(f, val());
        else if (f == "--mask" && a[0] == "remove-object") c.mask = val();
        else if (f == "--no-restore" && a[0] == "remove-object") c.no_restore = true;
        else fail(Errc::usage_error, "unknown option " + f);
    }
    if (c.input.empty() || c.output.empty()) fail(Errc::usage_error, "--input and --output are required");
    if (c.scale && c.width) fail(Errc::usage_error, "--scale excludes --width");
    if (a[0] == "seams" && (c.scale || c.width || c.height)) fail(Errc::usage_error, "seams takes --count, not a size");
    if (a[0] == "seams" && c.count < 1) fail(Errc::usage_error, "--count is required");
    if (a[0] == "remove-object" && c.mask.empty()) fail(Errc::usage_error, "--mask is required");
    if (a[0] == "remove-object" && (c.scale || c.width || c.height))
        fail(Errc::usage_error, "remove-object takes no size options");
    if (a[0] == "energy" && (c.scale || c.width || c.height || c.forward))
        fail(Errc::usage_error, "energy takes --input, --output and --energy only");
    return c;
}

namespace detail {
inline CarveConfig config_of(const ResizeCmd& cmd) {
    CarveConfig cfg;
    cfg.solver = *parse_solver(cmd.solver);
    cfg.energy_fn = cmd.energy == "e1" ? EnergyFn::e1 : cmd.energy == "e2" ? EnergyFn::e2
                  : cmd.energy == "hog" ? EnergyFn::hog : EnergyFn::entropy;
    cfg.forward = cmd.forward;
    return cfg;
}
} // namespace detail

/// cli.hpp:242-259 run_resize: carve_to_width then carve_to_height, in one device-resident carve.
inline int run_resize(const ResizeCmd& cmd) {
    detail::check_env_workers();
    PixelGrid img = load_image(cmd.input);
    const CarveConfig cfg = detail::config_of(cmd);
    ::carve::detail::check_config(cfg);
    const int tw = cmd.scale ? int(std::lround(*cmd.scale * img.width)) : cmd.width.value_or(img.width);
    const int th = cmd.height.value_or(img.height);
    if (tw > img.width) fail(Errc::invalid_target, "resize cannot grow the width; use the enlarge command");
    if (tw < 1) fail(Errc::invalid_target, "target width must be in [1, width]");
    if (th < 1 || th > img.height) fail(Errc::invalid_target, "target height must be in [1, height]");
    auto [out, report] = ::carve::detail::carve_device(img, tw, th, cfg);
    save_image(out, cmd.output);
    return 0;
}

/// cli.hpp:262-277 run_enlarge: enlarge_to_width, then enlarge_to_width of the
/// transpose for the height — both phases in one device-resident call.
inline int run_enlarge(const EnlargeCmd& cmd) {
    detail::check_env_workers();
    PixelGrid img = load_image(cmd.input);
    const CarveConfig cfg = detail::config_of(cmd);
    ::carve::detail::check_config(cfg);
    const int tw = cmd.scale ? int(std::lround(*cmd.scale * img.width)) : cmd.width.value_or(img.width);
    const int th = cmd.height.value_or(img.height);
    PixelGrid out(tw, th);
    const carve_cuda_config c = ::carve::detail::abi_config(cfg);
    ::carve::detail::check(carve_cuda_enlarge(img.bytes(), img.width, img.height, tw, th, &c, out.bytes(), nullptr));
    save_image(out, cmd.output);
    return 0;
}

/// cli.hpp:301-309 run_seams: record the next --count seams and paint them red
/// on the original image.
inline int run_seams(const SeamsCmd& cmd) {
    detail::check_env_workers();
    PixelGrid img = load_image(cmd.input);
    auto [recorded, report] = record_seams(img, cmd.count, detail::config_of(cmd));
    for (const Seam& seam : recorded)
        for (size_t i = 0; i < seam.size(); ++i) img.at(int(i), seam[i]) = Rgb{255, 0, 0};
    save_image(img, cmd.output);
    return 0;
}

/// cli.hpp:288-299 run_energy: the normalised energy map of the input as a gray PNG
/// (e1 on the device; the other energy functions are not on the B200 path).
inline int run_energy(const ResizeCmd& cmd) {
    auto ends_with_png = [](const std::string& s) {
        if (s.size() < 4) return false;
        std::string t = s.substr(s.size() - 4);
        for (char& ch : t) ch = char(std::tolower(static_cast<unsigned char>(ch)));
        return t == ".png";
    };
    if (!ends_with_png(cmd.output)) fail(Errc::usage_error, "energy output must be a .png path");
    PixelGrid img = load_image(cmd.input);
    if (cmd.energy != "e1") ::carve::detail::unsupported("energy " + cmd.energy);
    const EnergyMap energy = energy_e1(img);  // compute_energy(to_grayscale(img), e1), fused on the device
    save_gray_png(normalize_to_gray(energy), energy.width, energy.height, cmd.output);
    return 0;
}

/// cli.hpp:279-287 run_remove_object: mask_from_image of --mask, remove_object.
inline int run_remove_object(const ResizeCmd& cmd) {
    detail::check_env_workers();
    PixelGrid img = load_image(cmd.input);
    PixelGrid mask_img = load_image(cmd.mask);
    RemovalMask mask = mask_from_image(mask_img);
    auto [result, report] = remove_object(img, mask, detail::config_of(cmd), !cmd.no_restore);
    save_image(result, cmd.output);
    return 0;
}

inline int cli_main(int argc, char** argv) {
    try {
        const std::vector<std::string> args(argv + 1, argv + argc);
        if (args.empty() || args[0] == "--help" || args[0] == "-h") {
            std::printf("usage: carve resize  --input X --output Y [--scale S | --width W] [--height H]\n"
                        "                     [--solver dp|pardp] [--energy e1]\n"
                        "       carve enlarge --input X --output Y [--scale S | --width W] [--height H]\n"
                        "       carve seams   --input X --output Y --count N\n"
                        "       carve remove-object --input X --mask M --output Y [--no-restore]\n"
                        "       carve energy  --input X --output Y.png --energy e1\n");
            return args.empty() ? 1 : 0;
        }
        if (args[0] == "resize") return run_resize(parse_resize(args));
        if (args[0] == "enlarge") return run_enlarge(parse_resize(args));
        if (args[0] == "remove-object") return run_remove_object(parse_resize(args));
        if (args[0] == "energy") {
            const ResizeCmd c = parse_resize(args);
            if (c.input.empty() || c.output.empty()) fail(Errc::usage_error, "energy needs --input and --output");
            bool has_energy = false;
            for (const auto& a : args) has_energy = has_energy || a == "--energy";
            if (!has_energy) fail(Errc::usage_error, "energy: --energy is required");
            return run_energy(c);
        }
        if (args[0] == "seams") {
            SeamsCmd c;
            static_cast<ResizeCmd&>(c) = parse_resize(args);
            return run_seams(c);
        }
        fail(Errc::usage_error,
             "subcommand '" + args[0] +
                 "' is not supported by the B200 engine (resize, enlarge, seams, remove-object, energy)");
    } catch (const Error& err) {
        std::fprintf(stderr, "carve: %s\n", err.what());
        return err.code() == Errc::usage_error ? 1 : 2;
    } catch (const std::exception& err) {
        std::fprintf(stderr, "carve: %s\n", err.what());
        return 2;
    }
}

} // namespace carve::cli
