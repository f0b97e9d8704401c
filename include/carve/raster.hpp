// carve/raster.hpp — drop-in for the reference raster layer
// (/root/reference/proj/include/carve/raster.hpp). Value types keep the
// reference layout (packed 3-byte Rgb, row-major PixelGrid, FP64 LumaGrid);
// to_grayscale and transpose run on the B200 through libcarve_cuda.
#pragma once

#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "carve/error.hpp"
#include "carve/png_codec.hpp"

namespace carve {

struct Rgb {
    std::uint8_t r = 0, g = 0, b = 0;
    friend bool operator==(const Rgb&, const Rgb&) = default;
};
static_assert(sizeof(Rgb) == 3, "Rgb is the packed 3-byte pixel the C ABI expects");

struct PixelGrid {
    int width = 0;
    int height = 0;
    std::vector<Rgb> pixels;

    PixelGrid() = default;
    PixelGrid(int w, int h, Rgb fill = {}) : width(w), height(h) {
        if (w < 1 || h < 1) fail(Errc::empty_image, "PixelGrid dimensions must be >= 1");
        pixels.assign(size_t(w) * size_t(h), fill);
    }
    Rgb& at(int row, int col) { return pixels[size_t(row) * width + col]; }
    const Rgb& at(int row, int col) const { return pixels[size_t(row) * width + col]; }
    const std::uint8_t* bytes() const { return reinterpret_cast<const std::uint8_t*>(pixels.data()); }
    std::uint8_t* bytes() { return reinterpret_cast<std::uint8_t*>(pixels.data()); }

    friend bool operator==(const PixelGrid&, const PixelGrid&) = default;
};

struct LumaGrid {
    int width = 0;
    int height = 0;
    std::vector<double> values;

    double& at(int row, int col) { return values[size_t(row) * width + col]; }
    double at(int row, int col) const { return values[size_t(row) * width + col]; }
    double at_clamped(int row, int col) const {
        return at(std::clamp(row, 0, height - 1), std::clamp(col, 0, width - 1));
    }
};

/// BT.601 luma in FP64 on the device, bit-identical to the reference.
inline LumaGrid to_grayscale(const PixelGrid& grid) {
    LumaGrid out{grid.width, grid.height, std::vector<double>(grid.pixels.size())};
    detail::check(carve_cuda_to_grayscale(grid.bytes(), grid.width, grid.height, out.values.data()));
    return out;
}

inline PixelGrid transpose(const PixelGrid& grid) {
    PixelGrid out(grid.height, grid.width);
    detail::check(carve_cuda_transpose_rgb(grid.bytes(), grid.width, grid.height, out.bytes()));
    return out;
}

// ---- image IO: PNG (carve/png_codec.hpp, zlib) and binary PPM (raster.hpp:81-284) ----
namespace detail {

struct CFile {
    std::FILE* fp;
    CFile(const std::string& p, const char* mode) : fp(std::fopen(p.c_str(), mode)) {}
    ~CFile() { if (fp) std::fclose(fp); }
    CFile(const CFile&) = delete;
    CFile& operator=(const CFile&) = delete;
};

// next decimal header field of a P6 file; '#' comments and whitespace skipped
inline int ppm_field(std::FILE* fp) {
    int c;
    for (;;) {
        c = std::fgetc(fp);
        if (c == '#') {
            while (c != EOF && c != '\n') c = std::fgetc(fp);
            continue;
        }
        if (c == EOF || !std::isspace(c)) break;
    }
    if (c == EOF || !std::isdigit(c)) return -1;
    long v = 0;
    for (; c != EOF && std::isdigit(c); c = std::fgetc(fp))
        if ((v = v * 10 + (c - '0')) > 1000000) return -1;
    return int(v);
}

inline bool has_suffix(std::string s, std::string suf) {
    if (s.size() < suf.size()) return false;
    for (auto* x : {&s, &suf}) std::transform(x->begin(), x->end(), x->begin(), [](unsigned char ch) { return std::tolower(ch); });
    return s.compare(s.size() - suf.size(), suf.size(), suf) == 0;
}

} // namespace detail

inline PixelGrid load_image(const std::string& path) {
    detail::CFile f(path, "rb");
    if (!f.fp) fail(Errc::file_not_found, path + ": no such file");
    unsigned char sig[8] = {};
    const size_t got = std::fread(sig, 1, sizeof sig, f.fp);
    std::rewind(f.fp);
    static const unsigned char png_sig[8] = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
    if (got >= 8 && std::memcmp(sig, png_sig, 8) == 0) {
        const png::Image im = png::decode(png::read_file(f.fp), path);
        PixelGrid g(im.width, im.height);
        std::memcpy(g.bytes(), im.rgb.data(), im.rgb.size());
        return g;
    }
    if (got < 2 || sig[0] != 'P' || sig[1] != '6')
        fail(Errc::unsupported_format, path + ": expected PNG or binary PPM (P6)");
    std::fgetc(f.fp);
    std::fgetc(f.fp);
    const int w = detail::ppm_field(f.fp), h = detail::ppm_field(f.fp), maxval = detail::ppm_field(f.fp);
    if (w < 1 || h < 1) fail(Errc::corrupt_image, path + ": bad PPM header");
    if (maxval != 255) fail(Errc::unsupported_format, path + ": only maxval 255 PPM supported");
    PixelGrid g(w, h);
    if (std::fread(g.pixels.data(), 3, g.pixels.size(), f.fp) != g.pixels.size())
        fail(Errc::corrupt_image, path + ": truncated PPM payload");
    return g;
}

inline void save_image(const PixelGrid& grid, const std::string& path) {
    if (detail::has_suffix(path, ".png")) {
        png::write_file(path, png::encode(grid.bytes(), grid.width, grid.height, 3));
        return;
    }
    if (!detail::has_suffix(path, ".ppm"))
        fail(Errc::unsupported_format, path + ": unknown output extension (use .png or .ppm)");
    detail::CFile f(path, "wb");
    if (!f.fp) fail(Errc::io_failure, path + ": cannot open for writing");
    const std::string hdr = "P6\n" + std::to_string(grid.width) + " " + std::to_string(grid.height) + "\n255\n";
    if (std::fwrite(hdr.data(), 1, hdr.size(), f.fp) != hdr.size() ||
        std::fwrite(grid.pixels.data(), 3, grid.pixels.size(), f.fp) != grid.pixels.size())
        fail(Errc::io_failure, path + ": write failed");
}

/// 8-bit grayscale PNG, used for energy-map visualization (raster.hpp:262-283).
inline void save_gray_png(const std::vector<std::uint8_t>& gray, int width, int height, const std::string& path) {
    png::write_file(path, png::encode(gray.data(), width, height, 1));
}

} // namespace carve
