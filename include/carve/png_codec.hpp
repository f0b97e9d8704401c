// carve/png_codec.hpp — PNG reading and writing for the drop-in IO layer
// (SURVEY.md §8f row 3). The reference links libpng (raster.hpp:13, 93-147,
// 187-215), whose headers are absent from this image; this codec is written
// against zlib (inflate/deflate + crc32) instead and reproduces what the
// reference asks libpng for:
//   * 16-bit channels -> Errc::unsupported_format (raster.hpp:110-113)
//   * palette -> RGB, gray 1/2/4-bit expanded to 8 bits (v * 255 / (2^d - 1)),
//     gray -> RGB, tRNS / alpha discarded, Adam7 interlacing resolved
//     (raster.hpp:116-125)
//   * any structural error (bad CRC, truncated or malformed stream, invalid
//     IHDR, missing chunks) -> Errc::corrupt_image (raster.hpp:105-108)
//   * output: 8-bit RGB, non-interlaced (raster.hpp:206-207); gray PNG for
//     energy-map export (raster.hpp:262-283).
// Host-side file IO only: nothing here is on the GPU path. Link with -lz.
#pragma once

#include <zlib.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "carve/error.hpp"

namespace carve::png {

inline uint32_t be32(const uint8_t* p) { return uint32_t(p[0]) << 24 | uint32_t(p[1]) << 16 | uint32_t(p[2]) << 8 | p[3]; }

inline void put32(std::vector<uint8_t>& v, uint32_t x) {
    for (int s = 24; s >= 0; s -= 8) v.push_back(uint8_t(x >> s));
}

struct Image {
    int width = 0, height = 0;
    std::vector<uint8_t> rgb;  // packed 8-bit RGB, row-major
};

namespace detail {

[[noreturn]] inline void corrupt(const std::string& path, const std::string& why) {
    fail(Errc::corrupt_image, path + ": corrupt PNG (" + why + ")");
}

// PNG filter types 0..4 (PNG spec 9.2), in place on one scanline
inline bool unfilter(uint8_t type, uint8_t* cur, const uint8_t* prev, size_t n, size_t bpp) {
    switch (type) {
        case 0: return true;
        case 1:
            for (size_t i = bpp; i < n; ++i) cur[i] = uint8_t(cur[i] + cur[i - bpp]);
            return true;
        case 2:
            if (prev)
                for (size_t i = 0; i < n; ++i) cur[i] = uint8_t(cur[i] + prev[i]);
            return true;
        case 3:
            for (size_t i = 0; i < n; ++i) {
                const int a = i >= bpp ? cur[i - bpp] : 0, b = prev ? prev[i] : 0;
                cur[i] = uint8_t(cur[i] + ((a + b) >> 1));
            }
            return true;
        case 4:
            for (size_t i = 0; i < n; ++i) {
                const int a = i >= bpp ? cur[i - bpp] : 0, b = prev ? prev[i] : 0;
                const int c = (i >= bpp && prev) ? prev[i - bpp] : 0;
                const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
                cur[i] = uint8_t(cur[i] + ((pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c)));
            }
            return true;
        default: return false;
    }
}

}  // namespace detail

/// Decode a PNG byte stream to 8-bit RGB with the reference's libpng settings.
inline Image decode(const std::vector<uint8_t>& f, const std::string& path) {
    using detail::corrupt;
    static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
    if (f.size() < 8 || std::memcmp(f.data(), sig, 8) != 0) corrupt(path, "signature");
    size_t pos = 8;
    uint32_t w = 0, h = 0;
    int depth = 0, ctype = -1, interlace = 0;
    std::vector<std::array<uint8_t, 3>> palette;
    std::vector<uint8_t> idat;
    bool seen_ihdr = false, seen_iend = false;
    while (!seen_iend) {
        if (pos + 12 > f.size()) corrupt(path, "truncated chunk");
        const uint32_t len = be32(&f[pos]);
        if (len > 0x7fffffffu || pos + 12 + size_t(len) > f.size()) corrupt(path, "truncated chunk");
        const uint8_t* type = &f[pos + 4];
        const uint8_t* data = &f[pos + 8];
        const uint32_t crc = be32(&f[pos + 8 + len]);
        if (uint32_t(crc32(crc32(0L, type, 4), data, len)) != crc) corrupt(path, "CRC mismatch");
        const std::string t(reinterpret_cast<const char*>(type), 4);
        if (!seen_ihdr && t != "IHDR") corrupt(path, "IHDR must come first");
        if (t == "IHDR") {
            if (seen_ihdr || len != 13) corrupt(path, "IHDR");
            w = be32(data);
            h = be32(data + 4);
            depth = data[8];
            ctype = data[9];
            interlace = data[12];
            if (depth > 8 && (depth == 16 && (ctype == 0 || ctype == 2 || ctype == 4 || ctype == 6)))
                fail(Errc::unsupported_format, path + ": 16-bit channels not supported");
            const bool ok_combo = (ctype == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                                  (ctype == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                                  ((ctype == 2 || ctype == 4 || ctype == 6) && depth == 8);
            if (!ok_combo || data[10] != 0 || data[11] != 0 || interlace > 1) corrupt(path, "IHDR fields");
            if (w < 1 || h < 1 || w > 0x7fffffffu || h > 0x7fffffffu) corrupt(path, "IHDR size");
            seen_ihdr = true;
        } else if (t == "PLTE") {
            if (len % 3 || len == 0 || len > 768) corrupt(path, "PLTE");
            palette.resize(len / 3);
            for (uint32_t k = 0; k < len / 3; ++k) palette[k] = {data[3 * k], data[3 * k + 1], data[3 * k + 2]};
        } else if (t == "IDAT") {
            idat.insert(idat.end(), data, data + len);
        } else if (t == "IEND") {
            seen_iend = true;
        } else if (!(type[0] & 0x20)) {
            corrupt(path, "unknown critical chunk " + t);  // ancillary chunks (tRNS, gAMA, ...) are skipped
        }
        pos += 12 + size_t(len);
    }
    if (ctype == 3 && palette.empty()) corrupt(path, "palette image without PLTE");
    const int channels = ctype == 2 ? 3 : ctype == 4 ? 2 : ctype == 6 ? 4 : 1;
    const size_t bits = size_t(channels) * depth, bpp = std::max<size_t>(1, bits / 8);
    // Adam7 pass geometry (PNG spec 8.2); one pass covering everything when not interlaced
    struct Pass { int x0, y0, dx, dy; };
    static const Pass adam7[7] = {{0, 0, 8, 8}, {4, 0, 8, 8}, {0, 4, 4, 8}, {2, 0, 4, 4},
                                  {0, 2, 2, 4}, {1, 0, 2, 2}, {0, 1, 1, 2}};
    static const Pass whole = {0, 0, 1, 1};
    const int npass = interlace ? 7 : 1;
    size_t expect = 0;
    for (int p = 0; p < npass; ++p) {
        const Pass& q = interlace ? adam7[p] : whole;
        const size_t pw = w > uint32_t(q.x0) ? (w - q.x0 + q.dx - 1) / q.dx : 0;
        const size_t ph = h > uint32_t(q.y0) ? (h - q.y0 + q.dy - 1) / q.dy : 0;
        if (pw && ph) expect += ph * (1 + (pw * bits + 7) / 8);
    }
    std::vector<uint8_t> raw(expect);
    {
        z_stream zs{};
        if (inflateInit(&zs) != Z_OK) fail(Errc::io_failure, "zlib init failed");
        zs.next_in = idat.data();
        zs.avail_in = uInt(idat.size());
        zs.next_out = raw.data();
        zs.avail_out = uInt(raw.size());
        const int r = inflate(&zs, Z_FINISH);
        const size_t got = raw.size() - zs.avail_out;
        inflateEnd(&zs);
        if ((r != Z_STREAM_END && !(r == Z_BUF_ERROR && zs.avail_out == 0)) || got != expect)
            corrupt(path, "image data stream");
    }
    Image img;
    img.width = int(w);
    img.height = int(h);
    img.rgb.assign(size_t(w) * h * 3, 0);
    const int gray_scale = depth == 1 ? 255 : depth == 2 ? 85 : depth == 4 ? 17 : 1;  // expand_gray_1_2_4_to_8
    size_t off = 0;
    for (int p = 0; p < npass; ++p) {
        const Pass& q = interlace ? adam7[p] : whole;
        const size_t pw = w > uint32_t(q.x0) ? (w - q.x0 + q.dx - 1) / q.dx : 0;
        const size_t ph = h > uint32_t(q.y0) ? (h - q.y0 + q.dy - 1) / q.dy : 0;
        if (!pw || !ph) continue;
        const size_t rb = (pw * bits + 7) / 8;
        const uint8_t* prev = nullptr;
        for (size_t r = 0; r < ph; ++r) {
            uint8_t* line = &raw[off + 1];
            if (!detail::unfilter(raw[off], line, prev, rb, bpp)) corrupt(path, "filter type");
            const size_t y = q.y0 + r * q.dy;
            for (size_t c = 0; c < pw; ++c) {
                uint8_t* d = &img.rgb[(y * w + q.x0 + c * q.dx) * 3];
                auto sample = [&](size_t idx) -> int {  // idx-th sub-byte sample of the line
                    const size_t bit = idx * depth;
                    return (line[bit >> 3] >> (8 - depth - (bit & 7))) & ((1 << depth) - 1);
                };
                switch (ctype) {
                    case 0: {
                        const uint8_t g = uint8_t(depth == 8 ? line[c] : sample(c) * gray_scale);
                        d[0] = d[1] = d[2] = g;
                        break;
                    }
                    case 2: std::memcpy(d, line + 3 * c, 3); break;
                    case 3: {
                        const int idx = depth == 8 ? line[c] : sample(c);
                        // libpng keeps a 256-entry palette; entries past PLTE are black
                        if (size_t(idx) < palette.size()) std::memcpy(d, palette[idx].data(), 3);
                        break;
                    }
                    case 4: d[0] = d[1] = d[2] = line[2 * c]; break;
                    case 6: std::memcpy(d, line + 4 * c, 3); break;
                }
            }
            prev = line;
            off += 1 + rb;
        }
    }
    return img;
}

/// Encode 8-bit RGB (channels = 3) or gray (channels = 1), non-interlaced.
inline std::vector<uint8_t> encode(const uint8_t* px, int width, int height, int channels) {
    const size_t rb = size_t(width) * channels;
    std::vector<uint8_t> raw;
    raw.reserve((rb + 1) * height);
    for (int i = 0; i < height; ++i) {  // filter 1 (Sub) on every row: cheap and compresses well
        raw.push_back(1);
        const uint8_t* row = px + size_t(i) * rb;
        for (size_t k = 0; k < rb; ++k) raw.push_back(uint8_t(row[k] - (k >= size_t(channels) ? row[k - channels] : 0)));
    }
    uLongf zlen = compressBound(uLong(raw.size()));
    std::vector<uint8_t> z(zlen);
    if (compress2(z.data(), &zlen, raw.data(), uLong(raw.size()), 6) != Z_OK) fail(Errc::io_failure, "deflate failed");
    z.resize(zlen);
    std::vector<uint8_t> out = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
    auto chunk = [&](const char* type, const std::vector<uint8_t>& data) {
        put32(out, uint32_t(data.size()));
        const size_t start = out.size();
        out.insert(out.end(), type, type + 4);
        out.insert(out.end(), data.begin(), data.end());
        put32(out, uint32_t(crc32(0L, &out[start], uInt(4 + data.size()))));
    };
    std::vector<uint8_t> ihdr;
    put32(ihdr, uint32_t(width));
    put32(ihdr, uint32_t(height));
    ihdr.insert(ihdr.end(), {8, uint8_t(channels == 3 ? 2 : 0), 0, 0, 0});
    chunk("IHDR", ihdr);
    chunk("IDAT", z);
    chunk("IEND", {});
    return out;
}

inline std::vector<uint8_t> read_file(std::FILE* fp) {
    std::vector<uint8_t> buf;
    uint8_t tmp[1 << 16];
    size_t n;
    while ((n = std::fread(tmp, 1, sizeof tmp, fp)) > 0) buf.insert(buf.end(), tmp, tmp + n);
    return buf;
}

inline void write_file(const std::string& path, const std::vector<uint8_t>& bytes) {
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) fail(Errc::io_failure, path + ": cannot open for writing");
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), fp) == bytes.size();
    std::fclose(fp);
    if (!ok) fail(Errc::io_failure, path + ": PNG write failed");
}

}  // namespace carve::png
