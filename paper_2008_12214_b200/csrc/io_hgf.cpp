// io_hgf.cpp — the output formats on either side of the hot path (SURVEY
// §8 f3), host side:
//   * HGF1 field dumps: write_field_dump (src/io.cpp:168-186) and
//     read_field_dump (src/io.cpp:316-345), byte-identical format and the
//     same validation order and messages;
//   * the level <-> 8-bit grey encodings of write_hologram_png /
//     read_hologram_png (src/io.cpp:272-298);
//   * the "<png>.scale.txt" companion of write_replay_png (src/io.cpp:206-207).
// The device-side encodings of resident results (levels and replay → grey)
// are k_levels_gray8 / k_replay_* in capi.cu.
//   * PNG files: 8-bit greyscale, non-interlaced (what write_png_gray hands to
//     libpng's simplified API, io.cpp:221-237), written with zlib (deflate)
//     and CRC-32 chunks; the reader takes any 8-bit greyscale PNG
//     (all five scanline filters), as read_png_gray8 (io.cpp:239-258) does
//     through libpng.  libpng itself is absent from this image.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include <zlib.h>

#include "../../include/hologen_b200.h"
#include "errors.h"

namespace hg {
extern thread_local std::string g_err;  // capi.cu
}

namespace {

using hg::Failure;

[[noreturn]] void io_fail(const std::string& msg) { hg::fail(HGC_EIO, msg); }  // io.cpp:16 (runtime_error)

template <class F>
int io_guarded(F&& f) {
    try {
        f();
        return HGC_OK;
    } catch (const Failure& e) {
        hg::g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        hg::g_err = "host allocation failed";
        return HGC_EIO;
    } catch (const std::exception& e) {
        hg::g_err = e.what();
        return HGC_EIO;
    }
}

std::vector<uint8_t> read_file(const std::string& path) {  // io.cpp:18-25
    std::ifstream in(path, std::ios::binary);
    if (!in) io_fail("cannot open file: " + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) io_fail("read error: " + path);
    return bytes;
}

void write_file(const std::string& path, const uint8_t* data, size_t size) {  // io.cpp:27-32
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) io_fail("cannot create file: " + path);
    out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(size));
    if (!out) io_fail("write error: " + path);
}

void put_u32le(std::vector<uint8_t>& b, uint32_t v) {
    for (int k = 0; k < 4; ++k) b.push_back(static_cast<uint8_t>(v >> (8 * k)));
}
uint32_t get_u32le(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
           (static_cast<uint32_t>(p[3]) << 24);
}
// little-endian IEEE payload: bytewise, so the format is host-order independent
template <class T>
void put_le(std::vector<uint8_t>& b, T v) {
    uint8_t raw[sizeof(T)];
    std::memcpy(raw, &v, sizeof(T));
    uint64_t u = 0;
    std::memcpy(&u, raw, sizeof(T));
    for (size_t k = 0; k < sizeof(T); ++k) b.push_back(static_cast<uint8_t>(u >> (8 * k)));
}
template <class T>
T get_le(const uint8_t* p) {
    uint64_t u = 0;
    for (size_t k = 0; k < sizeof(T); ++k) u |= static_cast<uint64_t>(p[k]) << (8 * k);
    T v;
    std::memcpy(&v, &u, sizeof(T));
    return v;
}

std::string shortest(double v) {  // detail::format_double, numfmt.hpp:11-16
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof buf, v);
    if (res.ec != std::errc()) io_fail("format_double failed");
    return std::string(buf, res.ptr);
}

// ------------------------------------------------------------------ PNG
const uint8_t kPngSig[8] = {0x89, 'P', 'N', 'G', 0x0D, 0x0A, 0x1A, 0x0A};

void put_be32(std::vector<uint8_t>& out, uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) out.push_back(static_cast<uint8_t>(v >> s));
}
uint32_t get_be32(const uint8_t* p) {
    return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | (uint32_t)p[3];
}
void put_chunk(std::vector<uint8_t>& out, const char* type, const uint8_t* data, size_t n) {
    put_be32(out, static_cast<uint32_t>(n));
    const size_t at = out.size();
    out.insert(out.end(), type, type + 4);
    if (n) out.insert(out.end(), data, data + n);
    put_be32(out, static_cast<uint32_t>(crc32(crc32(0L, Z_NULL, 0), out.data() + at, static_cast<uInt>(n + 4))));
}

std::vector<uint8_t> encode_png_gray(const uint8_t* px, int w, int h) {
    std::vector<uint8_t> raw(static_cast<size_t>(w + 1) * h);
    for (int y = 0; y < h; ++y) {  // filter type 0 on every scanline
        raw[static_cast<size_t>(y) * (w + 1)] = 0;
        std::memcpy(&raw[static_cast<size_t>(y) * (w + 1) + 1], px + static_cast<size_t>(y) * w, w);
    }
    uLongf zn = compressBound(static_cast<uLong>(raw.size()));
    std::vector<uint8_t> z(zn);
    if (compress2(z.data(), &zn, raw.data(), static_cast<uLong>(raw.size()), 6) != Z_OK)
        io_fail("png encode failed: deflate error");
    std::vector<uint8_t> out(kPngSig, kPngSig + 8);
    uint8_t ihdr[13];
    for (int i = 0; i < 4; ++i) {
        ihdr[i] = static_cast<uint8_t>(static_cast<uint32_t>(w) >> (24 - 8 * i));
        ihdr[4 + i] = static_cast<uint8_t>(static_cast<uint32_t>(h) >> (24 - 8 * i));
    }
    ihdr[8] = 8;   // bit depth
    ihdr[9] = 0;   // greyscale
    ihdr[10] = 0;  // deflate
    ihdr[11] = 0;  // adaptive filtering
    ihdr[12] = 0;  // no interlace
    put_chunk(out, "IHDR", ihdr, 13);
    put_chunk(out, "IDAT", z.data(), zn);
    put_chunk(out, "IEND", nullptr, 0);
    return out;
}

std::vector<uint8_t> decode_png_gray8(const std::vector<uint8_t>& b, const std::string& path, int* w, int* h) {
    if (b.size() < 8 || std::memcmp(b.data(), kPngSig, 8) != 0) io_fail("not a PNG file: " + path);
    size_t at = 8;
    int W = 0, H = 0, depth = 0, ctype = -1, interlace = 0;
    std::vector<uint8_t> z;
    while (at + 12 <= b.size()) {
        const uint32_t n = get_be32(&b[at]);
        if (at + 12 + n > b.size()) break;
        const char* type = reinterpret_cast<const char*>(&b[at + 4]);
        const uint8_t* d = &b[at + 8];
        if (std::memcmp(type, "IHDR", 4) == 0 && n >= 13) {
            W = static_cast<int>(get_be32(d));
            H = static_cast<int>(get_be32(d + 4));
            depth = d[8];
            ctype = d[9];
            interlace = d[12];
        } else if (std::memcmp(type, "IDAT", 4) == 0) {
            z.insert(z.end(), d, d + n);
        } else if (std::memcmp(type, "IEND", 4) == 0) {
            break;
        }
        at += 12 + n;
    }
    if (W < 1 || H < 1) io_fail("png decode failed (" + path + "): missing IHDR");
    if (depth != 8 || ctype != 0 || interlace != 0)
        io_fail("png decode failed (" + path + "): only 8-bit greyscale non-interlaced images are supported");
    const size_t stride = static_cast<size_t>(W) + 1;
    std::vector<uint8_t> raw(stride * H);
    uLongf rn = static_cast<uLongf>(raw.size());
    if (uncompress(raw.data(), &rn, z.data(), static_cast<uLong>(z.size())) != Z_OK || rn != raw.size())
        io_fail("png decode failed (" + path + "): corrupt image data");
    std::vector<uint8_t> px(static_cast<size_t>(W) * H);
    for (int y = 0; y < H; ++y) {  // undo the scanline filters (PNG spec §9)
        const uint8_t f = raw[y * stride];
        const uint8_t* s = &raw[y * stride + 1];
        uint8_t* o = &px[static_cast<size_t>(y) * W];
        const uint8_t* up = y ? o - W : nullptr;
        for (int x = 0; x < W; ++x) {
            const int a = x ? o[x - 1] : 0, bb = up ? up[x] : 0, c = (x && up) ? up[x - 1] : 0;
            int v;
            switch (f) {
                case 0: v = s[x]; break;
                case 1: v = s[x] + a; break;
                case 2: v = s[x] + bb; break;
                case 3: v = s[x] + ((a + bb) >> 1); break;
                case 4: {
                    const int p = a + bb - c, pa = std::abs(p - a), pb = std::abs(p - bb), pc = std::abs(p - c);
                    v = s[x] + ((pa <= pb && pa <= pc) ? a : (pb <= pc ? bb : c));
                    break;
                }
                default: io_fail("png decode failed (" + path + "): bad scanline filter");
            }
            o[x] = static_cast<uint8_t>(v);
        }
    }
    *w = W;
    *h = H;
    return px;
}

}  // namespace

extern "C" {

int hgc_write_field_dump(const char* path, int nx, int ny, int precision, const void* data) {
    return io_guarded([&] {
        if (!path || !data) hg::invalid("field dump: null argument");
        if (nx <= 0 || ny <= 0) hg::invalid("ComplexField: dimensions must be positive");
        if (precision != 4 && precision != 8) hg::invalid("field dump: precision must be 4 (float) or 8 (double)");
        const size_t n = static_cast<size_t>(nx) * ny;
        std::vector<uint8_t> out;
        out.reserve(13 + n * 2 * precision);
        out.insert(out.end(), {'H', 'G', 'F', '1'});
        put_u32le(out, static_cast<uint32_t>(nx));
        put_u32le(out, static_cast<uint32_t>(ny));
        out.push_back(static_cast<uint8_t>(precision));
        if (precision == 4) {
            const float* f = static_cast<const float*>(data);
            for (size_t i = 0; i < 2 * n; ++i)  // require_finite(f, "field dump"), field.hpp:107-110
                if (!std::isfinite(f[i])) hg::invalid("field dump: field contains non-finite values");
            for (size_t i = 0; i < 2 * n; ++i) put_le<float>(out, f[i]);
        } else {
            const double* f = static_cast<const double*>(data);
            for (size_t i = 0; i < 2 * n; ++i)
                if (!std::isfinite(f[i])) hg::invalid("field dump: field contains non-finite values");
            for (size_t i = 0; i < 2 * n; ++i) put_le<double>(out, f[i]);
        }
        write_file(path, out.data(), out.size());
    });
}

int hgc_read_field_dump(const char* path, int* nx, int* ny, int* precision, void* data) {
    return io_guarded([&] {
        if (!path) hg::invalid("field dump: null path");
        const std::string p(path);
        const std::vector<uint8_t> b = read_file(p);
        if (b.size() < 13 || std::memcmp(b.data(), "HGF1", 4) != 0) io_fail("not an HGF1 field dump: " + p);
        const uint32_t w = get_u32le(b.data() + 4), h = get_u32le(b.data() + 8);
        const uint8_t code = b[12];
        if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20)) io_fail("HGF1: implausible dimensions in " + p);
        if (code == 2) io_fail("HGF1: 16-bit fields are not enabled in this build: " + p);
        if (code != 4 && code != 8) io_fail("HGF1: unknown precision code " + std::to_string(code) + " in " + p);
        const size_t count = static_cast<size_t>(w) * h;
        const size_t expected = 13 + count * 2 * code;
        if (b.size() != expected)
            io_fail("HGF1: size mismatch (expected " + std::to_string(expected) + " bytes) in " + p);
        if (nx) *nx = static_cast<int>(w);
        if (ny) *ny = static_cast<int>(h);
        if (precision) *precision = code;
        if (!data) return;  // header query
        const uint8_t* q = b.data() + 13;
        if (code == 4) {
            float* f = static_cast<float*>(data);
            for (size_t i = 0; i < 2 * count; ++i, q += 4) f[i] = get_le<float>(q);
            for (size_t i = 0; i < 2 * count; ++i)
                if (!std::isfinite(f[i])) hg::invalid("field dump " + p + ": field contains non-finite values");
        } else {
            double* f = static_cast<double*>(data);
            for (size_t i = 0; i < 2 * count; ++i, q += 8) f[i] = get_le<double>(q);
            for (size_t i = 0; i < 2 * count; ++i)
                if (!std::isfinite(f[i])) hg::invalid("field dump " + p + ": field contains non-finite values");
        }
    });
}

int hgc_levels_to_gray8(const int32_t* levels, int width, int height, int level_count, uint8_t* out) {
    return io_guarded([&] {
        if (level_count < 2 || level_count > 256)
            hg::invalid("write_hologram_png: level count must be in [2, 256] for a lossless 8-bit encoding");
        if (width < 1 || height < 1 || !levels || !out)
            hg::invalid("write_hologram_png: level buffer does not match dimensions");
        const size_t n = static_cast<size_t>(width) * height;
        for (size_t i = 0; i < n; ++i) {
            if (levels[i] < 0 || levels[i] >= level_count)
                hg::invalid("write_hologram_png: level index out of range");
            out[i] = static_cast<uint8_t>(std::lround(255.0 * levels[i] / (level_count - 1)));
        }
    });
}

int hgc_gray8_to_levels(const uint8_t* px, size_t n, int level_count, int32_t* out) {
    return io_guarded([&] {
        if (level_count < 2 || level_count > 256) hg::invalid("read_hologram_png: level count must be in [2, 256]");
        if (!px || !out) hg::invalid("read_hologram_png: null buffer");
        for (size_t i = 0; i < n; ++i) out[i] = static_cast<int32_t>(std::lround(px[i] * (level_count - 1) / 255.0));
    });
}

int hgc_write_replay_scale(const char* png_path, double peak) {
    return io_guarded([&] {
        if (!png_path) hg::invalid("replay scale: null path");
        const std::string text = "amplitude_at_255=" + shortest(peak) + "\n";
        write_file(std::string(png_path) + ".scale.txt", reinterpret_cast<const uint8_t*>(text.data()), text.size());
    });
}

int hgc_write_png_gray(const char* path, const uint8_t* pixels, int width, int height) {  // io.cpp:221-237
    return io_guarded([&] {
        if (width < 1 || height < 1 || !pixels)
            hg::fail(HGC_EINVAL, "write_png_gray: pixel buffer does not match dimensions");
        const std::vector<uint8_t> png = encode_png_gray(pixels, width, height);
        write_file(path, png.data(), png.size());
    });
}

int hgc_read_png_gray8(const char* path, int* width, int* height, uint8_t* pixels) {  // io.cpp:239-258
    return io_guarded([&] {
        int w = 0, h = 0;
        const std::vector<uint8_t> px = decode_png_gray8(read_file(path), path, &w, &h);
        if (width) *width = w;
        if (height) *height = h;
        if (pixels) std::memcpy(pixels, px.data(), px.size());
    });
}

}  // extern "C"
