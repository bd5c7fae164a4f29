// io_hgf.cpp — the output formats on either side of the hot path (SURVEY
// §8 f3), host side:
//   * HGF1 field dumps: write_field_dump (src/io.cpp:168-186) and
//     read_field_dump (src/io.cpp:316-345), byte-identical format and the
//     same validation order and messages;
//   * the level <-> 8-bit grey encodings of write_hologram_png /
//     read_hologram_png (src/io.cpp:272-298);
//   * the "<png>.scale.txt" companion of write_replay_png (src/io.cpp:206-207).
// The device-side encodings of resident results (levels and replay → grey)
// are k_levels_gray8 / k_replay_* in capi.cu.  PNG compression itself needs
// libpng, which this image does not have, and stays outside.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

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

}  // extern "C"
