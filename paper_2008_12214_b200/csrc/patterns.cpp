// patterns.cpp — the benchmark target generator, host side: the reference's
// patterns::smooth_blobs (patterns.hpp:55-80) and normalize_image
// (target.hpp:15-30) restated in C++ with the same operation order and the C
// library's exp, so the synthetic targets are bit-identical to the ones the
// reference's own bench builds (bench.cpp:115-116).
#include <cmath>
#include <cstddef>

#include "../../include/hologen_b200.h"

extern "C" {

int hgc_smooth_blobs(int width, int height, double* out) {
    if (width < 1 || height < 1 || !out) return HGC_EINVAL;
    struct Blob {
        double cx, cy, sigma, amp;
    };
    static constexpr Blob blobs[] = {
        {0.30, 0.35, 0.16, 1.00},
        {0.68, 0.28, 0.10, 0.75},
        {0.62, 0.70, 0.20, 0.90},
        {0.22, 0.74, 0.08, 0.60},
    };
    for (int y = 0; y < height; ++y) {
        const double fy = (y + 0.5) / height;
        for (int x = 0; x < width; ++x) {
            const double fx = (x + 0.5) / width;
            double v = 0.08 + 0.10 * fx + 0.06 * fy;
            for (const Blob& b : blobs) {
                const double dx = fx - b.cx, dy = fy - b.cy;
                v += b.amp * std::exp(-(dx * dx + dy * dy) / (2.0 * b.sigma * b.sigma));
            }
            out[static_cast<size_t>(y) * width + x] = v;
        }
    }
    return hgc_normalize_image(out, static_cast<size_t>(width) * height, 0);
}

int hgc_normalize_image(double* img, size_t n, int unit_energy) {
    if (!img && n) return HGC_EINVAL;
    double acc = 0.0;
    if (!unit_energy) {
        for (size_t i = 0; i < n; ++i) acc = img[i] > acc ? img[i] : acc;
        if (acc == 0.0) return HGC_OK;  // all-black stays all-black
    } else {
        for (size_t i = 0; i < n; ++i) acc += img[i] * img[i];
        if (acc <= 0.0) return HGC_EINVAL;  // "normalize_image: zero-energy image cannot be energy-normalized"
    }
    const double s = !unit_energy ? 1.0 / acc : std::sqrt(static_cast<double>(n) / acc);
    for (size_t i = 0; i < n; ++i) img[i] *= s;
    return HGC_OK;
}

}  // extern "C"
