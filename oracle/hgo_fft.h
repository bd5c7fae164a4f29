/*
 * hgo_fft.h — FFT used by the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * The reference's production FFT is FFTW3 (proj/src/fftw_backend.cpp:43-46,
 * :61-64: fftw(f)_plan_dft_2d(ny, nx, ..., FFTW_ESTIMATE|FFTW_UNALIGNED)),
 * which is not installed in this image nor on the GPU box.  FFTW is an
 * un-pinned third-party dependency (proj/CMakeLists.txt:14-17, no version);
 * its published contract is the unnormalised DFT
 *     Y[k] = sum_j X[j] exp(sign * 2*pi*i * j*k / n),  sign = -1 forward.
 * The reference wraps it as: execute (unnormalised, result in T), then
 * out[i] *= (T)(1/sqrt(nx*ny)) in T (fftw_backend.cpp:113-124).
 *
 * This file restates that contract in two flavours:
 *   hgo_fft2d_precise : double-accumulating (radix-2 for powers of two,
 *                       direct per-axis DFT otherwise), rounded to T=float
 *                       once, then scaled in float exactly like
 *                       fftw_backend.cpp:121-123.  Used for parity.
 *   hgo_fft2d_fast    : float Stockham radix-4/2 with precomputed twiddles,
 *                       rows then column blocks.  Used ONLY to time the
 *                       CPU baseline (a stand-in for FFTW's speed, labelled
 *                       as such wherever a CPU number is printed).
 *
 * Both the C restatement (hg_oracle.c) and the reference-headers build
 * (ref_shim.cpp, via default_fft_backend<T>) include this one file, so the
 * restatement and the compiled reference see bit-identical transforms.
 */
#ifndef HGO_FFT_H
#define HGO_FFT_H

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGO_TWO_PI 6.283185307179586476925286766559

static inline int hgo_is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* Twiddle table tw[k] = exp(sign*2*pi*i*k/n), k < n, from the exact angle. */
static double *hgo_twiddles_d(int n, int sign) {
    double *tw = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    for (int k = 0; k < n; ++k) {
        double a = sign * HGO_TWO_PI * (double)k / (double)n;
        tw[2 * k] = cos(a);
        tw[2 * k + 1] = sin(a);
    }
    return tw;
}

/* In-place 1-D transform of n contiguous complex doubles (interleaved).
 * tw from hgo_twiddles_d(n, sign).  Radix-2 DIT for powers of two, direct
 * DFT with (k*j mod n) twiddle indexing otherwise (as fft.hpp:437-447). */
static void hgo_dft_line_d(double *buf, int n, const double *tw, double *scratch) {
    if (n == 1) return;
    if (hgo_is_pow2(n)) {
        for (int i = 1, j = 0; i < n; ++i) {
            int bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) {
                double tr = buf[2 * i], ti = buf[2 * i + 1];
                buf[2 * i] = buf[2 * j];
                buf[2 * i + 1] = buf[2 * j + 1];
                buf[2 * j] = tr;
                buf[2 * j + 1] = ti;
            }
        }
        for (int len = 2; len <= n; len <<= 1) {
            int half = len >> 1, step = n / len;
            for (int k = 0; k < half; ++k) {
                double wr = tw[2 * (size_t)k * step], wi = tw[2 * (size_t)k * step + 1];
                for (int s = 0; s < n; s += len) {
                    double *u = buf + 2 * (s + k), *v = buf + 2 * (s + k + half);
                    double xr = v[0] * wr - v[1] * wi;
                    double xi = v[0] * wi + v[1] * wr;
                    v[0] = u[0] - xr;
                    v[1] = u[1] - xi;
                    u[0] += xr;
                    u[1] += xi;
                }
            }
        }
        return;
    }
    for (int k = 0; k < n; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int j = 0; j < n; ++j) {
            size_t m = ((size_t)k * j) % (size_t)n;
            double wr = tw[2 * m], wi = tw[2 * m + 1];
            ar += buf[2 * j] * wr - buf[2 * j + 1] * wi;
            ai += buf[2 * j] * wi + buf[2 * j + 1] * wr;
        }
        scratch[2 * k] = ar;
        scratch[2 * k + 1] = ai;
    }
    memcpy(buf, scratch, sizeof(double) * 2 * (size_t)n);
}

/* Row then column passes over a double work array. */
static void hgo_fft2d_work(int nx, int ny, int sign, double *w) {
    int m = nx > ny ? nx : ny;
    double *line = (double *)malloc(sizeof(double) * 2 * (size_t)m);
    double *scratch = (double *)malloc(sizeof(double) * 2 * (size_t)m);
    double *twx = hgo_twiddles_d(nx, sign), *twy = hgo_twiddles_d(ny, sign);
    for (int y = 0; y < ny; ++y) hgo_dft_line_d(w + 2 * (size_t)y * nx, nx, twx, scratch);
    for (int x = 0; x < nx; ++x) {
        for (int y = 0; y < ny; ++y) {
            line[2 * y] = w[2 * ((size_t)y * nx + x)];
            line[2 * y + 1] = w[2 * ((size_t)y * nx + x) + 1];
        }
        hgo_dft_line_d(line, ny, twy, scratch);
        for (int y = 0; y < ny; ++y) {
            w[2 * ((size_t)y * nx + x)] = line[2 * y];
            w[2 * ((size_t)y * nx + x) + 1] = line[2 * y + 1];
        }
    }
    free(line);
    free(scratch);
    free(twx);
    free(twy);
}

/* Unnormalised 2-D DFT accumulated in double, rounded to float, then scaled
 * by (float)(1/sqrt(nx*ny)) in float (fftw_backend.cpp:119-123).
 * in == out allowed.  Row-major data[y*nx + x], interleaved floats. */
static void hgo_fft2d_precise(int nx, int ny, int sign, const float *in, float *out) {
    size_t n = (size_t)nx * ny;
    double *w = (double *)malloc(sizeof(double) * 2 * n);
    for (size_t i = 0; i < 2 * n; ++i) w[i] = (double)in[i];
    hgo_fft2d_work(nx, ny, sign, w);
    float norm = (float)(1.0 / sqrt((double)nx * ny));
    for (size_t i = 0; i < 2 * n; ++i) {
        float v = (float)w[i];
        out[i] = v * norm;
    }
    free(w);
}

/* Same contract, double in / double out (for T=double reference builds). */
static void hgo_fft2d_precise_d(int nx, int ny, int sign, const double *in, double *out) {
    size_t n = (size_t)nx * ny;
    double *w = (double *)malloc(sizeof(double) * 2 * n);
    memcpy(w, in, sizeof(double) * 2 * n);
    hgo_fft2d_work(nx, ny, sign, w);
    double norm = 1.0 / sqrt((double)nx * ny);
    for (size_t i = 0; i < 2 * n; ++i) out[i] = w[i] * norm;
    free(w);
}

/* ---- fast float path (CPU-baseline timing only) ------------------------ */

/* One Stockham radix-2/4 transform of a contiguous line of n (pow2) complex
 * floats; x and y are ping-pong buffers, result returned pointer.  tw holds
 * exp(sign*2*pi*i*k/n) for k < n. */
static float *hgo_stockham_f(float *x, float *y, int n, const float *tw) {
    int l = 1; /* current sub-transform length */
    while (l < n) {
        int rem = n / l;
        if (rem % 4 == 0) {
            int m = n / 4; /* butterflies */
            int stride = n / (4 * l);
            for (int j = 0; j < l; ++j) {
                const float *w1 = tw + 2 * (size_t)(j * stride);
                const float *w2 = tw + 2 * (size_t)(2 * j * stride);
                const float *w3 = tw + 2 * (size_t)(3 * j * stride);
                float w1r = w1[0], w1i = w1[1], w2r = w2[0], w2i = w2[1], w3r = w3[0], w3i = w3[1];
                for (int k = 0; k < rem / 4; ++k) {
                    const float *a = x + 2 * (size_t)(j + l * k);
                    const float *b = a + 2 * (size_t)m;
                    const float *c = b + 2 * (size_t)m;
                    const float *d = c + 2 * (size_t)m;
                    /* twiddle inputs 1..3 */
                    float br = b[0] * w1r - b[1] * w1i, bi = b[0] * w1i + b[1] * w1r;
                    float cr = c[0] * w2r - c[1] * w2i, ci = c[0] * w2i + c[1] * w2r;
                    float dr = d[0] * w3r - d[1] * w3i, di = d[0] * w3i + d[1] * w3r;
                    float t0r = a[0] + cr, t0i = a[1] + ci;
                    float t1r = a[0] - cr, t1i = a[1] - ci;
                    float t2r = br + dr, t2i = bi + di;
                    float t3r = br - dr, t3i = bi - di;
                    /* multiply t3 by sign*i: forward sign=-1 -> -i */
                    float sr, si;
                    if (tw[2 * (size_t)(n / 4) + 1] < 0) { sr = t3i; si = -t3r; }
                    else { sr = -t3i; si = t3r; }
                    float *o = y + 2 * (size_t)(j + 4 * l * k);
                    o[0] = t0r + t2r; o[1] = t0i + t2i;
                    o[2 * l] = t1r + sr; o[2 * l + 1] = t1i + si;
                    o[4 * l] = t0r - t2r; o[4 * l + 1] = t0i - t2i;
                    o[6 * l] = t1r - sr; o[6 * l + 1] = t1i - si;
                }
            }
            l *= 4;
        } else {
            int m = n / 2;
            int stride = n / (2 * l);
            for (int j = 0; j < l; ++j) {
                const float *w1 = tw + 2 * (size_t)(j * stride);
                float wr = w1[0], wi = w1[1];
                for (int k = 0; k < rem / 2; ++k) {
                    const float *a = x + 2 * (size_t)(j + l * k);
                    const float *b = a + 2 * (size_t)m;
                    float br = b[0] * wr - b[1] * wi, bi = b[0] * wi + b[1] * wr;
                    float *o = y + 2 * (size_t)(j + 2 * l * k);
                    o[0] = a[0] + br; o[1] = a[1] + bi;
                    o[2 * l] = a[0] - br; o[2 * l + 1] = a[1] - bi;
                }
            }
            l *= 2;
        }
        float *t = x; x = y; y = t;
    }
    return x;
}

/* Float 2-D transform for pow2 sizes; non-pow2 falls back to the precise
 * path.  Same normalisation as fftw_backend.cpp:121-123. */
static void hgo_fft2d_fast(int nx, int ny, int sign, const float *in, float *out) {
    if (!hgo_is_pow2(nx) || !hgo_is_pow2(ny)) { hgo_fft2d_precise(nx, ny, sign, in, out); return; }
    size_t n = (size_t)nx * ny;
    int m = nx > ny ? nx : ny;
    const int B = 8; /* column block */
    float *twx = (float *)malloc(sizeof(float) * 2 * (size_t)nx);
    float *twy = (float *)malloc(sizeof(float) * 2 * (size_t)ny);
    for (int k = 0; k < nx; ++k) {
        double a = sign * HGO_TWO_PI * (double)k / nx;
        twx[2 * k] = (float)cos(a); twx[2 * k + 1] = (float)sin(a);
    }
    for (int k = 0; k < ny; ++k) {
        double a = sign * HGO_TWO_PI * (double)k / ny;
        twy[2 * k] = (float)cos(a); twy[2 * k + 1] = (float)sin(a);
    }
    float *b0 = (float *)malloc(sizeof(float) * 2 * (size_t)m * B);
    float *b1 = (float *)malloc(sizeof(float) * 2 * (size_t)m * B);
    if (out != in) memcpy(out, in, sizeof(float) * 2 * n);
    for (int y = 0; y < ny; ++y) {
        float *row = out + 2 * (size_t)y * nx;
        memcpy(b0, row, sizeof(float) * 2 * (size_t)nx);
        float *r = hgo_stockham_f(b0, b1, nx, twx);
        memcpy(row, r, sizeof(float) * 2 * (size_t)nx);
    }
    for (int x0 = 0; x0 < nx; x0 += B) {
        int bw = nx - x0 < B ? nx - x0 : B;
        for (int c = 0; c < bw; ++c) {
            float *col = b0 + 2 * (size_t)c * ny;
            for (int y = 0; y < ny; ++y) {
                col[2 * y] = out[2 * ((size_t)y * nx + x0 + c)];
                col[2 * y + 1] = out[2 * ((size_t)y * nx + x0 + c) + 1];
            }
        }
        for (int c = 0; c < bw; ++c) {
            float *col = b0 + 2 * (size_t)c * ny;
            float *alt = b1 + 2 * (size_t)c * ny;
            float *r = hgo_stockham_f(col, alt, ny, twy);
            if (r != col) memcpy(col, r, sizeof(float) * 2 * (size_t)ny);
        }
        for (int c = 0; c < bw; ++c) {
            float *col = b0 + 2 * (size_t)c * ny;
            for (int y = 0; y < ny; ++y) {
                out[2 * ((size_t)y * nx + x0 + c)] = col[2 * y];
                out[2 * ((size_t)y * nx + x0 + c) + 1] = col[2 * y + 1];
            }
        }
    }
    float norm = (float)(1.0 / sqrt((double)nx * ny));
    for (size_t i = 0; i < 2 * n; ++i) out[i] *= norm;
    free(twx); free(twy); free(b0); free(b1);
}

#ifdef __cplusplus
}
#endif
#endif
