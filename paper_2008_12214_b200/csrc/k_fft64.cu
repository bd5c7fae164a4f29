// k_fft64.cu — the double-precision 2-D transform behind FftBackend<double>
// (fft.hpp:17-27; FftwBackend's double plans, fftw_backend.cpp:43-46, scaled
// by 1/sqrt(nx*ny) in double, :121-123) — SURVEY §8 f4.
//
// The same register/shared-memory Stockham core as the f32 hot path
// (fft.cuh, instantiated on double2) with 8 elements per thread, so a 4096
// line keeps 32 registers of data.  Row-major layout (ComplexField<double>),
// rows pass then columns pass, the unitary scale applied by the last pass.
#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <mutex>

#include "errors.h"
#include "fft.cuh"
#include "launch.h"

namespace hg {

namespace {

constexpr int kEM64 = 8;

__global__ void k_init_twiddles64(double2* tw) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 1 || idx >= 2 * kMaxLine) return;
    int N = 1;
    while (N * 2 <= idx) N *= 2;
    const int m = idx - N;
    double s, c;
    sincospi(-2.0 * (double)m / (double)N, &s, &c);
    tw[idx] = make_double2(c, s);
}

const double2* device_twiddles64() {
    static std::mutex mu;
    static std::map<int, double2*> tables;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = tables.find(dev);
    if (it != tables.end()) return it->second;
    double2* tw = nullptr;
    CK(cudaMalloc(&tw, sizeof(double2) * 2 * kMaxLine));
    k_init_twiddles64<<<(2 * kMaxLine + 255) / 256, 256>>>(tw);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    tables[dev] = tw;
    return tw;
}

template <int N>
struct Cfg64 {
    static constexpr int E = LineCfg<N, kEM64>::E, T = LineCfg<N, kEM64>::T;
    static constexpr int LINES = T >= 256 ? 1 : 256 / T;  // lines per CTA
    static constexpr int SMEM = N > E ? LINES * PaddedLen<N>::value * (int)sizeof(double2) : 0;
};

// Rows: LINES rows per CTA, contiguous per row.
template <int NX, int SIGN>
__global__ void __launch_bounds__(Cfg64<NX>::T * Cfg64<NX>::LINES) k_fft64_rows(double2* f, int ny, size_t bstride,
                                                                                 double norm, const double2* tw) {
    using C = Cfg64<NX>;
    constexpr int E = C::E, T = C::T;
    extern __shared__ __align__(16) double2 sm64[];
    const int lr = threadIdx.x / T, t = threadIdx.x % T;
    const int y = blockIdx.x * C::LINES + lr;
    const bool valid = y < ny;  // absent rows still join the CTA's barriers
    double2* row = f + bstride * blockIdx.y + (size_t)(valid ? y : 0) * NX;
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = row[t + e * T];
    fft_line<NX, SIGN, kEM64>(v, t, sm64, RowSmemIdx{lr * PaddedLen<NX>::value}, tw);
    if (!valid) return;
#pragma unroll
    for (int e = 0; e < E; ++e) row[t + e * T] = norm != 0.0 ? make_double2(v[e].x * norm, v[e].y * norm) : v[e];
}

// Columns: CC adjacent columns per CTA (interleaved in smem).
template <int NY, int CC, int SIGN>
__global__ void __launch_bounds__(Cfg64<NY>::T * CC) k_fft64_cols(double2* f, int nx, size_t bstride, double norm,
                                                                   const double2* tw) {
    constexpr int E = Cfg64<NY>::E, T = Cfg64<NY>::T;
    extern __shared__ __align__(16) double2 sm64[];
    const int c = threadIdx.x % CC, t = threadIdx.x / CC;
    const int x = blockIdx.x * CC + c;
    double2* col = f + bstride * blockIdx.y + x;
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = col[(size_t)(t + e * T) * nx];
    fft_line<NY, SIGN, kEM64>(v, t, sm64, ColSmemIdx<CC>{c}, tw);
#pragma unroll
    for (int e = 0; e < E; ++e)
        col[(size_t)(t + e * T) * nx] = norm != 0.0 ? make_double2(v[e].x * norm, v[e].y * norm) : v[e];
}

template <class K>
void allow_smem(K k, int bytes) {
    if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <int NX, int SIGN>
void rows64(double2* f, int ny, int batch, size_t bstride, double norm, const double2* tw, cudaStream_t st) {
    using C = Cfg64<NX>;
    auto k = k_fft64_rows<NX, SIGN>;
    allow_smem(k, C::SMEM);
    k<<<dim3((ny + C::LINES - 1) / C::LINES, batch), C::T * C::LINES, C::SMEM, st>>>(f, ny, bstride, norm, tw);
    CK(cudaGetLastError());
}

template <int NY, int CC, int SIGN>
void cols64_c(double2* f, int nx, int batch, size_t bstride, double norm, const double2* tw, cudaStream_t st) {
    constexpr int smem = NY > Cfg64<NY>::E ? PaddedLen<NY>::value * CC * (int)sizeof(double2) : 0;
    auto k = k_fft64_cols<NY, CC, SIGN>;
    allow_smem(k, smem);
    k<<<dim3(nx / CC, batch), Cfg64<NY>::T * CC, smem, st>>>(f, nx, bstride, norm, tw);
    CK(cudaGetLastError());
}

template <int NY, int SIGN>
void cols64(double2* f, int nx, int batch, size_t bstride, double norm, const double2* tw, cudaStream_t st) {
    // up to ~64 KiB of columns per CTA, at most 1024 threads and nx columns
    constexpr int CMAX0 = 4096 / NY < 1 ? 1 : (4096 / NY > 16 ? 16 : 4096 / NY);
    constexpr int CMAX = Cfg64<NY>::T * CMAX0 > 1024 ? 1024 / Cfg64<NY>::T : CMAX0;
    const int cc = nx < CMAX ? nx : CMAX;
    switch (cc) {
        case 1: cols64_c<NY, 1, SIGN>(f, nx, batch, bstride, norm, tw, st); break;
        case 2: if constexpr (CMAX >= 2) cols64_c<NY, 2, SIGN>(f, nx, batch, bstride, norm, tw, st); break;
        case 4: if constexpr (CMAX >= 4) cols64_c<NY, 4, SIGN>(f, nx, batch, bstride, norm, tw, st); break;
        case 8: if constexpr (CMAX >= 8) cols64_c<NY, 8, SIGN>(f, nx, batch, bstride, norm, tw, st); break;
        case 16: if constexpr (CMAX >= 16) cols64_c<NY, 16, SIGN>(f, nx, batch, bstride, norm, tw, st); break;
        default: fail(HGC_EUNSUPPORTED, "fft64: column tile unsupported");
    }
}

template <int SIGN>
void rows64_any(int nx, double2* f, int ny, int batch, size_t bs, double norm, const double2* tw, cudaStream_t st) {
    switch (nx) {
#define HG_R64(N) \
    case N: rows64<N, SIGN>(f, ny, batch, bs, norm, tw, st); break;
        HG_R64(2) HG_R64(4) HG_R64(8) HG_R64(16) HG_R64(32) HG_R64(64) HG_R64(128) HG_R64(256) HG_R64(512)
        HG_R64(1024) HG_R64(2048) HG_R64(4096)
#undef HG_R64
        default: fail(HGC_EUNSUPPORTED, "fft64: row length unsupported");
    }
}
template <int SIGN>
void cols64_any(int ny, double2* f, int nx, int batch, size_t bs, double norm, const double2* tw, cudaStream_t st) {
    switch (ny) {
#define HG_C64(N) \
    case N: cols64<N, SIGN>(f, nx, batch, bs, norm, tw, st); break;
        HG_C64(2) HG_C64(4) HG_C64(8) HG_C64(16) HG_C64(32) HG_C64(64) HG_C64(128) HG_C64(256) HG_C64(512)
        HG_C64(1024) HG_C64(2048) HG_C64(4096)
#undef HG_C64
        default: fail(HGC_EUNSUPPORTED, "fft64: column length unsupported");
    }
}

bool pow2_line(int n) { return n >= 2 && n <= kMaxLine && (n & (n - 1)) == 0; }

// ------------------------------------------------------------ Bluestein
// A line of any length N <= 2048 (FftBackend accepts any nx, ny >= 1,
// fft.hpp:17-27): X_k = w_k * sum_n (x_n w_n) conj(w_{k-n}), w_n =
// exp(SIGN i pi n^2 / N), as a length-M circular convolution (M = 2^j >=
// 2N - 1) through the power-of-two transforms above, all in double.
__device__ __forceinline__ double2 chirp(long long n, int N, int sign) {
    const long long r = (n * n) % (2LL * N);  // exp(i pi r / N) is 2N-periodic in n^2
    double s, c;
    sincospi((double)sign * (double)r / (double)N, &s, &c);
    return make_double2(c, s);
}
__global__ void k_blu_pre(const double2* in, int N, int M, size_t lines, int sign, double2* a) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < lines * M; i += (size_t)gridDim.x * blockDim.x) {
        const size_t l = i / M;
        const int n = (int)(i % M);
        double2 v = make_double2(0.0, 0.0);
        if (n < N) {
            const double2 x = in[l * N + n], w = chirp(n, N, sign);
            v = make_double2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x);
        }
        a[i] = v;
    }
}
__global__ void k_blu_kernel(int N, int M, int sign, double2* b) {  // conj(w_n) at n and M - n
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < M; n += gridDim.x * blockDim.x) {
        double2 v = make_double2(0.0, 0.0);
        const int m = n < N ? n : (M - n < N ? M - n : -1);
        if (m >= 0) {
            const double2 w = chirp(m, N, sign);
            v = make_double2(w.x, -w.y);
        }
        b[n] = v;
    }
}
__global__ void k_blu_mul(double2* a, const double2* bh, int M, size_t lines) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < lines * M; i += (size_t)gridDim.x * blockDim.x) {
        const double2 x = a[i], y = bh[i % M];
        a[i] = make_double2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
    }
}
__global__ void k_blu_post(const double2* a, int N, int M, size_t lines, int sign, double2* out) {
    const double inv = 1.0 / M;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < lines * N; i += (size_t)gridDim.x * blockDim.x) {
        const size_t l = i / N;
        const int k = (int)(i % N);
        const double2 x = a[l * M + k], w = chirp(k, N, sign);
        out[i] = make_double2((x.x * w.x - x.y * w.y) * inv, (x.x * w.y + x.y * w.x) * inv);
    }
}
__global__ void k_transpose64(const double2* in, int w, int h, size_t batch, double2* out) {  // [b][h][w] -> [b][w][h]
    const size_t n = (size_t)w * h;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n * batch; i += (size_t)gridDim.x * blockDim.x) {
        const size_t b = i / n, r = i % n, y = r / w, x = r % w;
        out[b * n + x * h + y] = in[i];
    }
}
dim3 grid_for(size_t n) { return dim3((unsigned)std::min<size_t>((n + 255) / 256, 148 * 16)); }

struct DevBuf64 {
    double2* p = nullptr;
    explicit DevBuf64(size_t n) { CK(cudaMalloc(&p, sizeof(double2) * (n ? n : 1))); }
    ~DevBuf64() { cudaFree(p); }
};

// Unnormalised transform of `lines` contiguous lines of length N, in place.
void lines64(double2* f, int N, size_t lines, int sign, const double2* tw, cudaStream_t st) {
    if (N == 1) return;
    if (pow2_line(N)) {
        if (sign < 0) rows64_any<-1>(N, f, (int)lines, 1, 0, 0.0, tw, st);
        else rows64_any<+1>(N, f, (int)lines, 1, 0, 0.0, tw, st);
        return;
    }
    if (N > kMaxLine / 2) fail(HGC_EUNSUPPORTED, "fft: non-power-of-two length " + std::to_string(N) + " > 2048");
    int M = 1;
    while (M < 2 * N - 1) M *= 2;
    DevBuf64 a(lines * M), b(M);
    k_blu_kernel<<<grid_for(M), 256, 0, st>>>(N, M, sign, b.p);
    rows64_any<-1>(M, b.p, 1, 1, 0, 0.0, tw, st);
    k_blu_pre<<<grid_for(lines * M), 256, 0, st>>>(f, N, M, lines, sign, a.p);
    rows64_any<-1>(M, a.p, (int)lines, 1, 0, 0.0, tw, st);
    k_blu_mul<<<grid_for(lines * M), 256, 0, st>>>(a.p, b.p, M, lines);
    rows64_any<+1>(M, a.p, (int)lines, 1, 0, 0.0, tw, st);
    k_blu_post<<<grid_for(lines * N), 256, 0, st>>>(a.p, N, M, lines, sign, f);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));  // a, b are freed on return
}

__global__ void k_scale64(double2* f, size_t n, double s) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        f[i] = make_double2(f[i].x * s, f[i].y * s);
}

}  // namespace

// Any nx, ny (non-powers of two up to 2048): rows, then columns as
// transpose + rows + transpose, then the unitary scale — in double.
void fft2d_any_f64(double2* f, int nx, int ny, int sign, int batch, cudaStream_t st) {
    const double2* tw = device_twiddles64();
    const size_t npix = (size_t)nx * ny, tot = npix * batch;
    lines64(f, nx, (size_t)ny * batch, sign, tw, st);
    if (ny > 1) {
        DevBuf64 t(tot);
        k_transpose64<<<grid_for(tot), 256, 0, st>>>(f, nx, ny, batch, t.p);
        lines64(t.p, ny, (size_t)nx * batch, sign, tw, st);
        k_transpose64<<<grid_for(tot), 256, 0, st>>>(t.p, ny, nx, batch, f);
    }
    k_scale64<<<grid_for(tot), 256, 0, st>>>(f, tot, 1.0 / std::sqrt((double)nx * ny));  // fftw_backend.cpp:121-123
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

// Unitary 2-D transform of `batch` row-major complex128 fields in place:
// rows, then columns with the (double)1/sqrt(nx*ny) scale.
void fft2d_f64(double2* f, int nx, int ny, int sign, int batch, cudaStream_t st) {
    const double2* tw = device_twiddles64();
    const size_t npix = (size_t)nx * ny;
    const double norm = 1.0 / std::sqrt((double)nx * ny);  // fftw_backend.cpp:121-123 with T = double
    if (sign < 0) {
        rows64_any<-1>(nx, f, ny, batch, npix, 0.0, tw, st);
        cols64_any<-1>(ny, f, nx, batch, npix, norm, tw, st);
    } else {
        rows64_any<+1>(nx, f, ny, batch, npix, 0.0, tw, st);
        cols64_any<+1>(ny, f, nx, batch, npix, norm, tw, st);
    }
}

}  // namespace hg
