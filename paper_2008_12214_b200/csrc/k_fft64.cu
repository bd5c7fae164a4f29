// k_fft64.cu — the double-precision 2-D transform behind FftBackend<double>
// (fft.hpp:17-27; FftwBackend's double plans, fftw_backend.cpp:43-46, scaled
// by 1/sqrt(nx*ny) in double, :121-123) — SURVEY §8 f4.
//
// The same register/shared-memory Stockham core as the f32 hot path
// (fft.cuh, instantiated on double2) with 8 elements per thread, so a 4096
// line keeps 32 registers of data.  Row-major layout (ComplexField<double>),
// rows pass then columns pass, the unitary scale applied by the last pass.
#include <cmath>
#include <map>
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

}  // namespace

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
