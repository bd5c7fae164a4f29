// common.cuh — shared device helpers for the HoloGen B200 hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HG_TWO_PI 6.283185307179586476925286766559
#ifndef HG_STREAM_LOADS
#define HG_STREAM_LOADS 1
#endif
#define HG_PI 3.1415926535897932384626433832795

// Complex products with every product/sum rounded separately (no FMA
// contraction), i.e. the way GCC evaluates std::complex<float> operator* on
// baseline x86-64: (a+bi)(c+di) = (ac - bd) + (ad + bc)i.  Used wherever the
// reference multiplies complex<T> values (quantise.hpp:201-205,
// propagation.hpp:85, :93) so results match bit for bit.
__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
    float ac = __fmul_rn(a.x, b.x), bd = __fmul_rn(a.y, b.y);
    float ad = __fmul_rn(a.x, b.y), bc = __fmul_rn(a.y, b.x);
    return make_float2(__fsub_rn(ac, bd), __fadd_rn(ad, bc));
}

// a * conj(b), evaluated as GCC does for z *= std::conj(q):
// (a+bi)(c-di): real = ac - b(-d) = ac + bd, imag = a(-d) + bc.
__device__ __forceinline__ float2 cmul_conj_rn(float2 a, float2 b) {
    float ac = __fmul_rn(a.x, b.x), bd = __fmul_rn(a.y, b.y);
    float ad = __fmul_rn(a.x, b.y), bc = __fmul_rn(a.y, b.x);
    return make_float2(__fadd_rn(ac, bd), __fsub_rn(bc, ad));
}

// Complex arithmetic of the transforms.  sm_100a executes the f32x2
// operations as FADD2 / FMUL2 / FFMA2, one instruction for both components,
// with lane broadcast, lane swap and negation as free operand modifiers and
// constant pairs in uniform registers.  Per component the roundings are
// exactly those of the scalar forms, so every choice below gives bit-identical
// fields:
//   cadd / csub: a.x +- b.x, a.y +- b.y;
//   cmul: fmaf(a.x, b.x, -(a.y*b.y)), fmaf(a.x, b.y, a.y*b.x), i.e.
//         (a.x, a.x) * b + (a.y, a.y) * (-b.y, b.x)  (negation is exact).
// HG_FFT_SCALAR: 0 everything packed, 1 everything scalar, 2 (default) packed
// adds with scalar products.  Packed instructions issue at half rate (2 warp
// instructions/clk/SM = 128 lane-ops, like scalar FADD/FFMA at 4; microbench
// tools/microbench/f32x2_tput.cu), so they save issue slots, not FP-pipe time.
// Measured at 4096^2 x 64 in the launch sequence: 11.66 ms per iteration
// (hybrid) vs 11.77 (packed) vs 12.45 (scalar).
__device__ __forceinline__ float2 f2swap(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 f2bx(float2 a) { return make_float2(a.x, a.x); }
__device__ __forceinline__ float2 f2by(float2 a) { return make_float2(a.y, a.y); }
#ifndef HG_FFT_SCALAR
#define HG_FFT_SCALAR 2
#endif
#if HG_FFT_SCALAR
#if HG_FFT_SCALAR == 2  // packed adds, scalar products
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
#endif
__device__ __forceinline__ float2 cmul_r(float2 a, float2 w, float2 wr) {
    return make_float2(fmaf(a.x, w.x, a.y * wr.x), fmaf(a.x, w.y, a.y * wr.y));
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a * w given w and its rotation wr = i*w = (-w.y, w.x)
__device__ __forceinline__ float2 cmul_r(float2 a, float2 w, float2 wr) {
    return __ffma2_rn(f2bx(a), w, __fmul2_rn(f2by(a), wr));
}
#endif
__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return cmul_r(a, b, make_float2(-b.y, b.x)); }
// double2 versions for the f64 transform (k_fft64.cu)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) {
#if HG_FFT_SCALAR
    return make_float2(__fmul_rn(a.x, s), __fmul_rn(a.y, s));
#else
    return __fmul2_rn(a, make_float2(s, s));
#endif
}

// Opaque copies: the compiler must recompute anything derived from the
// result instead of keeping it live in registers (used to stop 16 64-bit
// load addresses from staying live across an FFT until the stores).
__device__ __forceinline__ int opaque(int x) {
    int y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
template <class T>
__device__ __forceinline__ T* opaque(T* p) {
    unsigned long long y;
    asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"((unsigned long long)p));
    return (T*)y;
}

// ------------------------------------------------------------------ layouts
// LAY_ROW : row-major [y][x] (ComplexField order) — primitives, host I/O.
// LAY_QUAD: the plans' resident layout.  32-byte quads of 2 rows x 2 columns,
//   quad (y/2, x/2) at ((y/2)*(nx/2) + x/2)*4, inside it (y&1)*2 + (x&1).
//   A row pair is one contiguous block (row pass: 2 rows per CTA) and a
//   column pair reads whole 32 B sectors (column pass: 2 columns per CTA),
//   so both passes move full sectors with 64 KiB tiles (2 CTAs / SM).
// Per-pixel side arrays of the column pass (target, weights, OSPR sum, ROI)
// are column-pair major in LAY_QUAD: ((x/2)*ny + y)*2 + (x&1).
namespace hg {
enum Layout { LAY_ROW = 0, LAY_QUAD = 1 };

__host__ __device__ __forceinline__ size_t quad_index(int x, int y, int nx) {
    return (((size_t)(y >> 1) * (nx >> 1) + (x >> 1)) << 2) + ((y & 1) << 1) + (x & 1);
}
__host__ __device__ __forceinline__ size_t colpair_index(int x, int y, int ny) {
    return (((size_t)(x >> 1) * ny + y) << 1) + (x & 1);
}
}  // namespace hg

// Streaming loads that do not allocate in L1 (keeps the L1-resident twiddle
// table hot while tiles stream through).
__device__ __forceinline__ float2 ld_stream(const float2* p) {
#if HG_STREAM_LOADS
    float2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
#else
    return *p;
#endif
}
__device__ __forceinline__ float ld_stream(const float* p) {
#if HG_STREAM_LOADS
    float v;
    asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

// ------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One thread: expect `bytes` on the barrier and start a global->shared bulk copy
// (cp.async.bulk, the 1-D TMA path).  16 B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
}

__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 2-D tensor TMA (cp.async.bulk.tensor) through a tensor map in global memory.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* map, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
// One thread: shared -> global bulk copy (1-D), completed with bulk_commit /
// bulk_wait_read0.  16 B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int V>
struct IntC {
    static constexpr int value = V;
};

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
