// fft.cuh — register/shared-memory Stockham FFT for one line (row or column)
// of a complex64 field, the building block of the fused passes.
//
// Replaces the FFTW 2-D c2c transform behind FftBackend<float>
// (fft.hpp:17-27, fftw_backend.cpp:113-124).  A line of N points is owned by
// T = N/E threads; thread t holds elements t + e*T (e < E) in registers
// ("strided ownership") — the natural layout of a coalesced load/store.
// Each Stockham radix-R pass takes its butterfly inputs from the thread's
// own registers; outputs of every pass but the last are exchanged through
// shared memory; the last pass lands back in strided ownership, so the line
// is stored with the same coalesced pattern it was loaded with.
//
// Twiddles come from a per-length table tw[N + m] = exp(-2*pi*i*m/N)
// (N = 1..4096, 8192 entries), computed in double once per device and read
// through the read-only path.  The float2 arithmetic runs on packed FP32
// (common.cuh): with w and i*w at hand (one exact FMUL2 rotation) every
// twiddle product, forward or conjugated (inverse), is one FMUL2 + one FFMA2
// with only operand modifiers, bit-identical per component to the scalar
// fmaf forms.  SIGN = -1 forward, +1 inverse (unnormalised, like FFTW;
// the unitary 1/sqrt(nx*ny) scale is applied by the fused passes exactly
// where fftw_backend.cpp:121-123 applies it).
#pragma once
#include "common.cuh"

namespace hg {

constexpr int kMaxLine = 4096;
// Twiddle table layout: tw[N + m] = exp(-2 pi i m / N) for N = 1..4096, then
// at kTw256 the 16 x 16 table W_256^(r k) (r, k < 16) read directly by the
// radix-16 pass of span 256 (fft.cuh apply_twiddles).
constexpr int kTw256 = 2 * kMaxLine;
constexpr int kTwEntries = kTw256 + 256;

// Complex element type of a transform: float2 (the hot path) or double2 (the
// f64 FftBackend, k_fft64.cu).
template <class C2>
struct CT;
template <>
struct CT<float2> {
    using S = float;
    using TW = float2;
    static __device__ __forceinline__ float2 make(float x, float y) { return make_float2(x, y); }
};
template <>
struct CT<double2> {
    using S = double;
    using TW = double2;
    static __device__ __forceinline__ double2 make(double x, double y) { return make_double2(x, y); }
};

template <class C2>
__device__ __forceinline__ C2 cneg(C2 a) {
    return CT<C2>::make(-a.x, -a.y);
}

// ---------------------------------------------------------------- radix-R
template <int SIGN, class C2>
__device__ __forceinline__ C2 mul_si(C2 a) {  // a * (SIGN * i)
    return SIGN < 0 ? CT<C2>::make(a.y, -a.x) : CT<C2>::make(-a.y, a.x);
}

// Packed float2 forms (one instruction each; per component exact):
// a * (SIGN*i) = swap(a) * (-SIGN, SIGN), and t + SIGN*i*d = swap(d) * (-SIGN, SIGN) + t.
#if HG_FFT_SCALAR
template <int SIGN>
__device__ __forceinline__ float2 mul_si(float2 a) {
    return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
template <int SIGN>
__device__ __forceinline__ float2 add_si(float2 t, float2 d) {
    return cadd(t, mul_si<SIGN>(d));
}
#else
template <int SIGN>
__device__ __forceinline__ float2 mul_si(float2 a) {
    return __fmul2_rn(f2swap(a), make_float2(-(float)SIGN, (float)SIGN));
}
template <int SIGN>
__device__ __forceinline__ float2 add_si(float2 t, float2 d) {
    return __ffma2_rn(f2swap(d), make_float2(-(float)SIGN, (float)SIGN), t);
}
#endif

// W16^m = exp(SIGN*2*pi*i*m/16), applied to a (compile-time m).
template <int SIGN, int M, class C2>
__device__ __forceinline__ C2 tw16(C2 a) {
    using S = typename CT<C2>::S;
    constexpr int m = M & 15;
    constexpr S c1 = (S)0.923879532511286756128183189396788933L, s1 = (S)0.382683432365089771728459984030398866L,
                h = (S)0.707106781186547524400844362104849039L;
    if constexpr (m == 0) return a;
    else if constexpr (m == 4) return mul_si<SIGN>(a);
    else if constexpr (m == 8) return cneg(a);
    else if constexpr (m == 12) return mul_si<-SIGN>(a);
    else {
        // cos/sin of 2*pi*m/16 for the remaining m
        constexpr S cs[16] = {1, c1, h, s1, 0, -s1, -h, -c1, -1, -c1, -h, -s1, 0, s1, h, c1};
        constexpr S sn[16] = {0, s1, h, c1, 1, c1, h, s1, 0, -s1, -h, -c1, -1, -c1, -h, -s1};
        return cmul(a, CT<C2>::make(cs[m], SIGN * sn[m]));
    }
}

#ifndef HG_TW16_PACKED  // W16^2 / W16^6 = h(+-1 + SIGN i): one packed add + one packed scale
#define HG_TW16_PACKED 1
#endif
#if HG_TW16_PACKED
// float2 specialisation of tw16 for the (1 +- i)/sqrt(2) factors: a W16^2 =
// h (a + SIGN i a), a W16^6 = h (-a + SIGN i a): FADD2 / FFMA2 with operand
// modifiers + FMUL2 (2 instructions instead of the 4 of a general product).
template <int SIGN, int M>
__device__ __forceinline__ float2 tw16(float2 a) {
    constexpr int m = M & 15;
    constexpr float h = 0.707106781186547524400844362104849039f;
    if constexpr (m == 2 || m == 10) {
        const float2 t = add_si<SIGN>(a, a);
        return __fmul2_rn(t, make_float2(m == 2 ? h : -h, m == 2 ? h : -h));
    } else if constexpr (m == 6 || m == 14) {
        const float2 t = add_si<SIGN>(make_float2(-a.x, -a.y), a);
        return __fmul2_rn(t, make_float2(m == 6 ? h : -h, m == 6 ? h : -h));
    } else {
        return tw16<SIGN, M, float2>(a);
    }
}
#endif

template <int SIGN, class C2>
__device__ __forceinline__ void dft2(C2& a, C2& b) {
    C2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int SIGN, class C2>
__device__ __forceinline__ void dft4(C2& v0, C2& v1, C2& v2, C2& v3) {
    C2 t0 = cadd(v0, v2), t1 = csub(v0, v2);
    C2 t2 = cadd(v1, v3), t3 = mul_si<SIGN>(csub(v1, v3));
    v0 = cadd(t0, t2);
    v2 = csub(t0, t2);
    v1 = cadd(t1, t3);
    v3 = csub(t1, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
    const float2 t0 = cadd(v0, v2), t1 = csub(v0, v2);
    const float2 t2 = cadd(v1, v3), d = csub(v1, v3);
    v0 = cadd(t0, t2);
    v2 = csub(t0, t2);
    v1 = add_si<SIGN>(t1, d);   // t1 + (SIGN i) d
    v3 = add_si<-SIGN>(t1, d);  // t1 - (SIGN i) d
}

// In-place DFT of R values, natural order in and out:
//   x[k] <- sum_r x[r] exp(SIGN*2*pi*i*r*k/R)
template <int R, int SIGN, class C2>
__device__ __forceinline__ void dft(C2* x) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) {
        dft2<SIGN>(x[0], x[1]);
    } else if constexpr (R == 4) {
        dft4<SIGN>(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        // r = 2a + b; Y_b = DFT4_a(x[2a+b]); Y_b[k1] *= W8^(b k1); X[k1+4k2] = DFT2_b
        C2 y0[4] = {x[0], x[2], x[4], x[6]};
        C2 y1[4] = {x[1], x[3], x[5], x[7]};
        dft4<SIGN>(y0[0], y0[1], y0[2], y0[3]);
        dft4<SIGN>(y1[0], y1[1], y1[2], y1[3]);
        y1[1] = tw16<SIGN, 2>(y1[1]);
        y1[2] = tw16<SIGN, 4>(y1[2]);
        y1[3] = tw16<SIGN, 6>(y1[3]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            x[k1] = cadd(y0[k1], y1[k1]);
            x[k1 + 4] = csub(y0[k1], y1[k1]);
        }
    } else if constexpr (R == 16) {
        // r = 4a + b; Y_b = DFT4_a(x[4a+b]); Y_b[k1] *= W16^(b k1); X[k1+4k2] = DFT4_b
        C2 y[4][4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            y[b][0] = x[b];
            y[b][1] = x[4 + b];
            y[b][2] = x[8 + b];
            y[b][3] = x[12 + b];
            dft4<SIGN>(y[b][0], y[b][1], y[b][2], y[b][3]);
        }
        y[1][1] = tw16<SIGN, 1>(y[1][1]);
        y[1][2] = tw16<SIGN, 2>(y[1][2]);
        y[1][3] = tw16<SIGN, 3>(y[1][3]);
        y[2][1] = tw16<SIGN, 2>(y[2][1]);
        y[2][2] = tw16<SIGN, 4>(y[2][2]);
        y[2][3] = tw16<SIGN, 6>(y[2][3]);
        y[3][1] = tw16<SIGN, 3>(y[3][1]);
        y[3][2] = tw16<SIGN, 6>(y[3][2]);
        y[3][3] = tw16<SIGN, 9>(y[3][3]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            dft4<SIGN>(y[0][k1], y[1][k1], y[2][k1], y[3][k1]);
            x[k1] = y[0][k1];
            x[k1 + 4] = y[1][k1];
            x[k1 + 8] = y[2][k1];
            x[k1 + 12] = y[3][k1];
        }
    }
}

// Elements per thread for a line of N points (at most EM: 16, or 8 for the
// 32-register column variant).
template <int N, int EM = 16>
struct LineCfg {
    static constexpr int E = N < EM ? N : EM;
    static constexpr int T = N / E;
};

// Twiddle exp(SIGN*2*pi*i*m/N) from the forward table.
template <int N, int SIGN, class TW>
__device__ __forceinline__ TW twiddle(const TW* __restrict__ tw, int m) {
    TW w = __ldg(&tw[N + m]);
    if constexpr (SIGN > 0) w.y = -w.y;
    return w;
}

// x[r] *= w^r, w = exp(SIGN*2*pi*i*k/S), r = 1..R-1, k < S/R (S = the pass's
// span NS*R).  Every power a pass needs is read from the table of a shorter
// length at the same index k: w^4 = W_{S/4}^k, w^8 = W_{S/8}^k (exact: the
// table entries of W_S^{4k} and W_{S/4}^k are the same sincospi argument).  A
// warp's 16 consecutive k then touch one 128-B line per load instead of up to
// 16 (stride 4k / 8k in the length-S table).  For R = 16 only w, w^4 and w^8
// are loaded (the rest are <= 2 products of table values, error <= ~2 ulp):
// 3 loads instead of 15 keeps the pass within the register budget of a
// 1024-thread CTA (loading all 15 measured 10.1 vs 6.9 ms for the 4096^2 row
// pass: the extra live values spill).
template <int S, int SIGN, int R, class C2, class TW>
__device__ __forceinline__ void apply_twiddles(C2* x, const TW* __restrict__ tw, int k) {
    if constexpr (R == 16) {
        const TW w1 = twiddle<S, SIGN>(tw, k);
        const TW w4 = twiddle<S / 4, SIGN>(tw, k);
        const TW w8 = twiddle<S / 8, SIGN>(tw, k);
        const TW w2 = cmul(w1, w1), w3 = cmul(w2, w1), w12 = cmul(w8, w4);
        x[1] = cmul(x[1], w1);
        x[2] = cmul(x[2], w2);
        x[3] = cmul(x[3], w3);
        x[4] = cmul(x[4], w4);
        x[8] = cmul(x[8], w8);
        x[12] = cmul(x[12], w12);
        x[5] = cmul(x[5], cmul(w4, w1));
        x[6] = cmul(x[6], cmul(w4, w2));
        x[7] = cmul(x[7], cmul(w4, w3));
        x[9] = cmul(x[9], cmul(w8, w1));
        x[10] = cmul(x[10], cmul(w8, w2));
        x[11] = cmul(x[11], cmul(w8, w3));
        x[13] = cmul(x[13], cmul(w12, w1));
        x[14] = cmul(x[14], cmul(w12, w2));
        x[15] = cmul(x[15], cmul(w12, w3));
    } else if constexpr (R == 8) {
        const TW w1 = twiddle<S, SIGN>(tw, k);
        const TW w2 = twiddle<S / 2, SIGN>(tw, k);
        const TW w4 = twiddle<S / 4, SIGN>(tw, k);
        x[1] = cmul(x[1], w1);
        x[2] = cmul(x[2], w2);
        x[3] = cmul(x[3], cmul(w1, w2));
        x[4] = cmul(x[4], w4);
        x[5] = cmul(x[5], cmul(w4, w1));
        x[6] = cmul(x[6], cmul(w4, w2));
        x[7] = cmul(x[7], cmul(w4, cmul(w1, w2)));
    } else {
#pragma unroll
        for (int r = 1; r < R; ++r) x[r] = cmul(x[r], twiddle<S, SIGN>(tw, r * k));
    }
}

#ifndef HG_TW256
#define HG_TW256 0  // measured: 11.16-11.20 vs 11.09-11.14 ms per iteration (loads cost more than the products they save)
#endif
// float2 lines: twiddles as (w, i*w) pairs in the forward direction; the
// inverse applies conj(w) through lane swaps: a * conj(w) = (a.x, a.x) * swap(i*w)
// + (a.y, a.y) * swap(w).
struct Tw2 {
    float2 w, r;
};
__device__ __forceinline__ float2 f2rot(float2 w) {  // i*w = (-w.y, w.x), exact
#if HG_FFT_SCALAR
    return make_float2(-w.y, w.x);
#else
    return __fmul2_rn(f2swap(w), make_float2(-1.f, 1.f));
#endif
}
template <int N>
__device__ __forceinline__ Tw2 tw_load(const float2* __restrict__ tw, int m) {
    const float2 w = __ldg(&tw[N + m]);
    return Tw2{w, f2rot(w)};
}
__device__ __forceinline__ Tw2 tw_mul(Tw2 a, Tw2 b) {
    const float2 p = cmul_r(a.w, b.w, b.r);
    return Tw2{p, f2rot(p)};
}
template <int SIGN>
__device__ __forceinline__ float2 tw_apply(float2 a, Tw2 w) {
    if constexpr (SIGN < 0) return cmul_r(a, w.w, w.r);
    else return cmul_r(a, f2swap(w.r), f2swap(w.w));  // conj(w) and i*conj(w)
}
template <int S, int SIGN, int R>
__device__ __forceinline__ void apply_twiddles(float2* x, const float2* __restrict__ tw, int k) {
    if constexpr (R == 16 && S == 256 && HG_TW256) {
        // span 256 (k < 16): all 15 powers from the 16 x 16 table, one 128-B line
        // per warp load, instead of 3 loads + 12 products (fewer FP32 ops, and
        // each twiddle is the rounded exact value instead of a product of them)
#pragma unroll
        for (int r = 1; r < 16; ++r) x[r] = tw_apply<SIGN>(x[r], tw_load<kTw256>(tw, r * 16 + k));
    } else if constexpr (R == 16) {
        const Tw2 w1 = tw_load<S>(tw, k), w4 = tw_load<S / 4>(tw, k), w8 = tw_load<S / 8>(tw, k);
        const Tw2 w2 = tw_mul(w1, w1), w3 = tw_mul(w2, w1), w12 = tw_mul(w8, w4);
        x[1] = tw_apply<SIGN>(x[1], w1);
        x[2] = tw_apply<SIGN>(x[2], w2);
        x[3] = tw_apply<SIGN>(x[3], w3);
        x[4] = tw_apply<SIGN>(x[4], w4);
        x[8] = tw_apply<SIGN>(x[8], w8);
        x[12] = tw_apply<SIGN>(x[12], w12);
        x[5] = tw_apply<SIGN>(x[5], tw_mul(w4, w1));
        x[6] = tw_apply<SIGN>(x[6], tw_mul(w4, w2));
        x[7] = tw_apply<SIGN>(x[7], tw_mul(w4, w3));
        x[9] = tw_apply<SIGN>(x[9], tw_mul(w8, w1));
        x[10] = tw_apply<SIGN>(x[10], tw_mul(w8, w2));
        x[11] = tw_apply<SIGN>(x[11], tw_mul(w8, w3));
        x[13] = tw_apply<SIGN>(x[13], tw_mul(w12, w1));
        x[14] = tw_apply<SIGN>(x[14], tw_mul(w12, w2));
        x[15] = tw_apply<SIGN>(x[15], tw_mul(w12, w3));
    } else if constexpr (R == 8) {
        const Tw2 w1 = tw_load<S>(tw, k), w2 = tw_load<S / 2>(tw, k), w4 = tw_load<S / 4>(tw, k);
        const Tw2 w3 = tw_mul(w1, w2);
        x[1] = tw_apply<SIGN>(x[1], w1);
        x[2] = tw_apply<SIGN>(x[2], w2);
        x[3] = tw_apply<SIGN>(x[3], w3);
        x[4] = tw_apply<SIGN>(x[4], w4);
        x[5] = tw_apply<SIGN>(x[5], tw_mul(w4, w1));
        x[6] = tw_apply<SIGN>(x[6], tw_mul(w4, w2));
        x[7] = tw_apply<SIGN>(x[7], tw_mul(w4, w3));
    } else {
#pragma unroll
        for (int r = 1; r < R; ++r) x[r] = tw_apply<SIGN>(x[r], tw_load<S>(tw, r * k));
    }
}

// Barrier between the scatter and the gather of an exchange (the whole CTA).
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// Barrier of one thread group of a CTA (named barrier `id`, `n` threads).
struct GroupSync {
    int id, n;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};

// Exchange-buffer slot access (one element per slot).
template <class C2, class I>
__device__ __forceinline__ void smst(C2* sm, const I&, int s, C2 v) {
    sm[s] = v;
}
template <class C2, class I>
__device__ __forceinline__ C2 smld(const C2* sm, const I&, int s) {
    return sm[s];
}
// One Stockham pass (span NS) and, recursively, the rest.
//   butterfly j = t + b*T (b < E/R) reads elements b + r*(E/R);
//   twiddle by W_{NS*R}^{r*(j mod NS)}; DFT_R;
//   output r goes to position (j/NS)*NS*R + (j mod NS) + r*NS.
// SmemIdx maps a line position to a shared-memory slot for this thread's line.
template <int N, int SIGN, int NS, int EM = 16>
struct StockhamPass {
    template <class C2, class SmemIdx, class Sync>
    __device__ __forceinline__ static void run(C2 (&v)[LineCfg<N, EM>::E], int t, C2* sm, const SmemIdx& idx,
                                               const typename CT<C2>::TW* __restrict__ tw, const Sync& sync) {
        constexpr int E = LineCfg<N, EM>::E, T = LineCfg<N, EM>::T;
        constexpr int R = (N / NS >= E) ? E : N / NS;
        constexpr int B = E / R;
        constexpr bool last = (NS * R == N);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            C2 x[R];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = v[b + r * B];
            const int j = t + b * T;
            const int k = j & (NS - 1);
            if constexpr (NS > 1) apply_twiddles<NS * R, SIGN, R>(x, tw, k);
            dft<R, SIGN>(x);
            if constexpr (last) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[b + r * B] = x[r];
            } else {
                // positions base + r*NS; with NS == 1 (R <= 16) or NS % 16 == 0
                // the padded slots are linear in r: slot(base) + r*stride
                const int base = (j / NS) * NS * R + k;
                if constexpr (NS == 1 || NS % 16 == 0) {
                    const int s0 = idx(base);
                    constexpr int rs = (NS == 1) ? 1 : NS + NS / 16;
#pragma unroll
                    for (int r = 0; r < R; ++r) smst(sm, idx, s0 + r * rs * SmemIdx::kLineStride, x[r]);
                } else {
#pragma unroll
                    for (int r = 0; r < R; ++r) smst(sm, idx, idx(base + r * NS), x[r]);
                }
            }
        }
        if constexpr (!last) {
            sync();
            if constexpr (T % 16 == 0) {
                const int s0 = idx(t);
                constexpr int es = T + T / 16;
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = smld(sm, idx, s0 + e * es * SmemIdx::kLineStride);
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = smld(sm, idx, idx(t + e * T));
            }
            sync();
            StockhamPass<N, SIGN, NS * R, EM>::run(v, t, sm, idx, tw, sync);
        }
    }
};

// Full unnormalised 1-D transform of one line held in strided ownership.
// Every thread of the CTA (or of the Sync group) must call it (it contains
// barriers when N > E).
template <int N, int SIGN, int EM = 16, class C2, class SmemIdx, class Sync = CtaSync>
__device__ __forceinline__ void fft_line(C2 (&v)[LineCfg<N, EM>::E], int t, C2* sm, const SmemIdx& idx,
                                         const typename CT<C2>::TW* __restrict__ tw, const Sync& sync = Sync{}) {
    StockhamPass<N, SIGN, 1, EM>::run(v, t, sm, idx, tw, sync);
}

// Padded slot for position q of a line: one pad slot every 16 keeps the
// radix-16 scatter (stride 16) free of bank conflicts.
__device__ __forceinline__ int pad16(int q) { return q + (q >> 4); }
template <int N>
struct PaddedLen {
    static constexpr int value = N + (N >> 4) + 1;
};

// Row layout: each line owns a contiguous padded region.
struct RowSmemIdx {
    static constexpr int kLineStride = 1;  // slot step per position step
    int off;
    __device__ __forceinline__ int operator()(int q) const { return off + pad16(q); }
};
// Column layout: C lines interleaved (slot * C + c) so a warp spanning
// C adjacent columns hits adjacent banks.
template <int C>
struct ColSmemIdx {
    static constexpr int kLineStride = C;
    int c;
    __device__ __forceinline__ int operator()(int q) const { return pad16(q) * C + c; }
};

}  // namespace hg
