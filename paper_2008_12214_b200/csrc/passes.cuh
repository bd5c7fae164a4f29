// passes.cuh — the two fused HBM round trips of an IFTA iteration and the
// OSPR subframe passes.
//
// Layout in HBM: every field is complex64 row-major [target][ny][nx]
// (ComplexField<float>, field.hpp:27-46).  The 2-D inverse transform is done
// columns-first, the forward one rows-first, so one iteration of
// run_ifta (ifta.hpp:166-226) is exactly two passes:
//
//   ROW pass (aperture plane):  IFFT rows (completes P^-1)  -> *norm
//        -> *conj(Q) (Fresnel)  -> quantise (+levels)  -> *Q (Fresnel)
//        -> FFT rows (starts P)                                    [R+W field]
//   COL pass (replay plane):    FFT cols (completes P) -> *norm -> MSE partials
//        -> constraint (+WGS weights) -> IFFT cols (starts next P^-1) [R+W field,
//                                                            R target]
//   The last iteration's column pass stores the replay instead.
//
// OSPR (ospr.hpp:105-147) uses: seed kernel -> COL inverse -> ROW fused
// (levels out) -> COL forward with intensity accumulation + both MSE traces.
#pragma once
#include "fft.cuh"
#include "quant.cuh"

namespace hg {

// --------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV doubles; thread 0 writes them to out[0..NV).  Fixed order.
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* out) {
    __shared__ double red[32][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) red[warp][i] = v[i];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = lane < nw ? red[lane][i] : 0.0;
            x = warp_sum(x);
            if (lane == 0) out[i] = x;
        }
    }
}

// ---------------------------------------------------------------- row pass
enum RowMode { ROW_FUSED = 0, ROW_PLAIN = 1 };

struct RowArgs {
    const float2* tw;  // twiddle table (fft.cuh)
    float2* field;
    size_t bstride;   // elements per target
    int ny;
    float norm;       // (float)(1/sqrt(nx*ny)) applied after the row IFFT (fused) / the row FFT (plain, if apply_norm)
    int sign;         // ROW_PLAIN: -1 forward, +1 inverse
    int apply_norm;   // ROW_PLAIN
    const float2* fresnel_q;  // [ny][nx] or nullptr
    QuantParams q;
    uint8_t* levels8;         // [target][ny][nx] or nullptr
    uint16_t* levels16;
    size_t lv_bstride;
};

template <int NX>
struct RowCfg {
    static constexpr int E = LineCfg<NX>::E, T = LineCfg<NX>::T;
    static constexpr int RPC = T >= 256 ? 1 : 256 / T;  // rows per CTA
    static constexpr int THREADS = T * RPC;
    static constexpr int SMEM = (NX > E) ? RPC * PaddedLen<NX>::value * (int)sizeof(float2) : 0;
    static constexpr int MIN_BLOCKS = THREADS >= 256 ? 3 : 1;  // <= 85 registers: 24 warps / SM
};

template <int NX, int MODE, int QK>
__global__ void __launch_bounds__(RowCfg<NX>::THREADS, RowCfg<NX>::MIN_BLOCKS) k_row(RowArgs a) {
    using Cfg = RowCfg<NX>;
    constexpr int E = Cfg::E, T = Cfg::T;
    extern __shared__ float2 smem[];
    const int lr = threadIdx.x / T, t = threadIdx.x % T;
    const int y = blockIdx.x * Cfg::RPC + lr;
    const int b = blockIdx.y;
    RowSmemIdx idx{lr * PaddedLen<NX>::value};
    const bool valid = y < a.ny;  // (ny is a multiple of RPC except for tiny fields)
    float2* row = a.field + a.bstride * b + (size_t)(valid ? y : 0) * NX;
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = row[t + e * T];

    if constexpr (MODE == ROW_PLAIN) {
        // Propagator<float>::forward / inverse halves (propagation.hpp:81-95):
        // forward rows start from f*Q; inverse rows finish with *norm *conj(Q).
        const size_t rowbase = (size_t)y * NX;
        if (a.sign < 0) {
            if (a.fresnel_q)
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmul_rn(v[e], __ldg(&a.fresnel_q[rowbase + t + e * T]));
            fft_line<NX, -1>(v, t, smem, idx, a.tw);
        } else {
            fft_line<NX, +1>(v, t, smem, idx, a.tw);
        }
        if (a.apply_norm)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], a.norm);
        if (a.sign > 0 && a.fresnel_q)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cmul_conj_rn(v[e], __ldg(&a.fresnel_q[rowbase + t + e * T]));
    } else {
        fft_line<NX, +1>(v, t, smem, idx, a.tw);  // completes the 2-D inverse (propagation.hpp:89-95)
        const int rowbase = y * NX;
        const float norm = a.norm;
        const float2* __restrict__ fq = a.fresnel_q;
        uint8_t* __restrict__ lv8 = a.levels8 ? a.levels8 + a.lv_bstride * b : nullptr;
        uint16_t* __restrict__ lv16 = a.levels16 ? a.levels16 + a.lv_bstride * b : nullptr;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = rowbase + t + e * T;
            float2 f = cscale(v[e], norm);                        // fftw_backend.cpp:121-123
            if (fq) f = cmul_conj_rn(f, __ldg(&fq[i]));           // propagation.hpp:93
            const int k = quant_decide_kind<QK>(a.q, f.x, f.y, i);  // quantise.hpp:211-215
            if constexpr (QK == QK_BINARY) f = k ? a.q.s1 : a.q.s0;
            else f = quant_state(a.q, k, i);
            if (lv8 && valid) lv8[i] = (uint8_t)k;
            if (lv16 && valid) lv16[i] = (uint16_t)k;
            if (fq) f = cmul_rn(f, __ldg(&fq[i]));                // propagation.hpp:85
            v[e] = f;
        }
        fft_line<NX, -1>(v, t, smem, idx, a.tw);  // starts the forward transform
    }
    if (valid)
#pragma unroll
        for (int e = 0; e < E; ++e) row[t + e * T] = v[e];
}

// ------------------------------------------------------------- column pass
enum ColMode { COL_PLAIN = 0, COL_GS = 1, COL_OSPR = 2 };

struct ColArgs {
    const float2* tw;
    float2* field;
    size_t bstride;
    int nx;
    float norm;
    int sign;        // COL_PLAIN
    int apply_norm;  // COL_PLAIN
    // replay-plane constraint (ifta.hpp:185-224)
    const float* target;  // fp32 amplitude [target][ny][nx]
    size_t t_bstride;
    const uint8_t* roi;   // [ny][nx] (shared) or nullptr
    float* weights;       // WGS [target][ny][nx] or nullptr
    const float2* tphase_cs;  // phase-freedom-off: (cos, sin) of target phase [target][ny][nx]
    int phase_freedom, amp_outside_roi, scale_free;
    float clamp_lo, clamp_hi;
    int lt, lt_x0, lt_x1, lt_y0, lt_y1;
    int last;             // last iteration: store R, skip constraint + IFFT
    float2* replay_out;   // where the last iteration's R goes (may alias field)
    double* partials;     // per block: 8 doubles
    // OSPR accumulation
    float* S;             // [job][ny][nx] running sum of |R|^2
    size_t S_bstride;
    float inv_n;          // 1/n for the cumulative replay sqrt(S/n)
};

template <int NY>
struct ColCfg {
    static constexpr int E = LineCfg<NY>::E, T = LineCfg<NY>::T;
    static constexpr int CMAX = (16384 / NY) < 16 ? (16384 / NY) : 16;  // 128 KiB of complex64 per CTA
    static constexpr int C = CMAX < 1 ? 1 : CMAX;
    static constexpr int THREADS = T * C;
    static constexpr int SMEM = (NY > E) ? PaddedLen<NY>::value * C * (int)sizeof(float2) : 0;
};

template <int NY, int C, int MODE>
__global__ void __launch_bounds__(LineCfg<NY>::T * C) k_col(ColArgs a) {
    constexpr int E = LineCfg<NY>::E, T = LineCfg<NY>::T;
    extern __shared__ float2 smem[];
    const int c = threadIdx.x % C, t = threadIdx.x / C;
    const int x = blockIdx.x * C + c;
    const int b = blockIdx.y;
    const int nx = a.nx;
    ColSmemIdx<C> idx{c};
    float2* base = a.field + a.bstride * b + x;
    float2 v[E];
    {
        const float2* p0 = base + t * nx;
        const int st = T * nx;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = p0[e * st];
    }
    // stores recompute their addresses from an opaque base (keeps 16 64-bit
    // pointers from living across the transforms)
    auto store_col = [&](float2* dst) {
        float2* p1 = opaque(dst) + t * nx;
        const int st = opaque(T * nx);
#pragma unroll
        for (int e = 0; e < E; ++e) p1[e * st] = v[e];
    };

    if constexpr (MODE == COL_PLAIN) {
        if (a.sign < 0) fft_line<NY, -1>(v, t, smem, idx, a.tw);
        else fft_line<NY, +1>(v, t, smem, idx, a.tw);
        if (a.apply_norm)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], a.norm);
        store_col(base);
        return;
    } else {
        fft_line<NY, -1>(v, t, smem, idx, a.tw);  // completes the forward transform
        const float* tg = a.target + a.t_bstride * b + x;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if constexpr (MODE == COL_GS) {
            float* w = a.weights ? a.weights + a.t_bstride * b + x : nullptr;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int y = t + e * T;
                const int off = y * nx;
                float2 R = cscale(v[e], a.norm);
                const bool in_roi = !a.roi || a.roi[off + x];
                float amp = __ldg(&tg[off]);
                float r = sqrtf(R.x * R.x + R.y * R.y);
                if (in_roi) {  // mse partials (metrics.hpp:70-97)
                    float d = amp - r;
                    acc[0] += d * d;
                    acc[1] += amp * r;
                    acc[2] += r * r;
                    acc[3] += amp * amp;
                }
                if (!a.last) {  // replay-plane constraint, ifta.hpp:190-223
                    if (in_roi) {
                        const bool active = !a.lt || (x >= a.lt_x0 && x < a.lt_x1 && y >= a.lt_y0 && y < a.lt_y1);
                        if (active) {
                            if (w && amp > 0.f) {
                                float cand = w[off] * amp / fmaxf(r, 1e-12f);
                                float wn = fminf(fmaxf(cand, a.clamp_lo), a.clamp_hi);
                                w[off] = wn;
                                amp *= wn;
                            }
                            if (a.phase_freedom) {
                                if (r > 0.f) {
                                    float s = amp / r;
                                    R = make_float2(R.x * s, R.y * s);
                                } else {
                                    R = make_float2(amp, 0.f);
                                }
                            } else {
                                float2 cs = a.tphase_cs[a.t_bstride * b + off + x];
                                R = make_float2(amp * cs.x, amp * cs.y);
                            }
                        }
                    } else if (!a.amp_outside_roi) {
                        R = make_float2(0.f, 0.f);
                    }
                }
                v[e] = R;
            }
            if (a.last) {
                store_col(a.replay_out + a.bstride * b + x);
            } else {
                fft_line<NY, +1>(v, t, smem, idx, a.tw);  // starts the next inverse transform
                store_col(base);
            }
        } else {  // COL_OSPR: ospr.hpp:134-145
            float* S = a.S + a.S_bstride * b + x;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int y = t + e * T;
                const int off = y * nx;
                float2 R = cscale(v[e], a.norm);
                float I = R.x * R.x + R.y * R.y;
                float s = S[off] + I;
                S[off] = s;
                if (!a.roi || a.roi[off + x]) {
                    float amp = __ldg(&tg[off]);
                    float r = sqrtf(I);
                    float d = amp - r;
                    acc[0] += d * d;
                    acc[1] += amp * r;
                    acc[2] += I;
                    acc[3] += amp * amp;
                    float rc = sqrtf(s * a.inv_n);
                    float dc = amp - rc;
                    acc[4] += dc * dc;
                    acc[5] += amp * rc;
                    acc[6] += rc * rc;
                }
            }
        }
        // per-thread float partials (<= 16 terms) -> fixed-order double block sums
        const size_t blk = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        constexpr int NV = MODE == COL_GS ? 4 : 7;
        double dacc[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) dacc[i] = (double)acc[i];
        block_sum_store<NV>(dacc, a.partials + blk * 8);
    }
}

}  // namespace hg
