// f64path.cuh — kernels of the double-precision loops:
// run_ifta<double> (ifta.hpp:86-235) and run_ospr_impl<double>
// (ospr.hpp:68-164) on the device.  Row-major complex128 fields; the
// transforms are the f64 ones of k_fft64.cu (any size).  Every elementwise
// step replays the reference's double arithmetic without FMA contraction
// (__dmul_rn / __dadd_rn / __dsqrt_rn), so per pixel it is bit-identical to
// the reference given the same inputs; reductions run in a fixed block order.
#pragma once
#include "common.cuh"

namespace hg {

// Quantiser<double> (quantise.hpp:136-231): states and illumination in double.
struct Q64 {
    int mode, L, full_circle;
    double min_arg, inv_spac, range, min_amp;
    const double2* states;
    const double* illum_arg;    // phase mode with illumination
    const double2* illum;       // phase mode
    const double2* illum_unit;  // amplitude mode
};

// std::complex<double> products as GCC evaluates them (no FMA)
__device__ __forceinline__ double2 cmul_rn64(double2 a, double2 b) {
    const double ac = __dmul_rn(a.x, b.x), bd = __dmul_rn(a.y, b.y), ad = __dmul_rn(a.x, b.y), bc = __dmul_rn(a.y, b.x);
    return make_double2(__dsub_rn(ac, bd), __dadd_rn(ad, bc));
}
__device__ __forceinline__ double2 cmul_conj_rn64(double2 a, double2 q) {  // a * conj(q)
    const double ac = __dmul_rn(a.x, q.x), bd = __dmul_rn(a.y, q.y), ad = __dmul_rn(a.x, q.y), bc = __dmul_rn(a.y, q.x);
    return make_double2(__dadd_rn(ac, bd), __dsub_rn(bc, ad));
}
__device__ __forceinline__ double abs_rn64(double2 z) {  // std::sqrt(re * re + im * im)
    return __dsqrt_rn(__dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y)));
}

// Quantiser::decide in double (quantise.hpp:175-198)
__device__ __forceinline__ int decide64(const Q64& q, size_t i, double2 v) {
    if (q.mode == 1) {
        double ang = atan2(v.y, v.x);
        if (q.illum_arg) ang = __dsub_rn(ang, q.illum_arg[i]);
        double d = __dsub_rn(ang, q.min_arg);
        d = __dsub_rn(d, __dmul_rn(HG_TWO_PI, floor(__ddiv_rn(d, HG_TWO_PI))));
        if (q.full_circle) {
            const int k = (int)llround(__dmul_rn(d, q.inv_spac));
            return k >= q.L ? 0 : k;
        }
        if (d <= q.range) {
            const int k = (int)llround(__dmul_rn(d, q.inv_spac));
            return k > q.L - 1 ? q.L - 1 : k;
        }
        return (__dsub_rn(d, q.range) <= __dsub_rn(HG_TWO_PI, d)) ? q.L - 1 : 0;
    }
    long long k = llround(__dmul_rn(__dsub_rn(abs_rn64(v), q.min_amp), q.inv_spac));
    if (k < 0) k = 0;
    if (k > q.L - 1) k = q.L - 1;
    return (int)k;
}

// Quantiser::apply (quantise.hpp:208-216) + level indices
static __global__ void k_quant64(double2* f, int32_t* levels, size_t n, Q64 q) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = decide64(q, i, f[i]);
        double2 s = q.states[k];
        if (q.mode == 1 && q.illum) s = cmul_rn64(q.illum[i], s);
        if (q.mode == 0 && q.illum_unit) s = cmul_rn64(q.illum_unit[i], s);
        f[i] = s;
        if (levels) levels[i] = k;
    }
}

// Propagator<double>: forward input f*Q (propagation.hpp:85), inverse output *conj(Q) (:93)
static __global__ void k_mulq64(double2* f, const double2* Q, size_t n, int conj_q) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        f[i] = conj_q ? cmul_conj_rn64(f[i], Q[i]) : cmul_rn64(f[i], Q[i]);
}

__device__ __forceinline__ double block_sum64(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;  // thread 0
}

// mse (metrics.hpp:70-97), phase-insensitive, in two passes so the
// scale-free gain g = max(0, sum T|R| / sum |R|^2) is applied exactly as the
// reference does.  The replay magnitude comes from a field (mode 0) or, for
// OSPR's cumulative replay, from sqrt(S / n) (mode 1, ospr.hpp:140-145).
struct Mag64 {
    const double2* R;
    const double* S;
    double n;
    __device__ __forceinline__ double operator()(size_t i) const {
        return R ? abs_rn64(R[i]) : __dsqrt_rn(__ddiv_rn(S[i], n));
    }
};
static __global__ void k_mse64_gain(const double* T, Mag64 mag, const uint8_t* mask, size_t n, double* part) {
    __shared__ double red[32];
    double s_tr = 0.0, s_rr = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (mask && !mask[i]) continue;
        const double r = mag(i);
        s_tr = __dadd_rn(s_tr, __dmul_rn(T[i], r));
        s_rr = __dadd_rn(s_rr, __dmul_rn(r, r));
    }
    s_tr = block_sum64(s_tr, red);
    s_rr = block_sum64(s_rr, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = s_tr;
        part[2 * blockIdx.x + 1] = s_rr;
    }
}
static __global__ void k_mse64_g(const double* part, int nblk, int scale_free, double* g) {
    if (threadIdx.x != 0) return;
    double s_tr = 0.0, s_rr = 0.0;
    for (int b = 0; b < nblk; ++b) {
        s_tr += part[2 * b];
        s_rr += part[2 * b + 1];
    }
    double v = 1.0;
    if (scale_free) {
        v = s_rr > 0.0 ? s_tr / s_rr : 0.0;
        if (v < 0.0) v = 0.0;
    }
    *g = v;
}
static __global__ void k_mse64_sum(const double* T, Mag64 mag, const uint8_t* mask, size_t n, const double* g, double* part) {
    __shared__ double red[32];
    const double gg = *g;
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (mask && !mask[i]) continue;
        const double d = __dsub_rn(T[i], __dmul_rn(gg, mag(i)));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    acc = block_sum64(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
static __global__ void k_mse64_final(const double* part, int nblk, double M, double* out) {
    if (threadIdx.x != 0) return;
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[b];
    *out = acc / M;
}

// Replay-plane constraint (ifta.hpp:185-224) in double.
struct Con64 {
    const double* amp;
    double* w;                 // WGS weights or nullptr
    const uint8_t* roi;
    const double2* tcs;        // (cos, sin) of the target phase (host libm) or nullptr (phase 0)
    int phase_freedom, amp_outside_roi;
    double lo, hi;
    int lt, x0, x1, y0, y1;
    int nx;
};
static __global__ void k_constrain64(double2* R, size_t n, Con64 c) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (!c.roi || c.roi[i]) {
            const int x = (int)(i % c.nx), y = (int)(i / c.nx);
            if (c.lt && !(x >= c.x0 && x < c.x1 && y >= c.y0 && y < c.y1)) continue;
            double a = c.amp[i];
            if (c.w && a > 0) {
                const double r = abs_rn64(R[i]);
                const double cand = __ddiv_rn(__dmul_rn(c.w[i], a), r < 1e-12 ? 1e-12 : r);  // std::max(r, 1e-12)
                const double cl = cand < c.lo ? c.lo : cand;                                 // std::max(cand, lo)
                c.w[i] = c.hi < cl ? c.hi : cl;                                              // std::min(., hi)
                a = __dmul_rn(a, c.w[i]);
            }
            if (c.phase_freedom) {
                const double2 z = R[i];
                const double r = abs_rn64(z);
                if (r > 0) {
                    const double s = __ddiv_rn(a, r);
                    R[i] = make_double2(__dmul_rn(z.x, s), __dmul_rn(z.y, s));
                } else {
                    R[i] = make_double2(a, 0.0);
                }
            } else {
                const double2 cs = c.tcs ? c.tcs[i] : make_double2(1.0, 0.0);
                R[i] = make_double2(__dmul_rn(a, cs.x), __dmul_rn(a, cs.y));
            }
        } else if (!c.amp_outside_roi) {
            R[i] = make_double2(0.0, 0.0);
        }
    }
}

// OSPR (ospr.hpp:105-116, :134-137): frame amplitude (adaptive budget) and
// the running intensity sum.
static __global__ void k_ospr_amp64(const double* T, const double* S, size_t n, int frame, double g, double* amp) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double t = T[i], t2 = __dmul_rn(t, t), nn = frame;
        const double budget = __dsub_rn(__dmul_rn(nn, t2), __dmul_rn(nn - 1.0, __ddiv_rn(S[i], nn - 1.0)));
        const double tn = __dsqrt_rn(budget > 0.0 ? budget : 0.0);  // std::max(0.0, budget)
        amp[i] = __dadd_rn(__dmul_rn(1.0 - g, t), __dmul_rn(g, tn));
    }
}
static __global__ void k_ospr_acc64(const double2* R, size_t n, double* S) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double2 z = R[i];
        S[i] = __dadd_rn(S[i], __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y)));
    }
}
static __global__ void k_ospr_out64(const double* S, size_t n, int N, double* mean, double2* replay) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double m = __ddiv_rn(S[i], (double)N);
        if (mean) mean[i] = m;
        if (replay) replay[i] = make_double2(__dsqrt_rn(m), 0.0);
    }
}

}  // namespace hg
