// quant.cuh — the SLM quantiser (Quantiser<T>::decide / state_value,
// quantise.hpp:175-205) as a device function fused into the row pass.
//
// Decision rule (phase mode): d = wrap_2pi(atan2(im, re) - illum_arg - min_arg);
//   full circle: k = lround(d/spac), k == L -> 0;
//   restricted : d <= range ? min(lround(d/spac), L-1)
//                           : (d - range <= 2pi - d ? L-1 : 0)   (watershed)
// amplitude mode: k = clamp(lround((|f| - min_amp)/spac), 0, L-1).
//
// The reference evaluates this in double (atan2/floor/lround).  Here a float
// fast path (atan2f) decides every pixel whose value is farther than a
// conservative margin from any decision boundary; pixels inside the margin
// (~1e-3 of them at 256 levels) are re-decided with the reference's exact
// double sequence (IEEE-rounded ops, no FMA contraction).  The margin bounds
// the float path's worst-case error, so the fast path never disagrees with
// the exact path; the only residual difference to the CPU is the ulp-level
// difference between CUDA's and glibc's double atan2 on exact-threshold inputs.
#pragma once
#include "common.cuh"

namespace hg {

struct QuantParams {
    int mode;  // 0 amplitude, 1 phase (SlmMode, quantise.hpp:14)
    int levels;
    int full_circle;
    int pad_;
    double min_arg, inv_spac, range, min_amp;  // exact (double) parameters
    float min_arg_f, inv_spac_f, range_f, min_amp_f;
    float wshed_f;    // watershed angle pi + range/2 (restricted phase mode)
    float margin_rad; // decision margin in radians (phase mode)
    float margin_u;   // same margin in level units
    float min_u_f;    // min_arg in level units (QK_FULL fast path)
    float2 s0, s1;    // states 0 and 1 (binary fast path)
    const float2* states;      // [levels] (T)allowed_states, quantise.hpp:147-149
    const double* illum_arg;   // [npix] arg(illumination) or nullptr
    const float2* illum;       // [npix] (T)illumination (phase mode) or nullptr
    const float2* illum_unit;  // [npix] (T)(illumination/|illumination|) or nullptr
};

// Exact reference sequence, quantise.hpp:175-198.  Out of line (scalar
// arguments, no struct copy) so the ~1e-3 of pixels that need it do not
// inflate every inlined copy of the fast path.
static __device__ __noinline__ int quant_decide_exact(int mode, int L, int full_circle, double min_arg, double inv_spac,
                                               double range, double min_amp, double illum_arg, float vr, float vi) {
    if (mode == 1) {
        double ang = atan2((double)vi, (double)vr);
        ang = __dsub_rn(ang, illum_arg);  // illum_arg = 0 without illumination (exact no-op)
        double d = __dsub_rn(ang, min_arg);
        d = __dsub_rn(d, __dmul_rn(HG_TWO_PI, floor(__ddiv_rn(d, HG_TWO_PI))));
        if (full_circle) {
            int k = (int)llround(__dmul_rn(d, inv_spac));
            return k >= L ? 0 : k;
        }
        if (d <= range) {
            int k = (int)llround(__dmul_rn(d, inv_spac));
            return k > L - 1 ? L - 1 : k;
        }
        return (__dsub_rn(d, range) <= __dsub_rn(HG_TWO_PI, d)) ? L - 1 : 0;
    }
    double re = vr, im = vi;
    double a = __dsqrt_rn(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
    long long k = llround(__dmul_rn(__dsub_rn(a, min_amp), inv_spac));
    if (k < 0) k = 0;
    if (k > L - 1) k = L - 1;
    return (int)k;
}

__device__ __forceinline__ int quant_decide(const QuantParams& q, float vr, float vi, size_t i) {
    const int L = q.levels;
    bool near;
    int k;
    if (q.mode == 1) {
        const float two_pi_f = 6.28318530717958648f;
        float ang = atan2f(vi, vr);
        if (q.illum_arg) ang -= (float)__ldg(&q.illum_arg[i]);
        float d = ang - q.min_arg_f;
        d -= two_pi_f * floorf(d * (1.0f / two_pi_f));
        float u = d * q.inv_spac_f;
        float fu = floorf(u);
        float fr = u - fu;
        near = fabsf(fr - 0.5f) < q.margin_u || d < q.margin_rad || d > two_pi_f - q.margin_rad;
        int kr = (int)fu + (fr >= 0.5f ? 1 : 0);
        if (q.full_circle) {
            k = kr >= L ? 0 : kr;
        } else if (d <= q.range_f) {
            k = kr > L - 1 ? L - 1 : kr;
        } else {
            near = near || fabsf(d - q.wshed_f) < q.margin_rad;
            k = d <= q.wshed_f ? L - 1 : 0;
        }
    } else {
        float a = sqrtf(vr * vr + vi * vi);
        float u = (a - q.min_amp_f) * q.inv_spac_f;
        float fu = floorf(u);
        float fr = u - fu;
        float m = (a * 4e-7f + fabsf(q.min_amp_f) * 2e-7f) * q.inv_spac_f + fabsf(u) * 4e-7f + 1e-6f;
        near = fabsf(fr - 0.5f) < m;
        int kr = (int)fu + (fr >= 0.5f ? 1 : 0);
        k = kr < 0 ? 0 : (kr > L - 1 ? L - 1 : kr);
    }
    if (near)
        k = quant_decide_exact(q.mode, L, q.full_circle, q.min_arg, q.inv_spac, q.range, q.min_amp,
                               q.illum_arg ? q.illum_arg[i] : 0.0, vr, vi);
    return k;
}

// ------------------------------------------------ specialised fast paths
// Quantiser kinds resolved on the host (launch template parameter):
//   QK_GENERIC  any SlmSpec (restricted ranges, amplitude, illumination)
//   QK_BINARY   SlmSpec::binary_phase() without illumination: the decision
//               is the sign of Re(f) (level 1 = pi state iff Re(f) < 0)
//   QK_FULL     full-circle phase without illumination
enum QuantKind { QK_GENERIC = 0, QK_BINARY = 1, QK_FULL = 2 };
#ifndef HG_STATES_SMEM  // QK_FULL row pass reads its state table from shared memory (<= 256 levels)
#define HG_STATES_SMEM 0
#endif

// atan2 in float without the library slow paths: odd degree-13 polynomial
// on [0,1] (max error 3.5e-7 rad in float) + octant fix-ups; total error
// < 2e-6 rad, far inside the 1e-5 rad decision margin.
__device__ __forceinline__ float fast_atan2f(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    float rmx;  // approximate reciprocal (<= 1 ulp); mx == 0 -> inf -> a = NaN, which the caller treats as "near"
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rmx) : "f"(mx));
    const float a = mn * rmx;
    const float s = a * a;
    float r = 0.0068426248975283f;
    r = fmaf(r, s, -0.03372593810402613f);
    r = fmaf(r, s, 0.07981120495604219f);
    r = fmaf(r, s, -0.13247522771620535f);
    r = fmaf(r, s, 0.19813213509066366f);
    r = fmaf(r, s, -0.3331830289944654f);
    r = fmaf(r, s, 0.999996634700673f);
    r *= a;
    r = ay > ax ? 1.5707963267948966f - r : r;
    r = x < 0.f ? 3.1415926535897932f - r : r;
    return copysignf(r, y);
}

template <int QK>
__device__ __forceinline__ int quant_decide_kind(const QuantParams& q, float vr, float vi, size_t i) {
    if constexpr (QK == QK_BINARY) {
        // atan2 within 1e-5 rad of +-pi/2 (or f == 0): defer to the exact path
        const bool near = !(fabsf(vr) > 1e-5f * fmaxf(fabsf(vr), fabsf(vi)));
        int k = vr < 0.f ? 1 : 0;
        if (near) k = quant_decide_exact(1, 2, 0, q.min_arg, q.inv_spac, q.range, 0.0, 0.0, vr, vi);
        return k;
    } else if constexpr (QK == QK_FULL) {
        // Directly in level units (L a power of two, quant_kind): u = atan2 * L/2pi
        // - min_arg * L/2pi, k = round(u) mod L.  The reference's wrap of the
        // angle into [0, 2pi) only adds multiples of L to u, so the mod takes its
        // place; the fast estimate's error (< 1e-4 levels at L = 256) stays far
        // inside margin_u.
        const float u = fmaf(fast_atan2f(vi, vr), q.inv_spac_f, -q.min_u_f);
        const float w = u + 0.5f;
        const float fk = floorf(w);
        const float fr = w - fk;  // 0 or 1 at a decision boundary
        const bool near = !(fabsf(fr - 0.5f) <= 0.5f - q.margin_u);  // NaN-safe
        int k = (int)fk & (q.levels - 1);
        if (near) k = quant_decide_exact(1, q.levels, 1, q.min_arg, q.inv_spac, q.range, 0.0, 0.0, vr, vi);
        return k;
    } else {
        return quant_decide(q, vr, vi, i);
    }
}

// Quantiser::state_value, quantise.hpp:201-205
__device__ __forceinline__ float2 quant_state(const QuantParams& q, int k, size_t i) {
    float2 s = __ldg(&q.states[k]);
    if (q.mode == 1) return q.illum ? cmul_rn(__ldg(&q.illum[i]), s) : s;
    return q.illum_unit ? cmul_rn(__ldg(&q.illum_unit[i]), s) : s;
}

}  // namespace hg
