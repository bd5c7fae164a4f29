/*
 * hg_oracle.c — CPU restatement of HoloGen's IFTA / OSPR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2008_12214_b200/ links, loads
 * or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker.
 *
 * Every function restates the reference (/root/reference/proj/include/
 * hologen/*.hpp) in plain C for T = float, citing file:line.  Arithmetic is
 * kept in the reference's order (double where the reference uses double,
 * float where it casts to T), and the file is compiled with
 * -ffp-contract=off so no FMA contraction changes a rounding.
 *
 * Pinning: tests/test_oracle_cpu.py checks this restatement bit-for-bit
 * against the reference headers compiled unmodified (oracle/_ref, built by
 * oracle/Makefile from /root/reference) and against the reference's golden
 * vectors (tests/golden/).  The FFT is the shared substitute in hgo_fft.h
 * (FFTW is absent; see that header).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hgo_fft.h"
#include "hgo_api.h"

#define TWO_PI 6.283185307179586476925286766559
#define PI_D 3.1415926535897932384626433832795

/* ---------------------------------------------------------------- rng ---- */

/* splitmix64 finaliser, rng.hpp:12-17 */
uint64_t hgo_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d4a2c62a2b3b9full;
    return z ^ (z >> 31);
}

/* Rng(seed).fork(stream) seeds its engine with this value, rng.hpp:42-44 */
uint64_t hgo_fork_seed(uint64_t seed, uint64_t stream) {
    return hgo_mix64(seed ^ hgo_mix64(stream + 1));
}

/* std::mt19937_64 (rng.hpp:25, :48): n=312, m=156, r=31,
 * a=0xB5026F5AA96619E9, standard seeding (f=6364136223846793005) and
 * tempering (u=29,d=0x5555555555555555, s=17,b=0x71D67FFFEDA60000,
 * t=37,c=0xFFF7EEE000000000, l=43). */
#define MT_N 312
#define MT_M 156
#define MT_UM 0xFFFFFFFF80000000ull
#define MT_LM 0x000000007FFFFFFFull
#define MT_A 0xB5026F5AA96619E9ull

typedef struct {
    uint64_t mt[MT_N];
    int idx;
} hgo_mt64;

void hgo_mt_seed(hgo_mt64 *s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = MT_N;
}

static void mt_twist(hgo_mt64 *s) {
    uint64_t *mt = s->mt;
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
        uint64_t x = (mt[i] & MT_UM) | (mt[i + 1] & MT_LM);
        mt[i] = mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    }
    for (; i < MT_N - 1; ++i) {
        uint64_t x = (mt[i] & MT_UM) | (mt[i + 1] & MT_LM);
        mt[i] = mt[i + MT_M - MT_N] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    }
    uint64_t x = (mt[MT_N - 1] & MT_UM) | (mt[0] & MT_LM);
    mt[MT_N - 1] = mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    s->idx = 0;
}

uint64_t hgo_mt_next(hgo_mt64 *s) {
    if (s->idx >= MT_N) mt_twist(s);
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

size_t hgo_mt_state_size(void) { return sizeof(hgo_mt64); }

/* n raw engine outputs after discarding `skip`, engine seeded with `seed`. */
void hgo_mt_draws(uint64_t seed, uint64_t skip, size_t n, uint64_t *out) {
    hgo_mt64 s;
    hgo_mt_seed(&s, seed);
    for (uint64_t i = 0; i < skip; ++i) (void)hgo_mt_next(&s);
    for (size_t i = 0; i < n; ++i) out[i] = hgo_mt_next(&s);
}

/* Rng::uniform01, rng.hpp:32 */
static double uniform01(hgo_mt64 *s) { return (double)(hgo_mt_next(s) >> 11) * 0x1.0p-53; }

/* seed_random_phase<float>, rng.hpp:54-67: one draw per pixel, row-major,
 * zero-amplitude pixels included. */
void hgo_seed_random_phase(const double *amp, size_t n, hgo_mt64 *s, float *out) {
    for (size_t i = 0; i < n; ++i) {
        double theta = TWO_PI * uniform01(s);
        double a = amp[i];
        out[2 * i] = (float)(a * cos(theta));
        out[2 * i + 1] = (float)(a * sin(theta));
    }
}

/* Convenience: Rng(seed).fork(0) stream, skipping `skip_pixels` draws. */
void hgo_seed_random_phase_seeded(const double *amp, size_t n, uint64_t seed,
                                  uint64_t skip_pixels, float *out) {
    hgo_mt64 s;
    hgo_mt_seed(&s, hgo_fork_seed(seed, 0));
    for (uint64_t i = 0; i < skip_pixels; ++i) (void)hgo_mt_next(&s);
    hgo_seed_random_phase(amp, n, &s, out);
}

/* ---------------------------------------------------------- quantiser ---- */

typedef struct {
    hgo_slm spec;
    size_t n;
    double spac, inv_spac, range;
    float *states; /* 2*levels */
    double *illum_arg;
    float *illum_unit, *illum;
} hgo_quant;

/* SlmSpec::spacing, quantise.hpp:99-104 */
static double slm_spacing(const hgo_slm *s) {
    if (s->mode == 1) return s->full_circle ? TWO_PI / s->levels : (s->max_arg - s->min_arg) / (s->levels - 1);
    return (s->max_amp - s->min_amp) / (s->levels - 1);
}

/* SlmSpec::validate, quantise.hpp:71-96 (returns message or NULL) */
const char *hgo_slm_validate(const hgo_slm *s, size_t n) {
    if (s->levels < 2) return "SlmSpec: levels must be >= 2";
    if (s->mode == 1) {
        if (!isfinite(s->min_arg) || !isfinite(s->max_arg)) return "SlmSpec: phase range must be finite";
        if (!(s->min_arg < s->max_arg) || s->max_arg - s->min_arg > TWO_PI * (1 + 1e-12))
            return "SlmSpec: phase range must satisfy min_arg < max_arg <= min_arg + 2*pi";
        if (s->full_circle && fabs((s->max_arg - s->min_arg) - TWO_PI) > 1e-9)
            return "SlmSpec: full_circle requires a 2*pi range";
    } else {
        if (!isfinite(s->min_amp) || !isfinite(s->max_amp)) return "SlmSpec: amplitude range must be finite";
        if (!(s->min_amp >= 0) || !(s->min_amp < s->max_amp)) return "SlmSpec: need 0 <= min_amp < max_amp";
    }
    if (s->illum) {
        for (size_t i = 0; i < n; ++i) {
            double re = s->illum[2 * i], im = s->illum[2 * i + 1];
            if (!isfinite(re) || !isfinite(im)) return "SlmSpec: illumination must be finite";
            if (re == 0.0 && im == 0.0) return "SlmSpec: illumination must be nowhere zero";
        }
    }
    return NULL;
}

/* Quantiser ctor, quantise.hpp:139-166; allowed_states :111-124 */
static void quant_init(hgo_quant *q, const hgo_slm *spec, size_t n) {
    q->spec = *spec;
    q->n = n;
    q->spac = slm_spacing(spec);
    q->inv_spac = 1.0 / q->spac;
    q->range = spec->mode == 1 ? spec->max_arg - spec->min_arg : 0.0;
    q->states = (float *)malloc(sizeof(float) * 2 * (size_t)spec->levels);
    for (int k = 0; k < spec->levels; ++k) {
        if (spec->mode == 1) {
            double a = spec->min_arg + k * q->spac;
            q->states[2 * k] = (float)cos(a);
            q->states[2 * k + 1] = (float)sin(a);
        } else {
            q->states[2 * k] = (float)(spec->min_amp + k * q->spac);
            q->states[2 * k + 1] = 0.0f;
        }
    }
    q->illum_arg = NULL;
    q->illum_unit = q->illum = NULL;
    if (spec->illum) {
        q->illum_arg = (double *)malloc(sizeof(double) * n);
        q->illum_unit = (float *)malloc(sizeof(float) * 2 * n);
        q->illum = (float *)malloc(sizeof(float) * 2 * n);
        for (size_t i = 0; i < n; ++i) {
            double re = spec->illum[2 * i], im = spec->illum[2 * i + 1];
            double a = hypot(re, im); /* std::abs(complex<double>) */
            q->illum_arg[i] = atan2(im, re);
            q->illum_unit[2 * i] = (float)(re / a);
            q->illum_unit[2 * i + 1] = (float)(im / a);
            q->illum[2 * i] = (float)re;
            q->illum[2 * i + 1] = (float)im;
        }
    }
}

static void quant_free(hgo_quant *q) {
    free(q->states);
    free(q->illum_arg);
    free(q->illum_unit);
    free(q->illum);
}

/* Quantiser::decide, quantise.hpp:175-198 */
static int quant_decide(const hgo_quant *q, size_t i, float vr, float vi) {
    const hgo_slm *s = &q->spec;
    int L = s->levels;
    if (s->mode == 1) {
        double ang = atan2((double)vi, (double)vr);
        if (q->illum_arg) ang -= q->illum_arg[i];
        double d = ang - s->min_arg;
        d -= TWO_PI * floor(d / TWO_PI);
        if (s->full_circle) {
            int k = (int)lround(d * q->inv_spac);
            return k >= L ? 0 : k;
        }
        if (d <= q->range) {
            int k = (int)lround(d * q->inv_spac);
            return k > L - 1 ? L - 1 : k;
        }
        return (d - q->range <= TWO_PI - d) ? L - 1 : 0;
    }
    double re = vr, im = vi;
    double a = sqrt(re * re + im * im);
    long k = lround((a - s->min_amp) * q->inv_spac);
    if (k < 0) k = 0;
    if (k > L - 1) k = L - 1;
    return (int)k;
}

/* complex<float> product as GCC evaluates it on x86-64 (no FMA):
 * (a+bi)(c+di) = (ac - bd) + (ad + bc)i, each product rounded to float. */
static inline void cmulf(float ar, float ai, float br, float bi, float *or_, float *oi) {
    float ac = ar * br, bd = ai * bi, ad = ar * bi, bc = ai * br;
    *or_ = ac - bd;
    *oi = ad + bc;
}

/* Quantiser::state_value, quantise.hpp:201-205 */
static inline void quant_state(const hgo_quant *q, size_t i, int k, float *or_, float *oi) {
    float sr = q->states[2 * k], si = q->states[2 * k + 1];
    if (q->spec.mode == 1) {
        if (!q->illum) { *or_ = sr; *oi = si; return; }
        cmulf(q->illum[2 * i], q->illum[2 * i + 1], sr, si, or_, oi);
        return;
    }
    if (!q->illum_unit) { *or_ = sr; *oi = si; return; }
    cmulf(q->illum_unit[2 * i], q->illum_unit[2 * i + 1], sr, si, or_, oi);
}

/* Quantiser::apply, quantise.hpp:208-216 */
static void quant_apply(const hgo_quant *q, float *f, int32_t *levels) {
    for (size_t i = 0; i < q->n; ++i) {
        int k = quant_decide(q, i, f[2 * i], f[2 * i + 1]);
        quant_state(q, i, k, &f[2 * i], &f[2 * i + 1]);
        if (levels) levels[i] = k;
    }
}

/* Public one-shot quantiser (quantise_field without the domain check). */
int hgo_quantise(const hgo_slm *spec, int nx, int ny, float *field, int32_t *levels) {
    size_t n = (size_t)nx * ny;
    if (hgo_slm_validate(spec, n)) return -1;
    hgo_quant q;
    quant_init(&q, spec, n);
    quant_apply(&q, field, levels);
    quant_free(&q);
    return 0;
}

/* Quantiser states as float (T-cast of allowed_states), quantise.hpp:147-149 */
void hgo_quant_states(const hgo_slm *spec, float *out) {
    hgo_quant q;
    quant_init(&q, spec, 0);
    memcpy(out, q.states, sizeof(float) * 2 * (size_t)spec->levels);
    quant_free(&q);
}

/* ---------------------------------------------------------- fresnel ---- */

/* make_fresnel_phase<float>, propagation.hpp:36-54 */
void hgo_fresnel_q(int nx, int ny, double wavelength, double distance, double px, double py, float *q) {
    double cx = nx / 2.0, cy = ny / 2.0;
    double scale = PI_D / (wavelength * distance);
    for (int y = 0; y < ny; ++y) {
        double dy = (y - cy) * py;
        double ty = dy * dy;
        for (int x = 0; x < nx; ++x) {
            double dx = (x - cx) * px;
            double phase = scale * (dx * dx + ty);
            size_t i = (size_t)y * nx + x;
            q[2 * i] = (float)cos(phase);
            q[2 * i + 1] = (float)sin(phase);
        }
    }
}

/* ------------------------------------------------------------- fft ---- */

/* FftBackend<float>::forward/inverse contract (fft.hpp:17-27) with the
 * substitute transform of hgo_fft.h.  sign -1 forward, +1 inverse. */
void hgo_fft2d(int nx, int ny, int sign, const float *in, float *out) {
    hgo_fft2d_precise(nx, ny, sign, in, out);
}
void hgo_fft2d_d(int nx, int ny, int sign, const double *in, double *out) {
    hgo_fft2d_precise_d(nx, ny, sign, in, out);
}
void hgo_fft2d_fastf(int nx, int ny, int sign, const float *in, float *out) {
    hgo_fft2d_fast(nx, ny, sign, in, out);
}

/* ------------------------------------------------------------- mse ---- */

/* mse(), phase-insensitive branch, metrics.hpp:70-97 and :123.
 * replay is complex float (T=float) or complex double (dbl != 0). */
static double mse_impl(const double *t, const void *replay, int dbl, const uint8_t *mask, size_t n,
                       int scale_free) {
    size_t m = 0;
    double acc = 0.0, g = 1.0;
    const float *rf = (const float *)replay;
    const double *rd = (const double *)replay;
#define RE(i) (dbl ? rd[2 * (i)] : (double)rf[2 * (i)])
#define IM(i) (dbl ? rd[2 * (i) + 1] : (double)rf[2 * (i) + 1])
    if (scale_free) {
        double s_tr = 0.0, s_rr = 0.0;
        for (size_t i = 0; i < n; ++i) {
            if (mask && mask[i] == 0) continue;
            double re = RE(i), im = IM(i);
            double r = sqrt(re * re + im * im);
            s_tr += t[i] * r;
            s_rr += r * r;
        }
        g = s_rr > 0.0 ? s_tr / s_rr : 0.0;
        if (g < 0.0) g = 0.0;
    }
    for (size_t i = 0; i < n; ++i) {
        if (mask && mask[i] == 0) continue;
        double re = RE(i), im = IM(i);
        double d = t[i] - g * sqrt(re * re + im * im);
        acc += d * d;
        ++m;
    }
#undef RE
#undef IM
    return acc / (double)m;
}

double hgo_mse(const double *t, const float *replay, const uint8_t *mask, size_t n, int scale_free) {
    return mse_impl(t, replay, 0, mask, n, scale_free);
}

/* ------------------------------------------------------------ ifta ---- */

/* ifta.hpp:74-84 */
static void lt_rect(int bx0, int by0, int bw, int bh, double fraction, int *x0, int *x1, int *y0, int *y1) {
    double side = sqrt(fraction);
    int aw = (int)lround(bw * side);
    int ah = (int)lround(bh * side);
    if (aw < 1) aw = 1;
    if (ah < 1) ah = 1;
    *x0 = bx0 + (bw - aw) / 2;
    *y0 = by0 + (bh - ah) / 2;
    *x1 = *x0 + aw;
    *y1 = *y0 + ah;
}

/* detail::run_ifta<float>, ifta.hpp:86-235.  Returns 0 or -1 (bad input).
 * hologram/replay: 2*npix floats; levels: npix int32 of the last
 * quantisation; trace: iterations doubles. */
/* Test hook (lock-step parity, tests/test_gpu_lockstep.py): at the start of
 * each iteration k listed in snap_iters[0..nsnap), the replay field R_{k-1}
 * (2*npix floats) and the WGS weights (npix doubles) are copied to slot j of
 * snaps_r / snaps_w, and the level indices of iteration k to snaps_lv. */
static int g_nsnap;
static const int *g_snap_iters;
static float *g_snaps_r;
static double *g_snaps_w;
static int32_t *g_snaps_lv;

int hgo_ifta_run(const hgo_ifta_cfg *cfg, const hgo_slm *slm, int nx, int ny, const double *amp,
                 const double *phase_turns, const uint8_t *roi, const float *init_field,
                 const double *init_weights, float *hologram, float *replay, int32_t *levels,
                 double *trace, float *snap_r, double *snap_w);

/* hgo_ifta_run with the snapshot lists above (not re-entrant: test use only). */
int hgo_ifta_run_snaps(const hgo_ifta_cfg *cfg, const hgo_slm *slm, int nx, int ny, const double *amp,
                       const double *phase_turns, const uint8_t *roi, float *hologram, float *replay,
                       int32_t *levels, double *trace, int nsnap, const int *snap_iters, float *snaps_r,
                       double *snaps_w, int32_t *snaps_lv) {
    g_nsnap = nsnap;
    g_snap_iters = snap_iters;
    g_snaps_r = snaps_r;
    g_snaps_w = snaps_w;
    g_snaps_lv = snaps_lv;
    int rc = hgo_ifta_run(cfg, slm, nx, ny, amp, phase_turns, roi, NULL, NULL, hologram, replay, levels, trace,
                          NULL, NULL);
    g_nsnap = 0;
    return rc;
}

int hgo_ifta_run(const hgo_ifta_cfg *cfg, const hgo_slm *slm, int nx, int ny, const double *amp,
                 const double *phase_turns, const uint8_t *roi, const float *init_field,
                 const double *init_weights, float *hologram, float *replay, int32_t *levels,
                 double *trace, float *snap_r, double *snap_w) {
    size_t n = (size_t)nx * ny;
    if (cfg->iterations < 1) return -1;
    if (hgo_slm_validate(slm, n)) return -1;
    hgo_quant q;
    quant_init(&q, slm, n);
    float *Q = NULL;
    if (cfg->fresnel) {
        Q = (float *)malloc(sizeof(float) * 2 * n);
        hgo_fresnel_q(nx, ny, cfg->wavelength, cfg->distance, cfg->pitch_x, cfg->pitch_y, Q);
    }
    double *tphase = NULL;
    if (phase_turns) {
        tphase = (double *)malloc(sizeof(double) * n);
        for (size_t i = 0; i < n; ++i) tphase[i] = TWO_PI * phase_turns[i];
    }
    float *R = (float *)malloc(sizeof(float) * 2 * n);
    float *f = (float *)malloc(sizeof(float) * 2 * n);
    float *tmp = (float *)malloc(sizeof(float) * 2 * n);
    int target_phase_init = cfg->init_phase == 0 && phase_turns && !cfg->phase_freedom;
    if (cfg->init_phase == 3) {
        memcpy(R, init_field, sizeof(float) * 2 * n);
    } else if (cfg->init_phase == 2) { /* :128-130 */
        for (size_t i = 0; i < n; ++i) { R[2 * i] = (float)amp[i]; R[2 * i + 1] = 0.0f; }
    } else if (target_phase_init) { /* :131-136 */
        for (size_t i = 0; i < n; ++i) {
            double a = amp[i];
            R[2 * i] = (float)(a * cos(tphase[i]));
            R[2 * i + 1] = (float)(a * sin(tphase[i]));
        }
    } else { /* :137-139 */
        hgo_mt64 s;
        hgo_mt_seed(&s, hgo_fork_seed(cfg->seed, 0));
        hgo_seed_random_phase(amp, n, &s, R);
    }
    double *w = NULL;
    if (cfg->variant == 1) { /* :141-142 */
        w = (double *)malloc(sizeof(double) * n);
        for (size_t i = 0; i < n; ++i) w[i] = init_weights ? init_weights[i] : 1.0;
    }
    /* LT schedule, ifta.hpp:55-63 and :144-163 */
    double *fractions = NULL;
    int bx0 = 0, by0 = 0, bw = nx, bh = ny;
    if (cfg->variant == 2) {
        int K = cfg->iterations;
        fractions = (double *)malloc(sizeof(double) * K);
        for (int k = 1; k < K; ++k)
            fractions[k - 1] = cfg->lt_initial_fraction + (1.0 - cfg->lt_initial_fraction) * (k - 1) / (K - 1);
        fractions[K - 1] = 1.0;
        if (roi) {
            bx0 = nx; by0 = ny;
            int bx1 = -1, by1 = -1;
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x)
                    if (roi[(size_t)y * nx + x]) {
                        if (x < bx0) bx0 = x;
                        if (x > bx1) bx1 = x;
                        if (y < by0) by0 = y;
                        if (y > by1) by1 = y;
                    }
            bw = bx1 - bx0 + 1;
            bh = by1 - by0 + 1;
        }
    }

    for (int k = 1; k <= cfg->iterations; ++k) {
        if (k == cfg->snapshot_iter) {
            if (snap_r) memcpy(snap_r, R, sizeof(float) * 2 * n);
            if (snap_w && w) memcpy(snap_w, w, sizeof(double) * n);
        }
        for (int j = 0; j < g_nsnap; ++j)
            if (g_snap_iters[j] == k) {
                memcpy(g_snaps_r + (size_t)j * 2 * n, R, sizeof(float) * 2 * n);
                if (g_snaps_w && w) memcpy(g_snaps_w + (size_t)j * n, w, sizeof(double) * n);
            }
        /* f = prop.inverse(R), propagation.hpp:89-95 */
        hgo_fft2d_precise(nx, ny, +1, R, f);
        if (Q)
            for (size_t i = 0; i < n; ++i) {
                float a = f[2 * i], b = f[2 * i + 1];
                cmulf(a, b, Q[2 * i], -Q[2 * i + 1], &f[2 * i], &f[2 * i + 1]);
            }
        /* quant.apply(f), ifta.hpp:172 */
        quant_apply(&q, f, levels);
        for (int j = 0; j < g_nsnap; ++j)
            if (g_snap_iters[j] == k && g_snaps_lv) memcpy(g_snaps_lv + (size_t)j * n, levels, sizeof(int32_t) * n);
        /* R = prop.forward(f), propagation.hpp:81-87 */
        if (Q) {
            for (size_t i = 0; i < n; ++i)
                cmulf(f[2 * i], f[2 * i + 1], Q[2 * i], Q[2 * i + 1], &tmp[2 * i], &tmp[2 * i + 1]);
            hgo_fft2d_precise(nx, ny, -1, tmp, R);
        } else {
            hgo_fft2d_precise(nx, ny, -1, f, R);
        }
        /* trace, ifta.hpp:180 */
        trace[k - 1] = mse_impl(amp, R, 0, roi, n, cfg->scale_freedom);
        if (k == cfg->iterations) break;
        /* replay-plane constraint, ifta.hpp:185-224 */
        int lt = cfg->variant == 2, ax0 = 0, ax1 = 0, ay0 = 0, ay1 = 0;
        if (lt) lt_rect(bx0, by0, bw, bh, fractions[k - 1], &ax0, &ax1, &ay0, &ay1);
        for (int y = 0; y < ny; ++y) {
            for (int x = 0; x < nx; ++x) {
                size_t i = (size_t)y * nx + x;
                if (!roi || roi[i]) {
                    if (lt && !(x >= ax0 && x < ax1 && y >= ay0 && y < ay1)) continue;
                    double a = amp[i];
                    if (w && a > 0) {
                        double re = R[2 * i], im = R[2 * i + 1];
                        double r = sqrt(re * re + im * im);
                        /* std::max / std::min operand order, ifta.hpp:201-202 */
                        double rr = (r < 1e-12) ? 1e-12 : r;
                        double cand = w[i] * a / rr;
                        double c = (cand < cfg->clamp_lo) ? cfg->clamp_lo : cand;
                        w[i] = (cfg->clamp_hi < c) ? cfg->clamp_hi : c;
                        a *= w[i];
                    }
                    if (cfg->phase_freedom) {
                        double re = R[2 * i], im = R[2 * i + 1];
                        double r = sqrt(re * re + im * im);
                        if (r > 0) {
                            double s = a / r;
                            R[2 * i] = (float)(re * s);
                            R[2 * i + 1] = (float)(im * s);
                        } else {
                            R[2 * i] = (float)a;
                            R[2 * i + 1] = 0.0f;
                        }
                    } else {
                        double ph = tphase ? tphase[i] : 0.0;
                        R[2 * i] = (float)(a * cos(ph));
                        R[2 * i + 1] = (float)(a * sin(ph));
                    }
                } else if (!cfg->amp_outside_roi) {
                    R[2 * i] = 0.0f;
                    R[2 * i + 1] = 0.0f;
                }
            }
        }
    }
    if (hologram) memcpy(hologram, f, sizeof(float) * 2 * n);
    if (replay) memcpy(replay, R, sizeof(float) * 2 * n);
    quant_free(&q);
    free(Q); free(tphase); free(R); free(f); free(tmp); free(w); free(fractions);
    return 0;
}

/* One IFTA iteration body without the constraint, for lock-step checks:
 * given R entering iteration k, produce f (quantised), levels, R' and mse. */

/* ------------------------------------------------------------ ospr ---- */

/* detail::run_ospr_impl<float>, ospr.hpp:68-164.
 * levels: N*npix int32 or NULL; frames: N*2*npix floats or NULL. */
int hgo_ospr_run(int adaptive, int subframes, uint64_t seed, double gain, const hgo_slm *slm, int nx,
                 int ny, const double *target, const uint8_t *roi, int scale_free, int32_t *levels,
                 float *frames, double *frame_mse, double *cum_mse, double *mean_intensity,
                 float *replay) {
    size_t n = (size_t)nx * ny;
    int N = subframes;
    if (N < 1) return -1;
    if (hgo_slm_validate(slm, n)) return -1;
    double g = adaptive ? gain : 0.0;
    hgo_quant q;
    quant_init(&q, slm, n);
    hgo_mt64 s;
    hgo_mt_seed(&s, hgo_fork_seed(seed, 0)); /* ospr.hpp:89 */
    double *t2 = (double *)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) t2[i] = target[i] * target[i];
    double *S = (double *)calloc(n, sizeof(double));
    double *amp = (double *)malloc(sizeof(double) * n);
    float *seeded = (float *)malloc(sizeof(float) * 2 * n);
    float *f = (float *)malloc(sizeof(float) * 2 * n);
    float *R = (float *)malloc(sizeof(float) * 2 * n);
    double *cum = (double *)malloc(sizeof(double) * 2 * n);
    for (int k = 1; k <= N; ++k) {
        if (!adaptive || k == 1) {
            memcpy(amp, target, sizeof(double) * n);
        } else { /* :111-115 */
            for (size_t i = 0; i < n; ++i) {
                double budget = k * t2[i] - (k - 1) * (S[i] / (k - 1));
                double tn = sqrt(budget > 0.0 ? budget : 0.0);
                amp[i] = (1.0 - g) * target[i] + g * tn;
            }
        }
        hgo_seed_random_phase(amp, n, &s, seeded);             /* :118 */
        hgo_fft2d_precise(nx, ny, +1, seeded, f);              /* :120 */
        quant_apply(&q, f, levels ? levels + (size_t)(k - 1) * n : NULL); /* :124 */
        hgo_fft2d_precise(nx, ny, -1, f, R);                   /* :128 */
        if (frames) memcpy(frames + (size_t)(k - 1) * 2 * n, f, sizeof(float) * 2 * n);
        for (size_t i = 0; i < n; ++i) {                       /* :134-137 */
            double re = R[2 * i], im = R[2 * i + 1];
            S[i] += re * re + im * im;
        }
        frame_mse[k - 1] = mse_impl(target, R, 0, roi, n, scale_free);   /* :138 */
        for (size_t i = 0; i < n; ++i) {                       /* :142-145 */
            cum[2 * i] = sqrt(S[i] / k);
            cum[2 * i + 1] = 0.0;
        }
        cum_mse[k - 1] = mse_impl(target, cum, 1, roi, n, scale_free);
    }
    for (size_t i = 0; i < n; ++i) {                           /* :149-156 */
        if (mean_intensity) mean_intensity[i] = S[i] / N;
        if (replay) {
            replay[2 * i] = (float)sqrt(S[i] / N);
            replay[2 * i + 1] = 0.0f;
        }
    }
    quant_free(&q);
    free(t2); free(S); free(amp); free(seeded); free(f); free(R); free(cum);
    return 0;
}

/* (1/sqrt(N)) * sum MSE_n, ospr.hpp:58-64 */
double hgo_subframe_mse_statistic(const double *per_frame, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += per_frame[i];
    return s / sqrt((double)n);
}
