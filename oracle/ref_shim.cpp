// ref_shim.cpp — the REFERENCE ITSELF, compiled here from its unmodified
// headers (/root/reference/proj/include/hologen/*.hpp), behind a flat
// extern "C" surface so Python tests can call it.  TEST INFRASTRUCTURE ONLY
// (oracle/_ref/libhgref.so; see oracle/Makefile).
//
// The only piece supplied here is the FFT: the reference's production
// backend (proj/src/fftw_backend.cpp) needs FFTW3, which is absent, so
// default_fft_backend<T>() (declared fft.hpp:82-83) is defined with the
// substitute transform of hgo_fft.h.  A process-wide switch selects the
// double-accumulating "precise" transform (parity) or the float
// "fast" transform (CPU-baseline timing only).
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "hologen/fft.hpp"
#include "hologen/ifta.hpp"
#include "hologen/metrics.hpp"
#include "hologen/ospr.hpp"
#include "hologen/patterns.hpp"
#include "hologen/propagation.hpp"
#include "hologen/quantise.hpp"
#include "hologen/rng.hpp"
#include "hologen/target.hpp"

#include "hgo_api.h"
#include "hgo_fft.h"

namespace {
std::atomic<int> g_fast_fft{0};
thread_local std::string g_err;

template <typename T>
class SubstituteBackend : public hologen::FftBackend<T> {
public:
    const char* name() const override { return g_fast_fft.load() ? "substitute-fast-f32" : "substitute-precise"; }
    void forward(int nx, int ny, const std::complex<T>* in, std::complex<T>* out) override { run(nx, ny, in, out, -1); }
    void inverse(int nx, int ny, const std::complex<T>* in, std::complex<T>* out) override { run(nx, ny, in, out, +1); }

private:
    static void run(int nx, int ny, const std::complex<T>* in, std::complex<T>* out, int sign) {
        if constexpr (std::is_same_v<T, float>) {
            auto* i = reinterpret_cast<const float*>(in);
            auto* o = reinterpret_cast<float*>(out);
            if (g_fast_fft.load()) hgo_fft2d_fast(nx, ny, sign, i, o);
            else hgo_fft2d_precise(nx, ny, sign, i, o);
        } else {
            hgo_fft2d_precise_d(nx, ny, sign, reinterpret_cast<const double*>(in),
                                reinterpret_cast<double*>(out));
        }
    }
};
}  // namespace

namespace hologen {
template <typename T>
FftBackend<T>& default_fft_backend() {
    static SubstituteBackend<T> b;
    return b;
}
template FftBackend<float>& default_fft_backend<float>();
template FftBackend<double>& default_fft_backend<double>();

template <typename T>
std::unique_ptr<FftBackend<T>> make_fft_backend(int) {
    return std::make_unique<SubstituteBackend<T>>();
}
template std::unique_ptr<FftBackend<float>> make_fft_backend<float>(int);
template std::unique_ptr<FftBackend<double>> make_fft_backend<double>(int);
}  // namespace hologen

using namespace hologen;

namespace {

SlmSpec to_spec(const hgo_slm* s, int nx, int ny) {
    SlmSpec spec;
    spec.mode = s->mode == 1 ? SlmMode::Phase : SlmMode::Amplitude;
    spec.levels = s->levels;
    spec.min_arg = s->min_arg;
    spec.max_arg = s->max_arg;
    spec.full_circle = s->full_circle != 0;
    spec.min_amp = s->min_amp;
    spec.max_amp = s->max_amp;
    if (s->illum) {
        ComplexField<double> il(nx, ny, Domain::Aperture);
        std::memcpy(il.data.data(), s->illum, sizeof(double) * 2 * il.data.size());
        spec.illumination = il;
    }
    return spec;
}

RealImage to_image(const double* p, int nx, int ny) {
    RealImage img(nx, ny);
    std::memcpy(img.data.data(), p, sizeof(double) * img.data.size());
    return img;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* hgr_last_error() { return g_err.c_str(); }
void hgr_set_fast_fft(int on) { g_fast_fft.store(on); }

uint64_t hgr_mix64(uint64_t z) { return detail::mix64(z); }
uint64_t hgr_fork_seed(uint64_t seed, uint64_t stream) { return Rng(seed).fork(stream).seed(); }

void hgr_mt_draws(uint64_t seed, uint64_t skip, size_t n, uint64_t* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < skip; ++i) (void)r.next_u64();
    for (size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

int hgr_seed_random_phase(const double* amp, int nx, int ny, uint64_t seed, uint64_t skip, float* out) {
    return guard([&] {
        Rng rng = Rng(seed).fork(0);
        for (uint64_t i = 0; i < skip; ++i) (void)rng.next_u64();
        auto f = seed_random_phase<float>(to_image(amp, nx, ny), rng);
        std::memcpy(out, f.data.data(), sizeof(float) * 2 * f.data.size());
    });
}

int hgr_quantise(const hgo_slm* s, int nx, int ny, float* field, int32_t* levels) {
    return guard([&] {
        Quantiser<float> q(to_spec(s, nx, ny), nx, ny);
        ComplexField<float> f(nx, ny, Domain::Aperture);
        std::memcpy(f.data.data(), field, sizeof(float) * 2 * f.data.size());
        std::vector<int32_t> lv;
        q.apply(f, &lv);
        std::memcpy(field, f.data.data(), sizeof(float) * 2 * f.data.size());
        if (levels) std::memcpy(levels, lv.data(), sizeof(int32_t) * lv.size());
    });
}

void hgr_quant_states(const hgo_slm* s, float* out) {
    auto st = allowed_states(to_spec(s, 1, 1));
    for (size_t k = 0; k < st.size(); ++k) {
        out[2 * k] = static_cast<float>(st[k].real());
        out[2 * k + 1] = static_cast<float>(st[k].imag());
    }
}

int hgr_fresnel_q(int nx, int ny, double wl, double z, double px, double py, float* q) {
    return guard([&] {
        FresnelParams p{wl, z, px, py};
        auto v = make_fresnel_phase<float>(nx, ny, p);
        std::memcpy(q, v.data(), sizeof(float) * 2 * v.size());
    });
}

// fft_forward / fft_inverse (fft.hpp:93-113) through the default backend,
// or the reference's own NaiveDftBackend (fft.hpp:32-77) when naive != 0.
int hgr_fft(int nx, int ny, int sign, int naive, const float* in, float* out) {
    return guard([&] {
        NaiveDftBackend<float> nb;
        FftBackend<float>* b = naive ? &nb : nullptr;
        ComplexField<float> f(nx, ny, sign < 0 ? Domain::Aperture : Domain::Replay);
        std::memcpy(f.data.data(), in, sizeof(float) * 2 * f.data.size());
        auto F = sign < 0 ? fft_forward(f, b) : fft_inverse(f, b);
        std::memcpy(out, F.data.data(), sizeof(float) * 2 * F.data.size());
    });
}

int hgr_fft_d(int nx, int ny, int sign, int naive, const double* in, double* out) {
    return guard([&] {
        NaiveDftBackend<double> nb;
        FftBackend<double>* b = naive ? &nb : nullptr;
        ComplexField<double> f(nx, ny, sign < 0 ? Domain::Aperture : Domain::Replay);
        std::memcpy(f.data.data(), in, sizeof(double) * 2 * f.data.size());
        auto F = sign < 0 ? fft_forward(f, b) : fft_inverse(f, b);
        std::memcpy(out, F.data.data(), sizeof(double) * 2 * F.data.size());
    });
}

int hgr_mse(const double* t, const float* r, const uint8_t* mask, int nx, int ny, int scale_free,
            double* out) {
    return guard([&] {
        MetricConfig c;
        c.scale_free = scale_free != 0;
        if (mask) {
            RegionMask m(nx, ny);
            std::memcpy(m.data.data(), mask, m.data.size());
            c.mask = m;
        }
        ComplexField<float> R(nx, ny, Domain::Replay);
        std::memcpy(R.data.data(), r, sizeof(float) * 2 * R.data.size());
        *out = mse(to_image(t, nx, ny), R, c);
    });
}

void hgr_smooth_blobs(int w, int h, double* out) {
    auto img = patterns::smooth_blobs(w, h);
    std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
}

int hgr_normalize(double* img, int w, int h, int unit_energy) {
    return guard([&] {
        RealImage r = to_image(img, w, h);
        normalize_image(r, unit_energy ? Normalization::UnitEnergy : Normalization::MaxToOne);
        std::memcpy(img, r.data.data(), sizeof(double) * r.data.size());
    });
}

// run_ifta<float> (ifta.hpp:86-263).  levels are re-derived from the
// returned hologram with Quantiser::decide, as runner.cpp:259-262 does.
int hgr_ifta_run(const hgo_ifta_cfg* c, const hgo_slm* s, int nx, int ny, const double* amp,
                 const double* phase_turns, const uint8_t* roi, float* hologram, float* replay,
                 int32_t* levels, double* trace, double* timing) {
    return guard([&] {
        IftaConfig cfg;
        cfg.variant = c->variant == 0   ? IftaVariant::GS
                      : c->variant == 1 ? IftaVariant::WeightedGS
                                        : IftaVariant::LiuTaghizadeh;
        cfg.iterations = c->iterations;
        cfg.slm = to_spec(s, nx, ny);
        cfg.target.amplitude = to_image(amp, nx, ny);
        if (phase_turns) cfg.target.phase = to_image(phase_turns, nx, ny);
        if (roi) {
            RegionMask m(nx, ny);
            std::memcpy(m.data.data(), roi, m.data.size());
            cfg.target.roi = m;
        }
        cfg.target.freedoms.amplitude_outside_roi = c->amp_outside_roi != 0;
        cfg.target.freedoms.phase = c->phase_freedom != 0;
        cfg.target.freedoms.scale = c->scale_freedom != 0;
        cfg.seed = c->seed;
        cfg.weight_clamp_lo = c->clamp_lo;
        cfg.weight_clamp_hi = c->clamp_hi;
        cfg.lt_initial_fraction = c->lt_initial_fraction;
        cfg.init_phase = c->init_phase == 1 ? InitPhase::Random
                         : c->init_phase == 2 ? InitPhase::Flat
                                              : InitPhase::Auto;
        std::unique_ptr<Propagator<float>> prop;
        if (c->fresnel) {
            FresnelParams p{c->wavelength, c->distance, c->pitch_x, c->pitch_y};
            prop = std::make_unique<Propagator<float>>(Propagator<float>::fresnel(nx, ny, p));
        }
        auto rep = run_ifta<float>(cfg, prop.get());
        size_t n = rep.hologram.data.size();
        if (hologram) std::memcpy(hologram, rep.hologram.data.data(), sizeof(float) * 2 * n);
        if (replay) std::memcpy(replay, rep.replay.data.data(), sizeof(float) * 2 * n);
        if (levels) {
            Quantiser<float> q(cfg.slm, nx, ny);
            for (size_t i = 0; i < n; ++i) levels[i] = q.decide(i, rep.hologram.data[i]);
        }
        if (trace)
            for (size_t k = 0; k < rep.trace.points.size(); ++k) trace[k] = rep.trace.points[k].second;
        if (timing) {  // RunReport::seconds and ::profile (report.hpp:38-65)
            timing[0] = rep.seconds;
            timing[1] = rep.profile.transform;
            timing[2] = rep.profile.constraint;
            timing[3] = rep.profile.metric;
            timing[4] = rep.profile.other;
        }
    });
}

// run_ifta<double> (ifta.hpp:86-235) — the oracle of the f64 device loop.
int hgr_ifta_run_d(const hgo_ifta_cfg* c, const hgo_slm* s, int nx, int ny, const double* amp,
                   const double* phase_turns, const uint8_t* roi, double* hologram, double* replay,
                   int32_t* levels, double* trace) {
    return guard([&] {
        IftaConfig cfg;
        cfg.variant = c->variant == 0   ? IftaVariant::GS
                      : c->variant == 1 ? IftaVariant::WeightedGS
                                        : IftaVariant::LiuTaghizadeh;
        cfg.iterations = c->iterations;
        cfg.slm = to_spec(s, nx, ny);
        cfg.target.amplitude = to_image(amp, nx, ny);
        if (phase_turns) cfg.target.phase = to_image(phase_turns, nx, ny);
        if (roi) {
            RegionMask m(nx, ny);
            std::memcpy(m.data.data(), roi, m.data.size());
            cfg.target.roi = m;
        }
        cfg.target.freedoms.amplitude_outside_roi = c->amp_outside_roi != 0;
        cfg.target.freedoms.phase = c->phase_freedom != 0;
        cfg.target.freedoms.scale = c->scale_freedom != 0;
        cfg.seed = c->seed;
        cfg.weight_clamp_lo = c->clamp_lo;
        cfg.weight_clamp_hi = c->clamp_hi;
        cfg.lt_initial_fraction = c->lt_initial_fraction;
        cfg.init_phase = c->init_phase == 1 ? InitPhase::Random
                         : c->init_phase == 2 ? InitPhase::Flat
                                              : InitPhase::Auto;
        std::unique_ptr<Propagator<double>> prop;
        if (c->fresnel) {
            FresnelParams p{c->wavelength, c->distance, c->pitch_x, c->pitch_y};
            prop = std::make_unique<Propagator<double>>(Propagator<double>::fresnel(nx, ny, p));
        }
        auto rep = run_ifta<double>(cfg, prop.get());
        size_t n = rep.hologram.data.size();
        if (hologram) std::memcpy(hologram, rep.hologram.data.data(), sizeof(double) * 2 * n);
        if (replay) std::memcpy(replay, rep.replay.data.data(), sizeof(double) * 2 * n);
        if (levels) {
            Quantiser<double> q(cfg.slm, nx, ny);
            for (size_t i = 0; i < n; ++i) levels[i] = q.decide(i, rep.hologram.data[i]);
        }
        if (trace)
            for (size_t k = 0; k < rep.trace.points.size(); ++k) trace[k] = rep.trace.points[k].second;
    });
}

// run_ospr_variant<double> (ospr.hpp:68-185).
int hgr_ospr_run_d(int adaptive, int subframes, uint64_t seed, double gain, const hgo_slm* s, int nx, int ny,
                   const double* target, const uint8_t* roi, int scale_free, int32_t* levels, double* frame_mse,
                   double* cum_mse, double* mean_intensity) {
    return guard([&] {
        OsprConfig cfg;
        cfg.variant = adaptive ? OsprVariant::AdaptiveOspr : OsprVariant::Ospr;
        cfg.subframes = subframes;
        cfg.slm = to_spec(s, nx, ny);
        cfg.target.amplitude = to_image(target, nx, ny);
        if (roi) {
            RegionMask m(nx, ny);
            std::memcpy(m.data.data(), roi, m.data.size());
            cfg.target.roi = m;
        }
        cfg.target.freedoms.scale = scale_free != 0;
        cfg.seed = seed;
        cfg.feedback_gain = gain;
        auto run = run_ospr_variant<double>(cfg);
        size_t n = static_cast<size_t>(nx) * ny;
        Quantiser<double> q(cfg.slm, nx, ny);
        for (int k = 0; k < subframes; ++k) {
            const auto& fr = run.set.frames[k];
            if (levels)
                for (size_t i = 0; i < n; ++i) levels[n * k + i] = q.decide(i, fr.data[i]);
            if (frame_mse) frame_mse[k] = run.set.per_frame_mse[k];
            if (cum_mse) cum_mse[k] = run.report.trace.points[k].second;
        }
        if (mean_intensity)
            std::memcpy(mean_intensity, run.set.mean_intensity.data.data(), sizeof(double) * n);
    });
}

// run_ospr_variant<float> (ospr.hpp:68-185).
int hgr_ospr_run(int adaptive, int subframes, uint64_t seed, double gain, const hgo_slm* s, int nx,
                 int ny, const double* target, const uint8_t* roi, int scale_free, int32_t* levels,
                 float* frames, double* frame_mse, double* cum_mse, double* mean_intensity,
                 float* replay, double* seconds) {
    return guard([&] {
        OsprConfig cfg;
        cfg.variant = adaptive ? OsprVariant::AdaptiveOspr : OsprVariant::Ospr;
        cfg.subframes = subframes;
        cfg.slm = to_spec(s, nx, ny);
        cfg.target.amplitude = to_image(target, nx, ny);
        if (roi) {
            RegionMask m(nx, ny);
            std::memcpy(m.data.data(), roi, m.data.size());
            cfg.target.roi = m;
        }
        cfg.target.freedoms.scale = scale_free != 0;
        cfg.seed = seed;
        cfg.feedback_gain = gain;
        auto run = run_ospr_variant<float>(cfg);
        size_t n = static_cast<size_t>(nx) * ny;
        Quantiser<float> q(cfg.slm, nx, ny);
        for (int k = 0; k < subframes; ++k) {
            const auto& fr = run.set.frames[k];
            if (frames) std::memcpy(frames + 2 * n * k, fr.data.data(), sizeof(float) * 2 * n);
            if (levels)
                for (size_t i = 0; i < n; ++i) levels[n * k + i] = q.decide(i, fr.data[i]);
            if (frame_mse) frame_mse[k] = run.set.per_frame_mse[k];
            if (cum_mse) cum_mse[k] = run.report.trace.points[k].second;
        }
        if (mean_intensity)
            std::memcpy(mean_intensity, run.set.mean_intensity.data.data(), sizeof(double) * n);
        if (replay) std::memcpy(replay, run.report.replay.data.data(), sizeof(float) * 2 * n);
        if (seconds) *seconds = run.report.seconds;
    });
}

double hgr_subframe_mse_statistic(const double* v, int n) {
    return subframe_mse_statistic(std::vector<double>(v, v + n));
}

}  // extern "C"
