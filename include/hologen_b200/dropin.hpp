// hologen_b200/dropin.hpp — C++ drop-in for the reference's float entry points.
//
// Include this header after the reference's own headers (proj/include) in
// every translation unit that calls the algorithms, and link
// libhologen_b200.so.  It adds explicit specialisations, for T = float, of
//
//   hologen::run_gs / run_weighted_gs / run_liu_taghizadeh / run_ifta
//                                                     (ifta.hpp:239-263)
//   hologen::run_ospr / run_adaptive_ospr / run_ospr_variant (ospr.hpp:168-185)
//
// so existing callers (runner.cpp:152-224, bench.cpp:111-184, tests) run the
// sm_100a path unchanged.  The value types are the reference's own
// (IftaConfig, OsprConfig, SlmSpec, TargetSpec, Propagator, RunReport,
// OsprRun); validation is the reference's own cfg.validate() (ifta.hpp:88,
// ospr.hpp:70), so errors and messages are identical.  The T = double
// instantiations stay the reference templates.  A Fresnel Propagator<float>
// is honoured by handing its quadratic phase (aperture_factor,
// propagation.hpp:100-103) to the GPU, so Q is bit-identical.
//
// Also provides hologen_b200::B200FftBackend / B200FftBackendF64,
// FftBackend<float> / FftBackend<double> (fft.hpp:17-27) on the GPU
// transforms, for default_fft_backend<T>().
#pragma once

#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hologen/fft.hpp"
#include "hologen/ifta.hpp"
#include "hologen/ospr.hpp"
#include "hologen_b200.h"

namespace hologen_b200 {

inline void throw_status(int rc) {
    if (rc == HGC_OK) return;
    std::string msg = hgc_last_error();
    if (rc == HGC_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline hgc_slm to_c(const hologen::SlmSpec& s) {
    hgc_slm c{};
    c.mode = s.mode == hologen::SlmMode::Phase ? 1 : 0;
    c.levels = s.levels;
    c.min_arg = s.min_arg;
    c.max_arg = s.max_arg;
    c.full_circle = s.full_circle ? 1 : 0;
    c.min_amp = s.min_amp;
    c.max_amp = s.max_amp;
    c.illumination = s.illumination ? reinterpret_cast<const double*>(s.illumination->data.data()) : nullptr;
    return c;
}

// FftBackend<float> on the B200 transform (host pointers in and out).
class B200FftBackend : public hologen::FftBackend<float> {
public:
    const char* name() const override { return "b200"; }
    void forward(int nx, int ny, const std::complex<float>* in, std::complex<float>* out) override {
        throw_status(hgc_fft2d(nx, ny, -1, 1, reinterpret_cast<const float*>(in), reinterpret_cast<float*>(out)));
    }
    void inverse(int nx, int ny, const std::complex<float>* in, std::complex<float>* out) override {
        throw_status(hgc_fft2d(nx, ny, +1, 1, reinterpret_cast<const float*>(in), reinterpret_cast<float*>(out)));
    }
};

// Route the calling threads round-robin over the GPUs (the runner's batch
// pool runs one job per thread, runner.cpp:387-421): call once at start-up.
inline void route_threads_over_devices() { throw_status(hgc_set_device_policy(1)); }

inline B200FftBackend& fft_backend() {
    static B200FftBackend b;
    return b;
}

// FftBackend<double> on the GPU's double-precision transform (hgc_fft2d_f64),
// for default_fft_backend<double>() / the T = double templates.
class B200FftBackendF64 : public hologen::FftBackend<double> {
public:
    const char* name() const override { return "b200-f64"; }
    void forward(int nx, int ny, const std::complex<double>* in, std::complex<double>* out) override {
        throw_status(
            hgc_fft2d_f64(nx, ny, -1, 1, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out)));
    }
    void inverse(int nx, int ny, const std::complex<double>* in, std::complex<double>* out) override {
        throw_status(
            hgc_fft2d_f64(nx, ny, +1, 1, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out)));
    }
};

inline B200FftBackendF64& fft_backend_f64() {
    static B200FftBackendF64 b;
    return b;
}

// RunReport::profile from the library's per-phase device times (hgc_*_io
// profile: transform, constraint, metric); "other" is the rest of the
// call as this wrapper timed it, so total() == seconds as in ifta.hpp:231-233.
template <class Rep>
inline void set_profile(Rep& rep, const double (&p)[4]) {
    rep.profile.transform = p[0];
    rep.profile.constraint = p[1];
    rep.profile.metric = p[2];
    rep.profile.other = std::max(0.0, rep.seconds - (p[0] + p[1] + p[2]));
}

// run_ifta<float> on the GPU (ifta.hpp:86-235 semantics).
inline hologen::RunReport<float> run_ifta_gpu(const hologen::IftaConfig& cfg, const hologen::Propagator<float>* prop) {
    auto t0 = std::chrono::steady_clock::now();
    cfg.validate();  // the reference's own validation (ifta.hpp:88)
    const auto& tgt = cfg.target;
    const int nx = tgt.width(), ny = tgt.height();
    const size_t n = static_cast<size_t>(nx) * ny;
    hgc_ifta_cfg c{};
    c.variant = static_cast<int>(cfg.variant);
    c.iterations = cfg.iterations;
    c.seed = cfg.seed;
    c.weight_clamp_lo = cfg.weight_clamp_lo;
    c.weight_clamp_hi = cfg.weight_clamp_hi;
    c.lt_initial_fraction = cfg.lt_initial_fraction;
    c.init_phase = static_cast<int>(cfg.init_phase);
    c.freedom_amplitude_outside_roi = tgt.freedoms.amplitude_outside_roi;
    c.freedom_phase = tgt.freedoms.phase;
    c.freedom_scale = tgt.freedoms.scale;
    hgc_slm s = to_c(cfg.slm);
    std::vector<std::complex<float>> q;
    if (prop && prop->is_fresnel()) {  // Q exactly as the reference computed it
        q.resize(n);
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) q[static_cast<size_t>(y) * nx + x] = prop->aperture_factor(x, y);
    }
    hologen::RunReport<float> rep;
    rep.seed = cfg.seed;
    rep.algorithm = cfg.variant == hologen::IftaVariant::GS           ? "gs"
                    : cfg.variant == hologen::IftaVariant::WeightedGS ? "wgs"
                                                                      : "lt";
    rep.hologram = hologen::ComplexField<float>(nx, ny, hologen::Domain::Aperture);
    rep.replay = hologen::ComplexField<float>(nx, ny, hologen::Domain::Replay);
    std::vector<double> trace(cfg.iterations);
    hgc_ifta_io io{};
    io.amplitude = tgt.amplitude.data.data();
    io.phase = tgt.phase ? tgt.phase->data.data() : nullptr;
    io.roi = tgt.roi ? tgt.roi->data.data() : nullptr;
    io.hologram = reinterpret_cast<float*>(rep.hologram.data.data());
    io.replay = reinterpret_cast<float*>(rep.replay.data.data());
    io.trace = trace.data();
    io.fresnel_q = q.empty() ? nullptr : reinterpret_cast<const float*>(q.data());
    double prof[4] = {0, 0, 0, 0};
    io.profile = prof;
    throw_status(hgc_ifta_run(&c, &s, nullptr, nx, ny, 1, &io));
    rep.trace.name = "mse";
    for (int k = 0; k < cfg.iterations; ++k) rep.trace.append(k + 1, trace[k]);
    rep.final_error = trace.back();
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    set_profile(rep, prof);  // fused passes: per-pass device time split by phase
    return rep;
}

// run_ospr_impl<float> on the GPU (ospr.hpp:68-164 semantics).
inline hologen::OsprRun<float> run_ospr_gpu(const hologen::OsprConfig& cfg, hologen::FftBackend<float>* backend) {
    if (backend && backend != &fft_backend())
        throw std::runtime_error("hologen_b200: OSPR with a caller-supplied FftBackend is not on the GPU path");
    auto t0 = std::chrono::steady_clock::now();
    cfg.validate();  // ospr.hpp:70
    const auto& tgt = cfg.target;
    const int nx = tgt.width(), ny = tgt.height(), N = cfg.subframes;
    const size_t n = static_cast<size_t>(nx) * ny;
    hgc_ospr_cfg c{};
    c.variant = static_cast<int>(cfg.variant);
    c.subframes = N;
    c.seed = cfg.seed;
    c.feedback_gain = cfg.feedback_gain;
    c.freedom_scale = tgt.freedoms.scale;
    hgc_slm s = to_c(cfg.slm);
    std::vector<std::complex<float>> frames(n * N);
    std::vector<double> fm(N), cm(N), mi(n);
    hologen::OsprRun<float> run;
    hologen::RunReport<float>& rep = run.report;
    rep.replay = hologen::ComplexField<float>(nx, ny, hologen::Domain::Replay);
    hgc_ospr_io io{};
    io.amplitude = tgt.amplitude.data.data();
    io.roi = tgt.roi ? tgt.roi->data.data() : nullptr;
    io.frames = reinterpret_cast<float*>(frames.data());
    io.frame_mse = fm.data();
    io.cumulative_mse = cm.data();
    io.mean_intensity = mi.data();
    io.replay = reinterpret_cast<float*>(rep.replay.data.data());
    double prof[4] = {0, 0, 0, 0};
    io.profile = prof;
    throw_status(hgc_ospr_run(&c, &s, nx, ny, 1, &io));
    const bool adaptive = cfg.variant == hologen::OsprVariant::AdaptiveOspr;
    rep.algorithm = adaptive ? "adaptive_ospr" : "ospr";
    rep.seed = cfg.seed;
    rep.trace.name = "cumulative_mse";
    hologen::MetricTrace frame_trace;
    frame_trace.name = "frame_mse";
    for (int k = 0; k < N; ++k) {
        hologen::ComplexField<float> f(nx, ny, hologen::Domain::Aperture);
        std::memcpy(f.data.data(), frames.data() + n * k, sizeof(std::complex<float>) * n);
        run.set.frames.push_back(std::move(f));
        run.set.per_frame_mse.push_back(fm[k]);
        frame_trace.append(k + 1, fm[k]);
        rep.trace.append(k + 1, cm[k]);
    }
    run.set.mean_intensity = hologen::RealImage(nx, ny);
    run.set.mean_intensity.data = mi;
    rep.hologram = run.set.frames.back();
    rep.final_error = cm.back();
    rep.evaluations = N;
    rep.extra_traces.push_back(std::move(frame_trace));
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    set_profile(rep, prof);
    return run;
}

// run_ifta<double> on the GPU f64 loop (hgc_ifta_run_f64, ifta.hpp:86-235 in double).
inline hologen::RunReport<double> run_ifta_gpu64(const hologen::IftaConfig& cfg,
                                                 const hologen::Propagator<double>* prop) {
    auto t0 = std::chrono::steady_clock::now();
    cfg.validate();
    const auto& tgt = cfg.target;
    const int nx = tgt.width(), ny = tgt.height();
    hgc_ifta_cfg c{};
    c.variant = static_cast<int>(cfg.variant);
    c.iterations = cfg.iterations;
    c.seed = cfg.seed;
    c.weight_clamp_lo = cfg.weight_clamp_lo;
    c.weight_clamp_hi = cfg.weight_clamp_hi;
    c.lt_initial_fraction = cfg.lt_initial_fraction;
    c.init_phase = static_cast<int>(cfg.init_phase);
    c.freedom_amplitude_outside_roi = tgt.freedoms.amplitude_outside_roi;
    c.freedom_phase = tgt.freedoms.phase;
    c.freedom_scale = tgt.freedoms.scale;
    hgc_slm s = to_c(cfg.slm);
    std::vector<std::complex<double>> q;
    if (prop && prop->is_fresnel()) {  // the Propagator's own Q (propagation.hpp:100-103)
        q.resize(static_cast<size_t>(nx) * ny);
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) q[static_cast<size_t>(y) * nx + x] = prop->aperture_factor(x, y);
    }
    hologen::RunReport<double> rep;
    rep.seed = cfg.seed;
    rep.algorithm = cfg.variant == hologen::IftaVariant::GS           ? "gs"
                    : cfg.variant == hologen::IftaVariant::WeightedGS ? "wgs"
                                                                      : "lt";
    rep.hologram = hologen::ComplexField<double>(nx, ny, hologen::Domain::Aperture);
    rep.replay = hologen::ComplexField<double>(nx, ny, hologen::Domain::Replay);
    std::vector<double> trace(cfg.iterations);
    hgc_ifta_io64 io{};
    io.amplitude = tgt.amplitude.data.data();
    io.phase = tgt.phase ? tgt.phase->data.data() : nullptr;
    io.roi = tgt.roi ? tgt.roi->data.data() : nullptr;
    io.hologram = reinterpret_cast<double*>(rep.hologram.data.data());
    io.replay = reinterpret_cast<double*>(rep.replay.data.data());
    io.trace = trace.data();
    io.fresnel_q = q.empty() ? nullptr : reinterpret_cast<const double*>(q.data());
    double prof[4] = {0, 0, 0, 0};
    io.profile = prof;
    throw_status(hgc_ifta_run_f64(&c, &s, nullptr, nx, ny, &io));
    rep.trace.name = "mse";
    for (int k = 0; k < cfg.iterations; ++k) rep.trace.append(k + 1, trace[k]);
    rep.final_error = trace.back();
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    set_profile(rep, prof);
    return rep;
}

// run_ospr_impl<double> on the GPU f64 loop (hgc_ospr_run_f64).
inline hologen::OsprRun<double> run_ospr_gpu64(const hologen::OsprConfig& cfg, hologen::FftBackend<double>* backend) {
    if (backend && backend != &fft_backend_f64())
        throw std::runtime_error("hologen_b200: OSPR with a caller-supplied FftBackend is not on the GPU path");
    auto t0 = std::chrono::steady_clock::now();
    cfg.validate();
    const auto& tgt = cfg.target;
    const int nx = tgt.width(), ny = tgt.height(), N = cfg.subframes;
    const size_t n = static_cast<size_t>(nx) * ny;
    hgc_ospr_cfg c{};
    c.variant = static_cast<int>(cfg.variant);
    c.subframes = N;
    c.seed = cfg.seed;
    c.feedback_gain = cfg.feedback_gain;
    c.freedom_scale = tgt.freedoms.scale;
    hgc_slm s = to_c(cfg.slm);
    std::vector<std::complex<double>> frames(n * N);
    std::vector<double> fm(N), cm(N), mi(n);
    hologen::OsprRun<double> run;
    hologen::RunReport<double>& rep = run.report;
    rep.replay = hologen::ComplexField<double>(nx, ny, hologen::Domain::Replay);
    hgc_ospr_io64 io{};
    io.amplitude = tgt.amplitude.data.data();
    io.roi = tgt.roi ? tgt.roi->data.data() : nullptr;
    io.frames = reinterpret_cast<double*>(frames.data());
    io.frame_mse = fm.data();
    io.cumulative_mse = cm.data();
    io.mean_intensity = mi.data();
    io.replay = reinterpret_cast<double*>(rep.replay.data.data());
    double prof[4] = {0, 0, 0, 0};
    io.profile = prof;
    throw_status(hgc_ospr_run_f64(&c, &s, nx, ny, &io));
    rep.algorithm = cfg.variant == hologen::OsprVariant::AdaptiveOspr ? "adaptive_ospr" : "ospr";
    rep.seed = cfg.seed;
    rep.trace.name = "cumulative_mse";
    hologen::MetricTrace frame_trace;
    frame_trace.name = "frame_mse";
    for (int k = 0; k < N; ++k) {
        hologen::ComplexField<double> f(nx, ny, hologen::Domain::Aperture);
        std::memcpy(f.data.data(), frames.data() + n * k, sizeof(std::complex<double>) * n);
        run.set.frames.push_back(std::move(f));
        run.set.per_frame_mse.push_back(fm[k]);
        frame_trace.append(k + 1, fm[k]);
        rep.trace.append(k + 1, cm[k]);
    }
    run.set.mean_intensity = hologen::RealImage(nx, ny);
    run.set.mean_intensity.data = mi;
    rep.hologram = run.set.frames.back();
    rep.final_error = cm.back();
    rep.evaluations = N;
    rep.extra_traces.push_back(std::move(frame_trace));
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    set_profile(rep, prof);
    return run;
}

}  // namespace hologen_b200

namespace hologen {

template <>
inline RunReport<float> run_gs<float>(const IftaConfig& cfg, const Propagator<float>* prop) {
    if (cfg.variant != IftaVariant::GS) throw std::invalid_argument("run_gs: config variant mismatch");
    return hologen_b200::run_ifta_gpu(cfg, prop);
}
template <>
inline RunReport<float> run_weighted_gs<float>(const IftaConfig& cfg, const Propagator<float>* prop) {
    if (cfg.variant != IftaVariant::WeightedGS) throw std::invalid_argument("run_weighted_gs: config variant mismatch");
    return hologen_b200::run_ifta_gpu(cfg, prop);
}
template <>
inline RunReport<float> run_liu_taghizadeh<float>(const IftaConfig& cfg, const Propagator<float>* prop) {
    if (cfg.variant != IftaVariant::LiuTaghizadeh)
        throw std::invalid_argument("run_liu_taghizadeh: config variant mismatch");
    return hologen_b200::run_ifta_gpu(cfg, prop);
}
template <>
inline RunReport<float> run_ifta<float>(const IftaConfig& cfg, const Propagator<float>* prop) {
    return hologen_b200::run_ifta_gpu(cfg, prop);
}
template <>
inline OsprRun<float> run_ospr<float>(const OsprConfig& cfg, FftBackend<float>* backend) {
    if (cfg.variant != OsprVariant::Ospr) throw std::invalid_argument("run_ospr: config variant mismatch");
    return hologen_b200::run_ospr_gpu(cfg, backend);
}
template <>
inline OsprRun<float> run_adaptive_ospr<float>(const OsprConfig& cfg, FftBackend<float>* backend) {
    if (cfg.variant != OsprVariant::AdaptiveOspr)
        throw std::invalid_argument("run_adaptive_ospr: config variant mismatch");
    return hologen_b200::run_ospr_gpu(cfg, backend);
}
template <>
inline OsprRun<float> run_ospr_variant<float>(const OsprConfig& cfg, FftBackend<float>* backend) {
    return hologen_b200::run_ospr_gpu(cfg, backend);
}

// T = double: the GPU f64 loops.
template <>
inline RunReport<double> run_gs<double>(const IftaConfig& cfg, const Propagator<double>* prop) {
    if (cfg.variant != IftaVariant::GS) throw std::invalid_argument("run_gs: config variant mismatch");
    return hologen_b200::run_ifta_gpu64(cfg, prop);
}
template <>
inline RunReport<double> run_weighted_gs<double>(const IftaConfig& cfg, const Propagator<double>* prop) {
    if (cfg.variant != IftaVariant::WeightedGS) throw std::invalid_argument("run_weighted_gs: config variant mismatch");
    return hologen_b200::run_ifta_gpu64(cfg, prop);
}
template <>
inline RunReport<double> run_liu_taghizadeh<double>(const IftaConfig& cfg, const Propagator<double>* prop) {
    if (cfg.variant != IftaVariant::LiuTaghizadeh)
        throw std::invalid_argument("run_liu_taghizadeh: config variant mismatch");
    return hologen_b200::run_ifta_gpu64(cfg, prop);
}
template <>
inline RunReport<double> run_ifta<double>(const IftaConfig& cfg, const Propagator<double>* prop) {
    return hologen_b200::run_ifta_gpu64(cfg, prop);
}
template <>
inline OsprRun<double> run_ospr<double>(const OsprConfig& cfg, FftBackend<double>* backend) {
    if (cfg.variant != OsprVariant::Ospr) throw std::invalid_argument("run_ospr: config variant mismatch");
    return hologen_b200::run_ospr_gpu64(cfg, backend);
}
template <>
inline OsprRun<double> run_adaptive_ospr<double>(const OsprConfig& cfg, FftBackend<double>* backend) {
    if (cfg.variant != OsprVariant::AdaptiveOspr)
        throw std::invalid_argument("run_adaptive_ospr: config variant mismatch");
    return hologen_b200::run_ospr_gpu64(cfg, backend);
}
template <>
inline OsprRun<double> run_ospr_variant<double>(const OsprConfig& cfg, FftBackend<double>* backend) {
    return hologen_b200::run_ospr_gpu64(cfg, backend);
}

}  // namespace hologen
