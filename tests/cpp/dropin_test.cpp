// dropin_test.cpp — the C++ drop-in (include/hologen_b200/dropin.hpp) used
// exactly as a reference caller would: reference headers + explicit float
// specialisations + libhologen_b200.so.  Built by __graft_entry__.build()
// when /root/reference is present; run by tests/test_gpu_dropin.py.
//
// The reference's own loop (detail::run_ifta / run_ospr_impl) is run beside
// the GPU path with default_fft_backend<float>() = the B200 FftBackend, so
// both sides use the same transform and only the fused kernels differ.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <thread>
#include <utility>
#include <vector>

#include "hologen/ifta.hpp"
#include "hologen/ospr.hpp"
#include "hologen/patterns.hpp"
#include "hologen/rng.hpp"
#include "hologen_b200/dropin.hpp"

namespace hologen {
template <typename T>
FftBackend<T>& default_fft_backend();
template <>
FftBackend<float>& default_fft_backend<float>() { return hologen_b200::fft_backend(); }
template <>
FftBackend<double>& default_fft_backend<double>() { return hologen_b200::fft_backend_f64(); }
}  // namespace hologen

using namespace hologen;

static int fails = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("CHECK failed line %d: %s\n", __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

static int level_mismatch(const SlmSpec& slm, const ComplexField<float>& a, const ComplexField<float>& b) {
    Quantiser<float> q(slm, a.nx, a.ny);
    int m = 0;
    for (size_t i = 0; i < a.data.size(); ++i) m += q.decide(i, a.data[i]) != q.decide(i, b.data[i]);
    return m;
}

int main() {
    RealImage amp = patterns::smooth_blobs(128, 128);
    normalize_image(amp, Normalization::UnitEnergy);

    // GS binary, Fourier
    IftaConfig cfg;
    cfg.iterations = 20;
    cfg.slm = SlmSpec::binary_phase();
    cfg.target.amplitude = amp;
    cfg.seed = 1;
    auto gpu = run_gs<float>(cfg);                    // drop-in specialisation
    auto ref = detail::run_ifta<float>(cfg, nullptr);  // the reference loop
    int mm = level_mismatch(cfg.slm, gpu.hologram, ref.hologram);
    double rel = std::abs(gpu.final_error - ref.final_error) / ref.final_error;
    std::printf("gs binary 128^2: level mismatches %d, mse %.9g vs %.9g (rel %.2e)\n", mm, gpu.final_error,
                ref.final_error, rel);
    CHECK(mm <= 4 && rel < 1e-4 && gpu.trace.size() == 20 && gpu.algorithm == "gs");
    // RunReport::profile: every phase attributed, the total is the run
    // (test_ifta.cpp:270-280 "profile accounts for the whole run"; bench.cpp:167-183)
    auto profile_ok = [](const auto& r) {
        const auto& q = r.profile;
        std::printf("  profile transform %.3g constraint %.3g metric %.3g other %.3g of %.3g s\n", q.transform,
                    q.constraint, q.metric, q.other, r.seconds);
        return q.transform > 0.0 && q.constraint > 0.0 && q.metric > 0.0 && q.other >= 0.0 && r.seconds > 0.0 &&
               std::abs(q.total() - r.seconds) <= 1e-9 * r.seconds;
    };
    CHECK(profile_ok(gpu));

    // WGS 256-level with a Fresnel propagator (lock-step not needed at 3 iterations)
    FresnelParams p{532e-9, 0.1, 8e-6, 8e-6};
    auto prop = Propagator<float>::fresnel(128, 128, p);
    IftaConfig w = cfg;
    w.variant = IftaVariant::WeightedGS;
    w.slm = SlmSpec::full_circle_phase(256);
    w.iterations = 2;
    auto gw = run_weighted_gs<float>(w, &prop);
    auto rw = detail::run_ifta<float>(w, &prop);
    rel = std::abs(gw.final_error - rw.final_error) / rw.final_error;
    std::printf("wgs fresnel 256-level: mse %.9g vs %.9g (rel %.2e)\n", gw.final_error, rw.final_error, rel);
    CHECK(rel < 1e-4 && gw.algorithm == "wgs");

    // OSPR
    OsprConfig o;
    o.subframes = 6;
    o.slm = SlmSpec::binary_phase();
    o.target.amplitude = amp;
    o.seed = 42;
    auto go = run_ospr<float>(o);
    auto ro = detail::run_ospr_impl<float>(o, nullptr);
    int om = 0;
    for (int k = 0; k < 6; ++k) om += level_mismatch(o.slm, go.set.frames[k], ro.set.frames[k]);
    rel = std::abs(go.report.final_error - ro.report.final_error) / ro.report.final_error;
    std::printf("ospr 6 frames: level mismatches %d, cumulative mse rel %.2e\n", om, rel);
    CHECK(om <= 6 && rel < 1e-4 && go.report.algorithm == "ospr" && go.set.frames.size() == 6);
    CHECK(profile_ok(go.report));

    // T = double: the GPU f64 loop against the reference's own double loop
    // (detail::run_ifta<double>, its transforms on the GPU f64 FftBackend)
    {
        IftaConfig d = cfg;
        d.iterations = 10;
        auto gd = run_gs<double>(d);
        auto rd = detail::run_ifta<double>(d, nullptr);
        int m = 0;
        Quantiser<double> qd(d.slm, 128, 128);
        for (size_t i = 0; i < gd.hologram.data.size(); ++i)
            m += qd.decide(i, gd.hologram.data[i]) != qd.decide(i, rd.hologram.data[i]);
        double rel64 = std::abs(gd.final_error - rd.final_error) / rd.final_error;
        std::printf("gs<double> binary 128^2: level mismatches %d, mse rel %.2e\n", m, rel64);
        CHECK(m == 0 && rel64 < 1e-9);
        CHECK(profile_ok(gd));
        auto p64 = Propagator<double>::fresnel(128, 128, p);
        IftaConfig wd = w;
        wd.iterations = 2;
        auto gw64 = run_weighted_gs<double>(wd, &p64);
        auto rw64 = detail::run_ifta<double>(wd, &p64);
        rel64 = std::abs(gw64.final_error - rw64.final_error) / rw64.final_error;
        std::printf("wgs<double> fresnel 256-level: mse rel %.2e\n", rel64);
        CHECK(rel64 < 1e-9);
        auto go64 = run_ospr<double>(o);
        auto ro64 = detail::run_ospr_impl<double>(o, nullptr);
        rel64 = std::abs(go64.report.final_error - ro64.report.final_error) / ro64.report.final_error;
        std::printf("ospr<double> 6 frames: cumulative mse rel %.2e\n", rel64);
        CHECK(rel64 < 1e-9 && go64.set.frames.size() == 6);
        CHECK(profile_ok(go64.report));
    }

    // the runner's batch pool (runner.cpp:387-421): one job per host thread,
    // threads routed round-robin over the GPUs; results equal the sequential runs
    hologen_b200::route_threads_over_devices();
    std::vector<RunReport<float>> seq, par(4);
    for (int s = 0; s < 4; ++s) {
        IftaConfig c = cfg;
        c.seed = 10 + s;
        c.iterations = 5;
        seq.push_back(run_gs<float>(c));
    }
    std::vector<std::thread> pool;
    for (int s = 0; s < 4; ++s)
        pool.emplace_back([&, s] {
            IftaConfig c = cfg;
            c.seed = 10 + s;
            c.iterations = 5;
            par[s] = run_gs<float>(c);
        });
    for (auto& t : pool) t.join();
    bool same = true;
    for (int s = 0; s < 4; ++s) same = same && par[s].hologram.data == seq[s].hologram.data && par[s].final_error == seq[s].final_error;
    std::printf("batch pool of 4 threads: %s\n", same ? "identical to sequential" : "DIFFERENT");
    CHECK(same);

    // FftBackend<double> on the GPU vs the reference's NaiveDftBackend (test_fft.cpp:90-98, 1e-10)
    {
        Rng r(3);
        ComplexField<double> f(32, 16, Domain::Aperture);
        for (auto& z : f.data) z = {r.uniform(-1.0, 1.0), r.uniform(-1.0, 1.0)};
        NaiveDftBackend<double> naive;
        auto g = fft_forward(f);  // default_fft_backend<double>() = B200FftBackendF64
        auto n = fft_forward(f, &naive);
        double err = 0.0;
        for (size_t i = 0; i < g.data.size(); ++i) err = std::max(err, std::abs(g.data[i] - n.data[i]));
        auto back = fft_inverse(g);
        double rt = 0.0;
        for (size_t i = 0; i < f.data.size(); ++i) rt = std::max(rt, std::abs(back.data[i] - f.data[i]));
        std::printf("fft<double> 32x16 vs naive DFT: max err %.2e, round trip %.2e\n", err, rt);
        CHECK(err < 1e-10 && rt < 1e-12);
        // any size (test_fft.cpp:90-98: 5x7 and 16x3 against the naive DFT at 1e-10)
        for (auto [w, h] : {std::pair{5, 7}, std::pair{16, 3}}) {
            ComplexField<double> g2(w, h, Domain::Aperture);
            for (auto& z : g2.data) z = {r.uniform(-1.0, 1.0), r.uniform(-1.0, 1.0)};
            auto a = fft_forward(g2), bnv = fft_forward(g2, &naive);
            double e2 = 0.0;
            for (size_t i = 0; i < a.data.size(); ++i) e2 = std::max(e2, std::abs(a.data[i] - bnv.data[i]));
            std::printf("fft<double> %dx%d vs naive DFT: max err %.2e\n", w, h, e2);
            CHECK(e2 < 1e-10);
        }
    }

    // errors keep the reference's exceptions and messages
    IftaConfig bad = cfg;
    bad.iterations = 0;
    try {
        (void)run_gs<float>(bad);
        CHECK(false);
    } catch (const std::invalid_argument& e) {
        CHECK(std::string(e.what()) == "IftaConfig: iterations must be >= 1");
    }
    try {
        (void)run_weighted_gs<float>(cfg);
        CHECK(false);
    } catch (const std::invalid_argument& e) {
        CHECK(std::string(e.what()) == "run_weighted_gs: config variant mismatch");
    }
    std::printf(fails ? "DROPIN FAILED\n" : "DROPIN OK\n");
    return fails ? 1 : 0;
}
