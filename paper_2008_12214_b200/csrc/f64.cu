// f64.cu — run_ifta<double> / run_ospr_variant<double> on the device
// (SURVEY §8 f4): the reference's double arithmetic per pixel, double
// transforms of any size, the same seed stream (hgc_ifta_run_f64,
// hgc_ospr_run_f64).
#include "capi_impl.cuh"

extern "C" {

struct Dev64 {  // device quantiser tables in double (Quantiser<double> constructor, quantise.hpp:139-170)
    Q64 q{};
    DBuf<double2> states, illum, illum_unit;
    DBuf<double> illum_arg;
    void build(const hgc_slm* s, size_t npix) {
        const int L = s->levels;
        const double spac = s->mode == 1 ? (s->full_circle ? kTwoPi / L : (s->max_arg - s->min_arg) / (L - 1))
                                         : (s->max_amp - s->min_amp) / (L - 1);
        std::vector<double2> st(L);
        for (int k = 0; k < L; ++k) {
            if (s->mode == 1) {
                const double a = s->min_arg + k * spac;
                st[k] = make_double2(std::cos(a), std::sin(a));
            } else {
                st[k] = make_double2(s->min_amp + k * spac, 0.0);
            }
        }
        states.alloc(L);
        CK(cudaMemcpy(states.p, st.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
        q.mode = s->mode;
        q.L = L;
        q.full_circle = s->full_circle ? 1 : 0;
        q.min_arg = s->min_arg;
        q.inv_spac = 1.0 / spac;
        q.range = s->mode == 1 ? s->max_arg - s->min_arg : 0.0;
        q.min_amp = s->min_amp;
        q.states = states.p;
        if (s->illumination) {
            std::vector<double> arg(npix);
            std::vector<double2> il(npix), iu(npix);
            for (size_t i = 0; i < npix; ++i) {
                const double re = s->illumination[2 * i], im = s->illumination[2 * i + 1];
                const double a = std::hypot(re, im);  // std::abs(complex<double>)
                arg[i] = std::atan2(im, re);
                il[i] = make_double2(re, im);
                iu[i] = make_double2(re / a, im / a);
            }
            if (s->mode == 1) {
                illum_arg.alloc(npix);
                illum.alloc(npix);
                CK(cudaMemcpy(illum_arg.p, arg.data(), sizeof(double) * npix, cudaMemcpyHostToDevice));
                CK(cudaMemcpy(illum.p, il.data(), sizeof(double2) * npix, cudaMemcpyHostToDevice));
                q.illum_arg = illum_arg.p;
                q.illum = illum.p;
            } else {
                illum_unit.alloc(npix);
                CK(cudaMemcpy(illum_unit.p, iu.data(), sizeof(double2) * npix, cudaMemcpyHostToDevice));
                q.illum_unit = illum_unit.p;
            }
        }
    }
};

// mse of `mag` against T into *out (device), two deterministic passes
static void mse64(const double* T, Mag64 mag, const uint8_t* mask, size_t n, size_t M, int scale_free, DBuf<double>& part,
                  DBuf<double>& g, double* out, cudaStream_t st) {
    const int nblk = (int)std::min<size_t>(148 * 2, (n + 255) / 256);
    if (part.n < (size_t)2 * nblk) part.alloc(2 * nblk);
    if (!g.p) g.alloc(1);
    k_mse64_gain<<<nblk, 256, 0, st>>>(T, mag, mask, n, part.p);
    k_mse64_g<<<1, 32, 0, st>>>(part.p, nblk, scale_free, g.p);
    k_mse64_sum<<<nblk, 256, 0, st>>>(T, mag, mask, n, g.p, part.p);
    k_mse64_final<<<1, 32, 0, st>>>(part.p, nblk, (double)M, out);
    CK(cudaGetLastError());
}

static void propagate64(DBuf<double2>& f, const DBuf<double2>& Q, int nx, int ny, int sign, cudaStream_t st) {
    const size_t n = (size_t)nx * ny;
    if (sign < 0 && Q.p) k_mulq64<<<ew_grid(n), 256, 0, st>>>(f.p, Q.p, n, 0);  // FFT(f * Q)
    fft2d_any_f64(f.p, nx, ny, sign, 1, st);
    if (sign > 0 && Q.p) k_mulq64<<<ew_grid(n), 256, 0, st>>>(f.p, Q.p, n, 1);  // IFFT(F) * conj(Q)
    CK(cudaGetLastError());
}

static void fresnel_q64(const hgc_fresnel* p, int nx, int ny, DBuf<double2>& Q) {  // propagation.hpp:36-54
    std::vector<double2> q((size_t)nx * ny);
    const double pi = 3.1415926535897932384626433832795;
    const double cx = nx / 2.0, cy = ny / 2.0, scale = pi / (p->wavelength * p->distance);
    for (int y = 0; y < ny; ++y) {
        const double dy = (y - cy) * p->pixel_pitch_y, ty = dy * dy;
        for (int x = 0; x < nx; ++x) {
            const double dx = (x - cx) * p->pixel_pitch_x, ph = scale * (dx * dx + ty);
            q[(size_t)y * nx + x] = make_double2(std::cos(ph), std::sin(ph));
        }
    }
    Q.alloc(q.size());
    CK(cudaMemcpy(Q.p, q.data(), sizeof(double2) * q.size(), cudaMemcpyHostToDevice));
}

int hgc_ifta_run_f64(const hgc_ifta_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny,
                     hgc_ifta_io64* io) {
    const auto t0 = std::chrono::steady_clock::now();
    return guarded([&] {
        validate_ifta_cfg(cfg);
        if (!io || !io->amplitude) invalid("TargetSpec: amplitude image is empty");
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        const size_t n = (size_t)nx * ny;
        validate_slm(slm, n);
        if (fresnel) validate_fresnel(fresnel);
        for (size_t i = 0; i < n; ++i) {  // TargetSpec::validate, target.hpp:52-73
            if (!std::isfinite(io->amplitude[i])) invalid("TargetSpec.amplitude: image contains non-finite values");
            if (io->amplitude[i] < 0) invalid("TargetSpec: amplitude must be non-negative");
            if (io->phase && !std::isfinite(io->phase[i])) invalid("TargetSpec.phase: image contains non-finite values");
        }
        const size_t M = roi_count(io->roi, n);
        if (cfg->init_phase == 3 && !io->init_field) invalid("IftaConfig: init_phase Given requires init_field");
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        Dev64 q;
        q.build(slm, n);
        DBuf<double2> R, f, Q, tcs;
        DBuf<double> amp, w, part, g, trace;
        DBuf<uint8_t> roi;
        DBuf<int32_t> lv;
        R.alloc(n);
        f.alloc(n);
        amp.alloc(n);
        trace.alloc(cfg->iterations);
        CK(cudaMemcpy(amp.p, io->amplitude, sizeof(double) * n, cudaMemcpyHostToDevice));
        if (io->roi) {
            roi.alloc(n);
            CK(cudaMemcpy(roi.p, io->roi, n, cudaMemcpyHostToDevice));
        }
        if (io->fresnel_q) {  // caller-supplied Q (e.g. a reference Propagator<double>)
            Q.alloc(n);
            CK(cudaMemcpy(Q.p, io->fresnel_q, sizeof(double2) * n, cudaMemcpyHostToDevice));
        } else if (fresnel) {
            fresnel_q64(fresnel, nx, ny, Q);
        }
        // target phase as (cos, sin) with the host libm, ifta.hpp:131-136 / :215-219
        const bool tphase_used = !cfg->freedom_phase || (cfg->init_phase == 0 && io->phase);
        std::vector<double2> h_tcs;
        if (io->phase && tphase_used) {
            h_tcs.resize(n);
            for (size_t i = 0; i < n; ++i) {
                const double ph = kTwoPi * io->phase[i];
                h_tcs[i] = make_double2(std::cos(ph), std::sin(ph));
            }
            tcs.alloc(n);
            CK(cudaMemcpy(tcs.p, h_tcs.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
        }
        // ---- R0, ifta.hpp:124-139
        const bool target_phase_init = cfg->init_phase == 0 && io->phase && !cfg->freedom_phase;
        if (cfg->init_phase == 3) {
            CK(cudaMemcpy(R.p, io->init_field, sizeof(double2) * n, cudaMemcpyHostToDevice));
        } else if (cfg->init_phase == 2 || target_phase_init) {
            std::vector<double2> r0(n);
            for (size_t i = 0; i < n; ++i) {
                const double a = io->amplitude[i];
                r0[i] = cfg->init_phase == 2 ? make_double2(a, 0.0) : make_double2(a * h_tcs[i].x, a * h_tcs[i].y);
            }
            CK(cudaMemcpy(R.p, r0.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
        } else {  // seed_random_phase<double>(amp, Rng(seed).fork(0))
            DBuf<uint64_t> sd;
            DBuf<MtState> mt;
            sd.alloc(1);
            const uint64_t es = fork_seed(cfg->seed, 0);
            CK(cudaMemcpy(sd.p, &es, sizeof es, cudaMemcpyHostToDevice));
            SeedChunks ch;
            ch.plan(n, 1);
            mt.alloc(ch.chunks);
            SeedArgs sa{};
            sa.amp = amp.p;
            sa.out64 = R.p;
            sa.out_stride = n;
            sa.npix = n;
            ch.launch(sa, sd.p, mt.p, 1, st);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
        }
        if (cfg->variant == 1) {  // WGS weights, ifta.hpp:141-142
            std::vector<double> w0(n, 1.0);
            if (io->init_weights && cfg->init_phase == 3) std::memcpy(w0.data(), io->init_weights, sizeof(double) * n);
            w.alloc(n);
            CK(cudaMemcpy(w.p, w0.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
        }
        // LT schedule, ifta.hpp:55-63, :144-163
        int bx0 = 0, by0 = 0, bw = nx, bh = ny;
        if (cfg->variant == 2 && io->roi) {
            int x0 = nx, y0 = ny, x1 = -1, y1 = -1;
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x)
                    if (io->roi[(size_t)y * nx + x]) {
                        x0 = std::min(x0, x);
                        x1 = std::max(x1, x);
                        y0 = std::min(y0, y);
                        y1 = std::max(y1, y);
                    }
            bx0 = x0;
            by0 = y0;
            bw = x1 - x0 + 1;
            bh = y1 - y0 + 1;
        }
        if (io->levels) lv.alloc(n);
        const int K = cfg->iterations;
        PhaseClock pc(st, io->profile != nullptr);
        for (int k = 1; k <= K; ++k) {
            pc.mark(3);
            CK(cudaMemcpyAsync(f.p, R.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            propagate64(f, Q, nx, ny, +1, st);                                           // f = prop.inverse(R)
            pc.mark(0);
            k_quant64<<<ew_grid(n), 256, 0, st>>>(f.p, k == K ? lv.p : nullptr, n, q.q);  // quant.apply(f)
            pc.mark(1);
            CK(cudaMemcpyAsync(R.p, f.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            propagate64(R, Q, nx, ny, -1, st);                                           // R = prop.forward(f)
            pc.mark(0);
            mse64(amp.p, Mag64{R.p, nullptr, 0.0}, roi.p, n, M, cfg->freedom_scale, part, g, trace.p + (k - 1), st);
            pc.mark(2);
            if (k == K) break;
            Con64 c{};
            c.amp = amp.p;
            c.w = w.p;
            c.roi = roi.p;
            c.tcs = tcs.p;
            c.phase_freedom = cfg->freedom_phase;
            c.amp_outside_roi = cfg->freedom_amplitude_outside_roi;
            c.lo = cfg->weight_clamp_lo;
            c.hi = cfg->weight_clamp_hi;
            c.nx = nx;
            if (cfg->variant == 2) {
                const double frac = cfg->lt_initial_fraction + (1.0 - cfg->lt_initial_fraction) * (k - 1) / (K - 1);
                const double side = std::sqrt(frac);
                const int aw = std::max(1, (int)std::lround(bw * side)), ah = std::max(1, (int)std::lround(bh * side));
                c.lt = 1;
                c.x0 = bx0 + (bw - aw) / 2;
                c.y0 = by0 + (bh - ah) / 2;
                c.x1 = c.x0 + aw;
                c.y1 = c.y0 + ah;
            }
            k_constrain64<<<ew_grid(n), 256, 0, st>>>(R.p, n, c);
            CK(cudaGetLastError());
            pc.mark(1);
        }
        std::vector<double> tr(K);
        CK(cudaMemcpyAsync(tr.data(), trace.p, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
        if (io->hologram) CK(cudaMemcpyAsync(io->hologram, f.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
        if (io->replay) CK(cudaMemcpyAsync(io->replay, R.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
        if (io->levels) CK(cudaMemcpyAsync(io->levels, lv.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (io->profile)
            pc.report(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), io->profile);
        CK(cudaStreamDestroy(st));
        if (io->trace) std::memcpy(io->trace, tr.data(), sizeof(double) * K);
        if (io->final_error) *io->final_error = tr.back();
    });
}

int hgc_ospr_run_f64(const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny, hgc_ospr_io64* io) {
    const auto t0 = std::chrono::steady_clock::now();
    return guarded([&] {
        validate_ospr_cfg(cfg);
        if (!io || !io->amplitude) invalid("TargetSpec: amplitude image is empty");
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        const size_t n = (size_t)nx * ny;
        validate_slm(slm, n);
        for (size_t i = 0; i < n; ++i) {
            if (!std::isfinite(io->amplitude[i])) invalid("TargetSpec.amplitude: image contains non-finite values");
            if (io->amplitude[i] < 0) invalid("TargetSpec: amplitude must be non-negative");
        }
        const size_t M = roi_count(io->roi, n);
        const int N = cfg->subframes;
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        Dev64 q;
        q.build(slm, n);
        DBuf<double2> f, R, none;
        DBuf<double> T, amp, S, part, g, fm, cm;
        DBuf<uint8_t> roi;
        DBuf<int32_t> lv;
        DBuf<uint64_t> sd;
        DBuf<MtState> mt;
        f.alloc(n);
        R.alloc(n);
        T.alloc(n);
        amp.alloc(n);
        S.alloc(n);
        fm.alloc(N);
        cm.alloc(N);
        CK(cudaMemcpy(T.p, io->amplitude, sizeof(double) * n, cudaMemcpyHostToDevice));
        CK(cudaMemsetAsync(S.p, 0, sizeof(double) * n, st));
        if (io->roi) {
            roi.alloc(n);
            CK(cudaMemcpy(roi.p, io->roi, n, cudaMemcpyHostToDevice));
        }
        if (io->levels) lv.alloc(n * N);
        sd.alloc(1);
        const uint64_t es = fork_seed(cfg->seed, 0);  // ospr.hpp:89
        CK(cudaMemcpy(sd.p, &es, sizeof es, cudaMemcpyHostToDevice));
        SeedChunks ch;
        ch.plan_stream(n, 1);
        mt.alloc(ch.chunks);
        PhaseClock pc(st, io->profile != nullptr);
        for (int k = 1; k <= N; ++k) {
            pc.mark(3);
            const bool budget = cfg->variant == 1 && k > 1;  // ospr.hpp:106-116
            if (budget) k_ospr_amp64<<<ew_grid(n), 256, 0, st>>>(T.p, S.p, n, k, cfg->feedback_gain, amp.p);
            SeedArgs sa{};
            sa.amp = budget ? amp.p : T.p;
            sa.out64 = f.p;
            sa.out_stride = n;
            sa.npix = n;
            ch.launch_stream(sa, sd.p, mt.p, 1, k == 1, st);                              // seed_random_phase<double>
            pc.mark(3);
            propagate64(f, none, nx, ny, +1, st);                                         // fft_inverse
            pc.mark(0);
            k_quant64<<<ew_grid(n), 256, 0, st>>>(f.p, io->levels ? lv.p + n * (k - 1) : nullptr, n, q.q);
            pc.mark(1);
            if (io->frames)
                CK(cudaMemcpyAsync(io->frames + 2 * n * (k - 1), f.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(R.p, f.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            pc.mark(3);
            propagate64(R, none, nx, ny, -1, st);                                         // fft_forward
            pc.mark(0);
            k_ospr_acc64<<<ew_grid(n), 256, 0, st>>>(R.p, n, S.p);                        // ospr.hpp:134-137
            mse64(T.p, Mag64{R.p, nullptr, 0.0}, roi.p, n, M, cfg->freedom_scale, part, g, fm.p + (k - 1), st);
            mse64(T.p, Mag64{nullptr, S.p, (double)k}, roi.p, n, M, cfg->freedom_scale, part, g, cm.p + (k - 1), st);
            CK(cudaGetLastError());
            pc.mark(2);
        }
        DBuf<double> mean;
        DBuf<double2> rep;
        if (io->mean_intensity) mean.alloc(n);
        if (io->replay) rep.alloc(n);
        k_ospr_out64<<<ew_grid(n), 256, 0, st>>>(S.p, n, N, mean.p, rep.p);  // ospr.hpp:149-156
        std::vector<double> hfm(N), hcm(N);
        CK(cudaMemcpyAsync(hfm.data(), fm.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hcm.data(), cm.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        if (io->levels) CK(cudaMemcpyAsync(io->levels, lv.p, sizeof(int32_t) * n * N, cudaMemcpyDeviceToHost, st));
        if (io->mean_intensity)
            CK(cudaMemcpyAsync(io->mean_intensity, mean.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        if (io->replay) CK(cudaMemcpyAsync(io->replay, rep.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (io->profile)
            pc.report(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), io->profile);
        CK(cudaStreamDestroy(st));
        if (io->frame_mse) std::memcpy(io->frame_mse, hfm.data(), sizeof(double) * N);
        if (io->cumulative_mse) std::memcpy(io->cumulative_mse, hcm.data(), sizeof(double) * N);
        if (io->final_error) *io->final_error = hcm.back();
    });
}


}  // extern "C"
