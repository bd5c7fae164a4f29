// primitives.cu — the single-operation entry points of the C ABI:
// FftBackend<float/double> (hgc_fft2d, hgc_fft2d_f64), Propagator<float>
// (hgc_propagate), Quantiser<float>::apply (hgc_quantise), seed_random_phase,
// mse, make_fresnel_phase, the replay-PNG pixel encoding, the MT jump-ahead.
#include "capi_impl.cuh"

extern "C" {
// ============================================================ primitives
// Propagator<float>::forward / inverse (propagation.hpp:81-95); Fourier when
// fresnel == NULL (fft_forward / fft_inverse, fft.hpp:93-113).  Same pass
// order as the fused loop: forward = rows then columns (+norm), inverse =
// columns then rows (+norm, *conj(Q)).
int hgc_propagate(int nx, int ny, int sign, const hgc_fresnel* fresnel, int batch, const float* in, float* out) {
    return guarded([&] {
        if (!in || !out) invalid("fft: null buffer");
        if (sign != -1 && sign != 1) invalid("fft: sign must be -1 or +1");
        if (batch < 1) invalid("fft: batch must be >= 1");
        if (fresnel) validate_fresnel(fresnel);
        check_size(nx, ny);
        const float2* tw = device_twiddles();
        prepare_kernels(nx, ny);
        const size_t npix = (size_t)nx * ny, tot = npix * batch;
        for (size_t i = 0; i < 2 * tot; ++i)  // require_finite, fft.hpp:95-97 / :106-108
            if (!std::isfinite(in[i]))
                invalid(std::string(sign < 0 ? "fft_forward" : "fft_inverse") + ": field contains non-finite values");
        DBuf<float2> f, q;
        f.alloc(tot);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (fresnel) {
            q.alloc(npix);
            double scale = 3.1415926535897932384626433832795 / (fresnel->wavelength * fresnel->distance);
            k_fresnel_q<<<ew_grid(npix), 256, 0, st>>>(nx, ny, scale, fresnel->pixel_pitch_x, fresnel->pixel_pitch_y,
                                                       q.p);
        }
        CK(cudaMemcpyAsync(f.p, in, sizeof(float2) * tot, cudaMemcpyHostToDevice, st));
        const float norm = (float)(1.0 / std::sqrt((double)nx * ny));  // fftw_backend.cpp:121
        RowArgs ra{};
        ra.tw = tw;
        ra.field = f.p;
        ra.bstride = npix;
        ra.ny = ny;
        ra.layout = LAY_ROW;
        ra.sign = sign;
        ra.norm = norm;
        ra.apply_norm = sign > 0;
        ra.fresnel_q = q.p;
        ColArgs ca{};
        ca.tw = tw;
        ca.field = f.p;
        ca.bstride = npix;
        ca.nx = nx;
        ca.sign = sign;
        ca.norm = norm;
        ca.apply_norm = sign < 0;
        if (sign < 0) {
            row_plain(nx, ra, batch, st);
            col_plain(ny, ca, batch, st);
        } else {
            col_plain(ny, ca, batch, st);
            row_plain(nx, ra, batch, st);
        }
        CK(cudaMemcpyAsync(out, f.p, sizeof(float2) * tot, cudaMemcpyDeviceToHost, st));
        cudaError_t e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        CK(e);
    });
}

// Sizes the fused power-of-two kernels take; other sizes go through the
// Bluestein path of k_fft64.cu (FftBackend accepts any nx, ny >= 1).
static bool fast_sizes(int nx, int ny) { return is_pow2(nx) && is_pow2(ny) && nx >= 2 && ny >= 2 && nx <= kMaxLine && ny <= kMaxLine; }
__global__ void k_c64_to_c128(const float2* a, double2* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = make_double2(a[i].x, a[i].y);
}
__global__ void k_c128_to_c64(const double2* a, float2* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = make_float2((float)a[i].x, (float)a[i].y);
}

int hgc_fft2d_f64(int nx, int ny, int sign, int batch, const double* in, double* out) {
    return guarded([&] {
        if (!in || !out) invalid("fft: null buffer");
        if (sign != -1 && sign != 1) invalid("fft: sign must be -1 or +1");
        if (batch < 1) invalid("fft: batch must be >= 1");
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        const bool fast = fast_sizes(nx, ny);
        const size_t tot = (size_t)nx * ny * batch;
        for (size_t i = 0; i < 2 * tot; ++i)  // require_finite, fft.hpp:95-97 / :106-108
            if (!std::isfinite(in[i]))
                invalid(std::string(sign < 0 ? "fft_forward" : "fft_inverse") + ": field contains non-finite values");
        DBuf<double2> f;
        f.alloc(tot);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CK(cudaMemcpyAsync(f.p, in, sizeof(double2) * tot, cudaMemcpyHostToDevice, st));
        if (fast) fft2d_f64(f.p, nx, ny, sign, batch, st);
        else fft2d_any_f64(f.p, nx, ny, sign, batch, st);
        CK(cudaMemcpyAsync(out, f.p, sizeof(double2) * tot, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamDestroy(st));
    });
}

int hgc_fft2d(int nx, int ny, int sign, int batch, const float* in, float* out) {
    if (nx > 0 && ny > 0 && !fast_sizes(nx, ny) && in && out && batch >= 1 && (sign == 1 || sign == -1))
        return guarded([&] {  // any size: Bluestein in double, rounded back to float
            const size_t tot = (size_t)nx * ny * batch;
            for (size_t i = 0; i < 2 * tot; ++i)
                if (!std::isfinite(in[i]))
                    invalid(std::string(sign < 0 ? "fft_forward" : "fft_inverse") + ": field contains non-finite values");
            DBuf<float2> f;
            DBuf<double2> d;
            f.alloc(tot);
            d.alloc(tot);
            cudaStream_t st;
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            CK(cudaMemcpyAsync(f.p, in, sizeof(float2) * tot, cudaMemcpyHostToDevice, st));
            k_c64_to_c128<<<ew_grid(tot), 256, 0, st>>>(f.p, d.p, tot);
            fft2d_any_f64(d.p, nx, ny, sign, batch, st);
            k_c128_to_c64<<<ew_grid(tot), 256, 0, st>>>(d.p, f.p, tot);
            CK(cudaMemcpyAsync(out, f.p, sizeof(float2) * tot, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaStreamDestroy(st));
        });
    return hgc_propagate(nx, ny, sign, nullptr, batch, in, out);
}

int hgc_quantise(const hgc_slm* slm, int nx, int ny, int batch, float* field, int32_t* levels) {
    return guarded([&] {
        if (!field) invalid("quantise: null field");
        if (nx <= 0 || ny <= 0 || batch < 1) invalid("Quantiser: field dimensions mismatch");
        const size_t npix = (size_t)nx * ny, tot = npix * batch;
        validate_slm(slm, npix);
        const float2* tw = device_twiddles();
        QuantDev q;
        build_quant(slm, nx, ny, q);
        DBuf<float2> f;
        DBuf<int32_t> lv;
        f.alloc(tot);
        if (levels) lv.alloc(tot);
        CK(cudaMemcpy(f.p, field, sizeof(float2) * tot, cudaMemcpyHostToDevice));
        k_quantise<<<ew_grid(tot), 256>>>(f.p, lv.p, npix, tot, q.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(field, f.p, sizeof(float2) * tot, cudaMemcpyDeviceToHost));
        if (levels) CK(cudaMemcpy(levels, lv.p, sizeof(int32_t) * tot, cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------ f64 loops
// run_ifta<double> / run_ospr_impl<double> on the device: the reference's
// double arithmetic per pixel (f64path.cuh), the f64 transforms of
// k_fft64.cu (any size), one target per call.
int hgc_replay_to_gray8(const float* replay, int nx, int ny, int batch, uint8_t* out, double* peak) {
    return guarded([&] {
        if (!replay || (!out && !peak)) invalid("replay image: null buffer");
        if (nx <= 0 || ny <= 0 || batch < 1) invalid("ComplexField: dimensions must be positive");
        const size_t npix = (size_t)nx * ny, tot = npix * batch;
        for (size_t i = 0; i < 2 * tot; ++i)  // require_finite(replay, "replay image"), io.cpp:190
            if (!std::isfinite(replay[i])) invalid("replay image: field contains non-finite values");
        DBuf<float2> f;
        DBuf<uint8_t> g;
        DBuf<double> pk;
        f.alloc(tot);
        g.alloc(tot);
        pk.alloc(batch);
        CK(cudaMemcpy(f.p, replay, sizeof(float2) * tot, cudaMemcpyHostToDevice));
        const AmpSrc src{2, f.p, nullptr, 0.0, nx, ny, npix};
        replay_gray8_dev(src, npix, batch, g.p, pk.p, nullptr);
        if (out) CK(cudaMemcpy(out, g.p, tot, cudaMemcpyDeviceToHost));
        if (peak) CK(cudaMemcpy(peak, pk.p, sizeof(double) * batch, cudaMemcpyDeviceToHost));
    });
}

int hgc_mt_jump_state(uint64_t engine_seed, uint64_t draws, uint64_t* window) {
    return guarded([&] {
        if (!window) invalid("mt_jump_state: null buffer");
        mt_jump_state_host(engine_seed, draws, window);
    });
}

int hgc_seed_random_phase(const double* amplitude, int nx, int ny, uint64_t engine_seed, uint64_t skip, float* out) {
    return guarded([&] {
        if (!amplitude || !out) invalid("seed_random_phase: null buffer");
        if (nx <= 0 || ny <= 0) invalid("RealImage: dimensions must be positive");
        const size_t npix = (size_t)nx * ny;
        require_finite_img(amplitude, npix, "seed_random_phase");
        const float2* tw = device_twiddles();
        CK(cudaFuncSetAttribute(k_seed_random_phase<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSeedSmem));
    CK(cudaFuncSetAttribute(k_seed_random_phase<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSeedSmem));
        DBuf<double> a;
        DBuf<float2> f;
        DBuf<MtState> mt;
        DBuf<uint64_t> sd;
        a.alloc(npix);
        f.alloc(npix);
        sd.alloc(1);
        CK(cudaMemcpy(a.p, amplitude, sizeof(double) * npix, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(sd.p, &engine_seed, sizeof(uint64_t), cudaMemcpyHostToDevice));
        SeedChunks ch;
        ch.plan(npix, 1, skip);  // skip: jump ahead instead of drawing
        mt.alloc(ch.chunks);
        SeedArgs sa{};
        sa.amp = a.p;
        sa.out = f.p;
        sa.npix = npix;
        ch.launch(sa, sd.p, mt.p, 1, nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, f.p, sizeof(float2) * npix, cudaMemcpyDeviceToHost));
    });
}

int hgc_mse(const double* target, const float* replay, const uint8_t* mask, int nx, int ny, int scale_free,
            double* out) {
    return guarded([&] {
        if (!target || !replay || !out) invalid("metric: null buffer");
        if (nx <= 0 || ny <= 0) invalid("metric: target and replay dimensions mismatch");
        const size_t n = (size_t)nx * ny;
        require_finite_img(target, n, "metric");
        for (size_t i = 0; i < 2 * n; ++i)
            if (!std::isfinite(replay[i])) invalid("metric: field contains non-finite values");
        if (mask) {
            size_t m = 0;
            for (size_t i = 0; i < n; ++i) m += mask[i] != 0;
            if (m == 0) invalid("MetricConfig: mask covers no pixels");
        }
        const float2* tw = device_twiddles();
        DBuf<double> t, part;
        DBuf<float2> r;
        DBuf<uint8_t> m;
        t.alloc(n);
        r.alloc(n);
        const int blocks = 148 * 2;
        part.alloc((size_t)blocks * 5);
        CK(cudaMemcpy(t.p, target, sizeof(double) * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(r.p, replay, sizeof(float2) * n, cudaMemcpyHostToDevice));
        if (mask) {
            m.alloc(n);
            CK(cudaMemcpy(m.p, mask, n, cudaMemcpyHostToDevice));
        }
        k_mse_partials<<<blocks, 256>>>(t.p, r.p, m.p, n, part.p);
        CK(cudaGetLastError());
        std::vector<double> h((size_t)blocks * 5);
        CK(cudaMemcpy(h.data(), part.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
        double s[5] = {0, 0, 0, 0, 0};
        for (int b = 0; b < blocks; ++b)
            for (int v = 0; v < 5; ++v) s[v] += h[(size_t)b * 5 + v];
        if (!scale_free) {
            *out = s[0] / s[4];
        } else {
            double g = s[2] > 0.0 ? s[1] / s[2] : 0.0;
            if (g < 0.0) g = 0.0;
            double v = s[3] - 2.0 * g * s[1] + g * g * s[2];
            *out = (v < 0 ? 0.0 : v) / s[4];
        }
    });
}

int hgc_fresnel_phase(int nx, int ny, const hgc_fresnel* prm, float* q) {
    return guarded([&] {
        if (!prm || !q) invalid("make_fresnel_phase: null argument");
        validate_fresnel(prm);
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        const size_t n = (size_t)nx * ny;
        DBuf<float2> d;
        d.alloc(n);
        double scale = 3.1415926535897932384626433832795 / (prm->wavelength * prm->distance);
        k_fresnel_q<<<ew_grid(n), 256>>>(nx, ny, scale, prm->pixel_pitch_x, prm->pixel_pitch_y, d.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(q, d.p, sizeof(float2) * n, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
