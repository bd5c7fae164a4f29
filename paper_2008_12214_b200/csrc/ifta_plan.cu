// ifta_plan.cu — the IFTA plan (run_gs / run_weighted_gs /
// run_liu_taghizadeh / run_ifta<float>, ifta.hpp:86-263) behind the C ABI:
// device-resident buffers, the whole run as one CUDA graph of fused passes,
// upload / execute / download, checkpoint, profile and efficiency outputs.
#include "capi_impl.cuh"

// =================================================================== IFTA
struct hgc_ifta_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    hgc_ifta_cfg cfg{};
    int nx = 0, ny = 0, batch = 0;
    size_t npix = 0;
    bool fresnel = false;
    hgc_fresnel fp{};
    QuantDev q;
    bool wide_levels = false;
    bool has_phase = false, has_roi = false;
    size_t M = 0;
    int tiles = 0;
    int cw = 0;  // columns per column-pass CTA (col_width_rt)
    int bx0 = 0, by0 = 0, bw = 0, bh = 0;  // LT roi bounding box
    DBuf<float2> field, Q, tphase_cs, init_field, scratch;
    cudaEvent_t done = nullptr;  // recorded after each execute on the execute stream
    cudaEvent_t up_ev = nullptr;  // end of the last upload's stream work
    DBuf<int> vflags;             // deferred TargetSpec validation flags
    DBuf<float> target_f, weights, init_weights;
    DBuf<double> amp_d, phase_d, partials, trace, stt, eff;  // stt: sum T^2 per target; eff: efficiency
    DBuf<double> scratch_d;
    DBuf<uint8_t> roi, roi_rm, lv8, lv1;
    DBuf<uint16_t> lv16;
    DBuf<MtState> mt;
    DBuf<uint64_t> seeds;
    SeedChunks chunking;
    DevTensorMap tmap;  // field as a TMA tensor (column pass), ny >= 512
    const float2* tw = nullptr;
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_sig = 0;
    int launches = 0;
    bool uploaded = false;
    bool init_weights_given = false;
    bool ckpt = false;  // hgc_ifta_io::checkpoint: the last iteration also constrains
    // Per-pass timing inside the graph (hgc_ifta_plan_set_kernel_timing;
    // external event record nodes, cudaEventRecordExternal):
    // kev[0] before the first group's row pass of iteration 1, kev[2k-1]
    // after its row pass of iteration k, kev[2k] after its column pass.
    bool ktime = false;
    std::vector<cudaEvent_t> kev;
    // HG_STAGGER=1 (experiment): the batch as two halves on two
    // streams of the graph, staggered by a pass, so half B's row pass runs beside
    // half A's column pass and vice versa.
    cudaStream_t sB = nullptr;
    cudaEvent_t evA = nullptr, evB = nullptr, evF = nullptr;
    int group0 = 0;  // targets of the first (timed) group

    // RunReport::profile (report.hpp:38-45) of a run of `seconds`: the device
    // time of the fused passes (in-graph events around the first group's
    // passes, scaled to the whole batch) split by phase.  A fused pass holds
    // several reference phases; the split uses the measured share of each
    // (the quantiser is kRowQuant of the row pass, the MSE
    // partials and constraint kColMetric / kColConstraint of the column pass,
    // the rest is transform).  "other" is the remainder (seed, copies, setup),
    // so the four add up to `seconds` like the reference's (ifta.hpp:231-233).
    void profile_split(double seconds, double* out) const {
        static constexpr double kRowQuant = 0.25, kColMetric = 0.05, kColConstraint = 0.05;
        double row = 0, col = 0;
        if (ktime && !kev.empty() && group0 > 0) {
            for (int k = 1; k <= cfg.iterations; ++k) {
                float a = 0.f, b = 0.f;
                CK(cudaEventElapsedTime(&a, kev[2 * k - 2], kev[2 * k - 1]));
                CK(cudaEventElapsedTime(&b, kev[2 * k - 1], kev[2 * k]));
                row += a;
                col += b;
            }
            const double scale = (double)batch / group0 * 1e-3;
            row *= scale;
            col *= scale;
        }
        double tr = row * (1 - kRowQuant) + col * (1 - kColMetric - kColConstraint);
        double cn = row * kRowQuant + col * kColConstraint, me = col * kColMetric;
        const double dev = tr + cn + me;
        if (dev > seconds && dev > 0) {  // (never expected: the passes run inside the call)
            tr *= seconds / dev;
            cn *= seconds / dev;
            me *= seconds / dev;
        }
        out[0] = tr;
        out[1] = cn;
        out[2] = me;
        out[3] = std::max(0.0, seconds - (tr + cn + me));
    }

    ~hgc_ifta_plan() {
        for (cudaEvent_t e : kev) cudaEventDestroy(e);
        for (cudaEvent_t e : {evA, evB, evF})
            if (e) cudaEventDestroy(e);
        if (sB) cudaStreamDestroy(sB);
        if (graph) cudaGraphExecDestroy(graph);
        if (done) cudaEventDestroy(done);
        if (up_ev) cudaEventDestroy(up_ev);
        if (stream) cudaStreamDestroy(stream);
    }

    bool random_init() const {
        bool target_phase_init = cfg.init_phase == 0 && has_phase && !cfg.freedom_phase;
        return cfg.init_phase != 2 && cfg.init_phase != 3 && !target_phase_init;
    }

    float norm() const { return (float)(1.0 / std::sqrt((double)nx * ny)); }

    // Targets per launch: as many as keep ~70% of L2 for their working set,
    // at least enough CTAs to fill the GPU twice.
    int group_size() const {
        if (const char* ev = getenv("HG_GROUP")) {  // tuning experiments
            int g = atoi(ev);
            if (g >= 1) return std::min(g, batch);
        }
        int dev = 0, l2 = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const double per = (double)npix * (8 + 4 + (cfg.variant == 1 ? 4 : 0));
        int g = (int)std::floor(0.7 * l2 / per);
        if (g < 1) return batch;  // one target overflows L2: no reuse to gain, keep the widest launches
        const int min_g = std::max(1, (int)std::ceil(2.0 * sms / (double)tiles));
        return std::min(std::max(g, min_g), batch);
    }

    SeedArgs seed_args() const {
        SeedArgs sa{};
        sa.states = mt.p;
        sa.seeds = seeds.p;
        sa.amp = amp_d.p;
        sa.amp_stride = npix;
        sa.out = field.p;
        sa.out_stride = npix;
        sa.npix = npix;
        sa.quad = 1;
        sa.nx = nx;
        sa.ny = ny;
        return sa;
    }

    // Aperture-plane pass of iteration k (levels only on the last one).
    RowArgs row_args(bool last) const {
        RowArgs ra{};
        ra.tw = tw;
        ra.field = field.p;
        ra.bstride = npix;
        ra.ny = ny;
        ra.layout = LAY_QUAD;
        ra.norm = norm();
        ra.fresnel_q = fresnel ? Q.p : nullptr;
        ra.q = q.p;
        if (last) {
            ra.levels8 = wide_levels ? nullptr : lv8.p;
            ra.levels16 = wide_levels ? lv16.p : nullptr;
        }
        ra.lv_bstride = npix;
        return ra;
    }

    // Replay-plane pass of iteration k (1-based), ifta.hpp:176-224.
    ColArgs col_args(int k) const {
        const bool last = k == cfg.iterations;
        ColArgs cg{};
        cg.tw = tw;
        cg.field = field.p;
        cg.bstride = npix;
        cg.nx = nx;
        cg.layout = LAY_QUAD;
        cg.norm = norm();
        cg.target = target_f.p;
        cg.t_bstride = npix;
        cg.roi = has_roi ? roi.p : nullptr;
        cg.weights = cfg.variant == 1 ? weights.p : nullptr;
        cg.tphase_cs = cfg.freedom_phase ? nullptr : tphase_cs.p;
        cg.phase_freedom = cfg.freedom_phase;
        cg.amp_outside_roi = cfg.freedom_amplitude_outside_roi;
        cg.scale_free = cfg.freedom_scale;
        cg.clamp_lo = (float)cfg.weight_clamp_lo;
        cg.clamp_hi = (float)cfg.weight_clamp_hi;
        if (cfg.variant == 2 && (!last || ckpt)) {  // LT schedule, ifta.hpp:55-63, :74-84, :189
            const int K = cfg.iterations;
            double frac = cfg.lt_initial_fraction + (1.0 - cfg.lt_initial_fraction) * (k - 1) / (K - 1);
            double side = std::sqrt(frac);
            int aw = std::max(1, (int)std::lround(bw * side));
            int ah = std::max(1, (int)std::lround(bh * side));
            cg.lt = 1;
            cg.lt_x0 = bx0 + (bw - aw) / 2;
            cg.lt_y0 = by0 + (bh - ah) / 2;
            cg.lt_x1 = cg.lt_x0 + aw;
            cg.lt_y1 = cg.lt_y0 + ah;
        }
        cg.last = last ? 1 : 0;
        cg.ckpt = ckpt ? 1 : 0;
        cg.replay_out = field.p;
        cg.partials = partials.p + (size_t)(k - 1) * batch * tiles * 8;
        cg.tmap = tmap.d.p;
        cg.tma_brows = ny / 2;
        cg.cw = cw;
        return cg;
    }

    // Row/column passes of the targets [g0, g0+gn) at iteration k.
    RowArgs row_args_g(int k, int g0) const {
        RowArgs ra = row_args(k == cfg.iterations);
        ra.field += (size_t)g0 * npix;
        if (ra.levels8) ra.levels8 += (size_t)g0 * npix;
        if (ra.levels16) ra.levels16 += (size_t)g0 * npix;
        return ra;
    }
    ColArgs col_args_g(int k, int g0) const {
        ColArgs cg = col_args(k);
        cg.field += (size_t)g0 * npix;
        cg.target += (size_t)g0 * npix;
        if (cg.weights) cg.weights += (size_t)g0 * npix;
        if (cg.tphase_cs) cg.tphase_cs += (size_t)g0 * npix;
        cg.replay_out += (size_t)g0 * npix;
        cg.partials += (size_t)g0 * tiles * 8;
        cg.tma_row0 = g0 * (ny / 2);
        return cg;
    }
    // The whole run_ifta sequence (ifta.hpp:124-226) as stream work.
    void record(cudaStream_t st) {
        launches = 0;
        const size_t tot = npix * batch;
        // ---- initial replay field R0
        if (cfg.init_phase == 3) {
            k_to_quad<<<ew_grid(tot), 256, 0, st>>>(init_field.p, field.p, nx, ny, tot);
            ++launches;
        } else if (cfg.init_phase == 2) {
            k_init_flat<<<ew_grid(tot), 256, 0, st>>>(amp_d.p, field.p, nx, ny, tot);
            ++launches;
        } else if (!random_init()) {
            k_init_target_phase<<<ew_grid(tot), 256, 0, st>>>(amp_d.p, phase_d.p, field.p, nx, ny, tot);
            ++launches;
        } else {
            launches += chunking.launch(seed_args(), seeds.p, mt.p, batch, st);
        }
        CK(cudaGetLastError());
        if (cfg.variant == 1) {
            if (init_weights_given) {
                k_to_colpair<float, float><<<ew_grid(tot), 256, 0, st>>>(init_weights.p, weights.p, nx, ny, tot);
                ++launches;
            } else {
                k_fill_f<<<ew_grid(tot), 256, 0, st>>>(weights.p, tot, 1.0f);
                ++launches;
            }
        }
        // ---- first half of P^-1(R0): inverse column transforms
        ColArgs ca{};
        ca.tw = tw;
        ca.field = field.p;
        ca.bstride = npix;
        ca.nx = nx;
        ca.layout = LAY_QUAD;
        ca.sign = +1;
        ca.tmap = tmap.d.p;
        ca.tma_brows = ny / 2;
        ca.cw = cw;
        col_plain(ny, ca, batch, st);
        ++launches;
        // Iterations run target-group by target-group: a group's field +
        // target (+ weights) is sized to stay L2-resident across the two
        // passes and successive iterations (126 MB L2 on B200).  (Running two
        // target halves on concurrent streams, staggered by a pass, measured
        // no gain at 4096^2: 3927 vs 3950 it/s.)
        const char* stg = getenv("HG_STAGGER");
        if (stg && atoi(stg) != 0 && batch >= 2 && !ktime) {
            if (!sB) {
                CK(cudaStreamCreateWithFlags(&sB, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&evF, cudaEventDisableTiming));
            }
            const int hA = batch / 2, hB = batch - hA;
            CK(cudaEventRecord(evF, st));
            CK(cudaStreamWaitEvent(sB, evF, 0));
            for (int k = 1; k <= cfg.iterations; ++k) {
                row_fused(nx, row_args_g(k, 0), hA, st);
                CK(cudaEventRecord(evA, st));          // A's row pass done
                CK(cudaStreamWaitEvent(sB, evA, 0));   // B's row pass beside A's column pass
                col_gs(ny, col_args_g(k, 0), hA, st);
                row_fused(nx, row_args_g(k, hA), hB, sB);
                CK(cudaEventRecord(evB, sB));          // B's row pass done
                CK(cudaStreamWaitEvent(st, evB, 0));   // A's next row pass beside B's column pass
                col_gs(ny, col_args_g(k, hA), hB, sB);
                launches += 4;
            }
            CK(cudaEventRecord(evF, sB));
            CK(cudaStreamWaitEvent(st, evF, 0));
            group0 = batch;
            k_finalize<<<batch, 32, 0, st>>>(partials.p, cfg.iterations, batch, tiles, (double)M, cfg.freedom_scale, 0,
                                             trace.p, stt.p, eff.p);
            ++launches;
            CK(cudaGetLastError());
            return;
        }
        const int G = group_size();
        group0 = std::min(G, batch);
        const bool tk = ktime && (int)kev.size() == 2 * cfg.iterations + 1;
        for (int g0 = 0; g0 < batch; g0 += G) {
            const int gn = std::min(G, batch - g0);
            if (tk && g0 == 0) CK(cudaEventRecordWithFlags(kev[0], st, cudaEventRecordExternal));
            for (int k = 1; k <= cfg.iterations; ++k) {
                row_fused(nx, row_args_g(k, g0), gn, st);
                if (tk && g0 == 0) CK(cudaEventRecordWithFlags(kev[2 * k - 1], st, cudaEventRecordExternal));
                col_gs(ny, col_args_g(k, g0), gn, st);
                if (tk && g0 == 0) CK(cudaEventRecordWithFlags(kev[2 * k], st, cudaEventRecordExternal));
                launches += 2;
            }
        }
        k_finalize<<<batch, 32, 0, st>>>(partials.p, cfg.iterations, batch, tiles, (double)M, cfg.freedom_scale, 0,
                                         trace.p, stt.p, eff.p);
        ++launches;
        CK(cudaGetLastError());
    }
};

// RunReport::profile for the unfused (f64) loops: events at the reference's
// phase boundaries (ifta.hpp:166-226, ospr.hpp:105-147) on the loop's stream;
// interval i is charged to phase ph[i] (0 transform, 1 constraint, 2 metric,
// 3 other).  Inactive (no events) unless the caller asked for a profile.
extern "C" {

int hgc_ifta_plan_create(hgc_ifta_plan** out, const hgc_ifta_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel,
                         int nx, int ny, int batch) {
    return guarded([&] {
        if (!out) invalid("hgc_ifta_plan_create: null plan pointer");
        *out = nullptr;
        validate_ifta_cfg(cfg);
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        validate_slm(slm, (size_t)nx * ny);
        if (fresnel) validate_fresnel(fresnel);
        if (batch < 1) invalid("hgc_ifta_plan_create: batch must be >= 1");
        check_size(nx, ny);
        const float2* tw = device_twiddles();
        auto p = std::make_unique<hgc_ifta_plan>();
        p->tw = tw;
        CK(cudaGetDevice(&p->device));
        CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        p->cfg = *cfg;
        p->nx = nx;
        p->ny = ny;
        p->batch = batch;
        p->npix = (size_t)nx * ny;
        p->fresnel = fresnel != nullptr;
        if (fresnel) p->fp = *fresnel;
        build_quant(slm, nx, ny, p->q);
        p->wide_levels = slm->levels > 256;
        p->cw = col_width_rt(nx, ny, batch);
        p->tiles = nx / p->cw;
        const size_t tot = p->npix * batch;
        p->field.alloc(tot);
        if (ny >= 512) p->tmap.make(p->field.p, nx, p->cw, (size_t)batch * ny / 2);
        p->target_f.alloc(tot);
        p->amp_d.alloc(tot);
        if (cfg->variant == 1) p->weights.alloc(tot);
        if (p->wide_levels) p->lv16.alloc(tot);
        else p->lv8.alloc(tot);
        p->partials.alloc((size_t)cfg->iterations * batch * p->tiles * 8);
        p->trace.alloc((size_t)cfg->iterations * batch);
        p->eff.alloc(batch);
        p->stt.alloc(batch);
        if (p->random_init()) p->chunking.plan(p->npix, batch);
        p->mt.alloc((size_t)batch * p->chunking.chunks);
        p->seeds.alloc(batch);
        if (fresnel) {
            p->Q.ensure(p->npix);
            double scale = 3.1415926535897932384626433832795 / (fresnel->wavelength * fresnel->distance);
            k_fresnel_q<<<ew_grid(p->npix), 256, 0, p->stream>>>(nx, ny, scale, fresnel->pixel_pitch_x,
                                                                  fresnel->pixel_pitch_y, p->Q.p);
            CK(cudaGetLastError());
        }
        prepare_kernels(nx, ny);
        CK(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->up_ev, cudaEventDisableTiming));
        p->vflags.alloc(1);
        CK(cudaStreamSynchronize(p->stream));
        *out = p.release();
    });
}

int hgc_ifta_plan_upload(hgc_ifta_plan* p, const hgc_ifta_io* io) {
    return guarded([&] {
        if (!p || !io) invalid("hgc_ifta_plan_upload: null argument");
        CK(cudaSetDevice(p->device));
        const size_t npix = p->npix, tot = npix * p->batch;
        if (!io->amplitude) invalid("TargetSpec: amplitude image is empty");
        CK(cudaMemcpyAsync(p->amp_d.p, io->amplitude, sizeof(double) * tot, cudaMemcpyHostToDevice, p->stream));
        p->has_phase = io->phase != nullptr;
        if (io->phase) {
            p->phase_d.ensure(tot);
            CK(cudaMemcpyAsync(p->phase_d.p, io->phase, sizeof(double) * tot, cudaMemcpyHostToDevice, p->stream));
        }
        p->M = roi_count(io->roi, npix);
        launch_validate(p->amp_d.p, io->phase ? p->phase_d.p : nullptr, tot, p->vflags.p, p->stream);
        if (io->roi) {
            p->roi_rm.ensure(npix);
            CK(cudaMemcpyAsync(p->roi_rm.p, io->roi, npix, cudaMemcpyHostToDevice, p->stream));
        }
        if (p->cfg.freedom_scale) {  // only the scale-free MSE uses it
            p->scratch_d.ensure((size_t)kTeBlocks * p->batch);
            k_target_energy_part<<<dim3(kTeBlocks, p->batch), 256, 0, p->stream>>>(
                p->amp_d.p, io->roi ? p->roi_rm.p : nullptr, npix, p->scratch_d.p);
            k_target_energy_fin<<<p->batch, 32, 0, p->stream>>>(p->scratch_d.p, kTeBlocks, p->stt.p);
            CK(cudaGetLastError());
        }
        to_colpair<double, float>(p->amp_d.p, p->target_f.p, p->nx, p->ny, p->batch, p->stream);
        CK(cudaGetLastError());
        if (io->phase) {
            if (!p->cfg.freedom_phase) {
                p->tphase_cs.ensure(tot);
                k_phase_cs<<<ew_grid(tot), 256, 0, p->stream>>>(p->phase_d.p, p->tphase_cs.p, p->nx, p->ny, tot);
            }
        } else if (!p->cfg.freedom_phase) {
            // no target phase: the constraint enforces phase 0 (ifta.hpp:216)
            p->tphase_cs.ensure(tot);
            k_fill_c<<<ew_grid(tot), 256, 0, p->stream>>>(p->tphase_cs.p, tot, make_float2(1.f, 0.f));
            CK(cudaGetLastError());
        }
        if (io->fresnel_q) {  // caller-supplied Q (e.g. from a reference Propagator<float>)
            p->Q.ensure(npix);
            CK(cudaMemcpyAsync(p->Q.p, io->fresnel_q, sizeof(float2) * npix, cudaMemcpyHostToDevice, p->stream));
            p->fresnel = true;
        }
        p->has_roi = io->roi != nullptr;
        p->bx0 = 0;
        p->by0 = 0;
        p->bw = p->nx;
        p->bh = p->ny;
        if (io->roi) {  // column-pair major for the column pass
            p->roi.ensure(npix);
            k_to_colpair<uint8_t, uint8_t><<<ew_grid(npix), 256, 0, p->stream>>>(p->roi_rm.p, p->roi.p, p->nx, p->ny,
                                                                               npix);
            CK(cudaGetLastError());
            if (p->cfg.variant == 2) {  // roi bounding box, ifta.hpp:148-161
                int bx0 = p->nx, by0 = p->ny, bx1 = -1, by1 = -1;
                for (int y = 0; y < p->ny; ++y)
                    for (int x = 0; x < p->nx; ++x)
                        if (io->roi[(size_t)y * p->nx + x]) {
                            bx0 = std::min(bx0, x);
                            bx1 = std::max(bx1, x);
                            by0 = std::min(by0, y);
                            by1 = std::max(by1, y);
                        }
                p->bx0 = bx0;
                p->by0 = by0;
                p->bw = bx1 - bx0 + 1;
                p->bh = by1 - by0 + 1;
            }
        }
        std::vector<uint64_t> es(p->batch);
        for (int b = 0; b < p->batch; ++b) es[b] = fork_seed(io->seeds ? io->seeds[b] : p->cfg.seed, 0);  // ifta.hpp:124
        CK(cudaMemcpyAsync(p->seeds.p, es.data(), sizeof(uint64_t) * p->batch, cudaMemcpyHostToDevice, p->stream));
        if (p->cfg.init_phase == 3) {
            if (!io->init_field) invalid("IftaConfig: init_phase Given requires init_field");
            p->init_field.ensure(tot);
            CK(cudaMemcpyAsync(p->init_field.p, io->init_field, sizeof(float2) * tot, cudaMemcpyHostToDevice, p->stream));
            p->init_weights_given = io->init_weights != nullptr && p->cfg.variant == 1;
            if (p->init_weights_given) {
                p->init_weights.ensure(tot);
                CK(cudaMemcpyAsync(p->init_weights.p, io->init_weights, sizeof(float) * tot, cudaMemcpyHostToDevice,
                                   p->stream));
            }
        }
        p->ckpt = io->checkpoint != 0;
        CK(cudaEventRecord(p->up_ev, p->stream));  // execute waits on it; no host sync
        const uint64_t sig = ((uint64_t)p->ckpt << 59) ^ (uint64_t)(uintptr_t)p->roi.p ^ ((uint64_t)(uintptr_t)p->phase_d.p << 1) ^
                             ((uint64_t)(uintptr_t)p->tphase_cs.p << 2) ^ ((uint64_t)(uintptr_t)p->init_field.p << 3) ^
                             ((uint64_t)(uintptr_t)p->init_weights.p << 4) ^ ((uint64_t)(uintptr_t)p->Q.p << 5) ^
                             ((uint64_t)p->has_roi << 60) ^
                             ((uint64_t)p->has_phase << 61) ^ ((uint64_t)p->init_weights_given << 62) ^ p->M;
        if (p->graph && sig != p->graph_sig) {  // recorded structure changed: rebuild
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        p->graph_sig = sig;
        p->uploaded = true;
    });
}

int hgc_ifta_plan_execute(hgc_ifta_plan* p, void* stream) {
    return guarded([&] {
        if (!p) invalid("hgc_ifta_plan_execute: null plan");
        if (!p->uploaded) invalid("hgc_ifta_plan_execute: inputs not uploaded");
        CK(cudaSetDevice(p->device));
        cudaStream_t st = stream ? (cudaStream_t)stream : p->stream;
        if (!p->graph) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
            try {
                p->record(p->stream);
            } catch (...) {
                cudaStreamEndCapture(p->stream, &g);
                throw;
            }
            CK(cudaStreamEndCapture(p->stream, &g));
            CK(cudaGraphInstantiate(&p->graph, g, 0));
            cudaGraphDestroy(g);
        }
        CK(cudaStreamWaitEvent(st, p->up_ev, 0));  // the last upload's copies and conversions
        CK(cudaGraphLaunch(p->graph, st));
        CK(cudaEventRecord(p->done, st));
    });
}

int hgc_ifta_plan_download(hgc_ifta_plan* p, hgc_ifta_io* io) {
    return guarded([&] {
        if (!p || !io) invalid("hgc_ifta_plan_download: null argument");
        CK(cudaSetDevice(p->device));
        CK(cudaEventSynchronize(p->done));  // this plan's last execute only (other plans keep running)
        {
            int h = 0;
            CK(cudaMemcpy(&h, p->vflags.p, sizeof(int), cudaMemcpyDeviceToHost));
            raise_validation(h);  // deferred from upload
        }
        const size_t tot = p->npix * p->batch;
        const int K = p->cfg.iterations;
        if (io->replay) {  // resident quad layout -> row-major
            p->scratch.ensure(tot);
            k_from_quad<<<ew_grid(tot), 256, 0, p->stream>>>(p->field.p, p->scratch.p, p->nx, p->ny, tot);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(p->stream));
            CK(cudaMemcpy(io->replay, p->scratch.p, sizeof(float2) * tot, cudaMemcpyDeviceToHost));
        }
        if (io->weights) {  // WGS weights (column-pair major -> row-major); 1 when not WGS
            if (p->cfg.variant != 1) {
                std::fill(io->weights, io->weights + tot, 1.0f);
            } else {
                DBuf<float> w;
                w.alloc(tot);
                k_from_colpair<float><<<ew_grid(tot), 256, 0, p->stream>>>(p->weights.p, w.p, p->nx, p->ny, tot);
                CK(cudaGetLastError());
                CK(cudaStreamSynchronize(p->stream));
                CK(cudaMemcpy(io->weights, w.p, sizeof(float) * tot, cudaMemcpyDeviceToHost));
            }
        }
        std::vector<double> tr;
        if (io->trace || io->final_error) {
            tr.resize((size_t)K * p->batch);
            CK(cudaMemcpy(tr.data(), p->trace.p, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost));
            if (io->trace) std::memcpy(io->trace, tr.data(), sizeof(double) * tr.size());
            if (io->final_error)
                for (int b = 0; b < p->batch; ++b) io->final_error[b] = tr[(size_t)b * K + K - 1];
        }
        if (io->efficiency)
            CK(cudaMemcpy(io->efficiency, p->eff.p, sizeof(double) * p->batch, cudaMemcpyDeviceToHost));
        if (io->hologram_gray8) {  // runner.cpp:251-259 hologram.png pixels
            DBuf<uint8_t> g;
            g.alloc(tot);
            levels_gray8_dev(p->wide_levels ? nullptr : p->lv8.p, p->wide_levels ? p->lv16.p : nullptr, tot,
                             p->q.p.levels, g.p, p->stream);
            CK(cudaMemcpy(io->hologram_gray8, g.p, tot, cudaMemcpyDeviceToHost));
        }
        if (io->replay_gray8 || io->replay_peak) {  // runner.cpp:261-265 replay.png pixels + scale
            const AmpSrc src{0, p->field.p, nullptr, 0.0, p->nx, p->ny, p->npix};
            DBuf<uint8_t> g;
            DBuf<double> pk;
            g.alloc(tot);
            pk.alloc(p->batch);
            replay_gray8_dev(src, p->npix, p->batch, g.p, pk.p, p->stream);
            if (io->replay_gray8) CK(cudaMemcpy(io->replay_gray8, g.p, tot, cudaMemcpyDeviceToHost));
            if (io->replay_peak)
                CK(cudaMemcpy(io->replay_peak, pk.p, sizeof(double) * p->batch, cudaMemcpyDeviceToHost));
        }
        if (io->levels1) levels1_dev(p->lv8.p, tot, p->q.p.levels, io->levels1, p->lv1, p->stream);
        if (!p->wide_levels && io->levels8 && !io->levels16 && !io->hologram) {
            CK(cudaMemcpy(io->levels8, p->lv8.p, tot, cudaMemcpyDeviceToHost));  // straight into the caller's buffer
        } else if (io->levels8 || io->levels16 || io->hologram) {
            std::vector<uint8_t> l8;
            std::vector<uint16_t> l16;
            if (p->wide_levels) {
                l16.resize(tot);
                CK(cudaMemcpy(l16.data(), p->lv16.p, sizeof(uint16_t) * tot, cudaMemcpyDeviceToHost));
                if (io->levels8) invalid("hgc_ifta_io: levels8 requested with more than 256 levels");
                if (io->levels16) std::memcpy(io->levels16, l16.data(), sizeof(uint16_t) * tot);
            } else {
                l8.resize(tot);
                CK(cudaMemcpy(l8.data(), p->lv8.p, tot, cudaMemcpyDeviceToHost));
                if (io->levels8) std::memcpy(io->levels8, l8.data(), tot);
                if (io->levels16)
                    for (size_t i = 0; i < tot; ++i) io->levels16[i] = l8[i];
            }
            if (io->hologram)
                levels_to_states(p->q, p->wide_levels ? l16.data() : nullptr, p->wide_levels ? nullptr : l8.data(),
                                 p->npix, tot, io->hologram);
        }
    });
}

int hgc_ifta_plan_device_ptrs(hgc_ifta_plan* p, void** field, void** levels, void** trace) {
    return guarded([&] {
        if (!p) invalid("null plan");
        if (field) *field = p->field.p;
        if (levels) *levels = p->wide_levels ? (void*)p->lv16.p : (void*)p->lv8.p;
        if (trace) *trace = p->trace.p;
    });
}

int hgc_ifta_plan_launches(hgc_ifta_plan* p) { return p ? p->launches : -1; }

// Per-kernel device time of the plan's passes (CUDA events on the plan's
// stream, `reps` back-to-back launches each).  Runs extra iterations on the
// resident field: call after the timed work.
int hgc_ifta_plan_set_kernel_timing(hgc_ifta_plan* p, int on) {
    return guarded([&] {
        if (!p) invalid("hgc_ifta_plan_set_kernel_timing: null plan");
        if (p->graph) invalid("hgc_ifta_plan_set_kernel_timing: call before the first execute");
        CK(cudaSetDevice(p->device));
        p->ktime = on != 0;
        if (p->ktime && p->kev.empty()) {
            p->kev.resize(2 * p->cfg.iterations + 1);
            for (cudaEvent_t& e : p->kev) CK(cudaEventCreate(&e));
        }
    });
}

int hgc_ifta_plan_kernel_times(hgc_ifta_plan* p, double* ms_row, double* ms_col, int* n) {
    return guarded([&] {
        if (!p || !p->ktime || p->kev.empty() || !p->graph)
            invalid("hgc_ifta_plan_kernel_times: timing not enabled or nothing executed");
        CK(cudaSetDevice(p->device));
        CK(cudaEventSynchronize(p->kev.back()));
        // iterations 1 .. K-1 (the last one stores levels and the replay instead)
        const int K = p->cfg.iterations, m = K > 1 ? K - 1 : 1;
        double r = 0, c = 0;
        for (int k = 1; k <= m; ++k) {
            float a = 0.f, b = 0.f;
            CK(cudaEventElapsedTime(&a, p->kev[2 * k - 2], p->kev[2 * k - 1]));
            CK(cudaEventElapsedTime(&b, p->kev[2 * k - 1], p->kev[2 * k]));
            r += a;
            c += b;
        }
        if (ms_row) *ms_row = r / m;
        if (ms_col) *ms_col = c / m;
        if (n) *n = m;
    });
}

int hgc_ifta_plan_profile(hgc_ifta_plan* p, int reps, double* ms_seed, double* ms_row, double* ms_col) {
    return guarded([&] {
        if (!p || !p->uploaded) invalid("hgc_ifta_plan_profile: plan not ready");
        CK(cudaSetDevice(p->device));
        cudaStream_t st = p->stream;
        const int b = p->batch;
        if (ms_seed)
            *ms_seed = time_launches(st, reps, [&] {
                p->chunking.launch(p->seed_args(), p->seeds.p, p->mt.p, b, st);
            });
        const int k = p->cfg.iterations > 1 ? 1 : p->cfg.iterations;  // a constraining iteration when K > 1
        if (ms_row) *ms_row = time_launches(st, reps, [&] { row_fused(p->nx, p->row_args(false), b, st); });
        if (ms_col) *ms_col = time_launches(st, reps, [&] { col_gs(p->ny, p->col_args(k), b, st); });
        CK(cudaGetLastError());
    });
}

int hgc_ifta_plan_destroy(hgc_ifta_plan* p) {
    return guarded([&] {
        if (p) {
            cudaSetDevice(p->device);
            cudaStreamSynchronize(p->stream);
        }
        delete p;
    });
}

int hgc_ifta_run(const hgc_ifta_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny, int batch,
                 hgc_ifta_io* io) {
    auto t0 = std::chrono::steady_clock::now();
    hgc_ifta_plan* p = nullptr;
    int rc = guarded([] { route_device(); });
    if (rc == HGC_OK) rc = hgc_ifta_plan_create(&p, cfg, slm, fresnel, nx, ny, batch);
    if (rc == HGC_OK && io && io->profile) rc = hgc_ifta_plan_set_kernel_timing(p, 1);
    if (rc == HGC_OK) rc = hgc_ifta_plan_upload(p, io);
    if (rc == HGC_OK) rc = guarded([&] { check_validation(p->vflags.p, p->stream); });  // eager in the one-shot run
    if (rc == HGC_OK) rc = hgc_ifta_plan_execute(p, nullptr);
    if (rc == HGC_OK) rc = hgc_ifta_plan_download(p, io);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc == HGC_OK && io && io->profile) rc = guarded([&] { p->profile_split(secs, io->profile); });
    if (p) {
        std::string keep = g_err;
        hgc_ifta_plan_destroy(p);
        g_err = keep;
    }
    if (rc == HGC_OK && io && io->seconds) *io->seconds = secs;
    return rc;
}

}  // extern "C"

