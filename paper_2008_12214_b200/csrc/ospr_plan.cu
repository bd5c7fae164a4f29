// ospr_plan.cu — the OSPR plan (run_ospr / run_adaptive_ospr /
// run_ospr_variant<float>, ospr.hpp:68-185) behind the C ABI: batched jobs,
// subframe blocks across ranks, Fresnel OSPR (extension).
#include "capi_impl.cuh"
#include "launch_impl.cuh"

// =================================================================== OSPR
struct hgc_ospr_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    hgc_ospr_cfg cfg{};
    int nx = 0, ny = 0, jobs = 0, per_job = 0;
    size_t npix = 0;
    QuantDev q;
    bool wide_levels = false, has_roi = false;
    size_t M = 0;
    int tiles = 0;
    int cw = 0;  // columns per column-pass CTA (col_width_rt)
    DBuf<float2> field, field2;  // double-buffered seeded field (plain OSPR)
    DBuf<float> target_f, S;
    DBuf<double> amp_d, partials, traces;
    DBuf<uint8_t> roi, lv8, lv1;
    DBuf<uint16_t> lv16;
    DBuf<MtState> mt;
    DBuf<uint64_t> seeds;
    SeedChunks chunking;
    DevTensorMap tmap1, tmap2;  // field / field2 as TMA tensors (column passes), ny >= 512
    // subframe-block mode: this plan runs global subframes
    // [first, first + cfg.subframes) of a total_subframes job
    int first = 0, total_subframes = 0;
    bool block_mode = false;
    DBuf<float> snaps;            // [cfg.subframes][npix] local S after each frame
    DBuf<double> cum_part, cum_tr;
    int cum_tiles = 0;
    const float2* tw = nullptr;
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_sig = 0;
    int launches = 0;
    bool uploaded = false;
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_seed = nullptr, ev_pass[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;  // recorded after each execute on the execute stream
    cudaEvent_t up_ev = nullptr;  // end of the last upload's stream work
    bool fresnel = false;  // hgc_ospr_plan_set_fresnel
    DBuf<float2> Q;
    // Rows-first subframe (ospr_rows.cuh): plain Fourier OSPR, one MT stream
    // per job walked frame by frame (wst) into per-tile start windows (ck,
    // double-buffered); S accumulates row-major in S_rm and is converted to the
    // column-pair S at the end; the pass C target is row-major fp32.
    bool rows_ok = false;
    int rtiles = 0, qk = 0;
    DBuf<MtState> wst, ck;
    DBuf<float> S_rm, target_rm;
    bool rows_raw = false;  // HG_OSPR_ROWS=3: the walk stores every raw word (no re-twist in the seed pass)
    DBuf<uint64_t> raw;
    bool rows() const { return rows_ok && !fresnel; }
    // RunReport::profile (hgc_ospr_run with io->profile): external events
    // around each subframe's column-inverse, row and accumulating passes
    std::vector<cudaEvent_t> pev;
    void profile_on() {
        if (!pev.empty() || graph) return;
        pev.resize(4 * (size_t)cfg.subframes);
        for (cudaEvent_t& e : pev) CK(cudaEventCreate(&e));
    }
    void pmark(size_t i, cudaStream_t st) {
        if (i < pev.size()) CK(cudaEventRecordWithFlags(pev[i], st, cudaEventRecordExternal));
    }
    // ospr.hpp:118-146 phases: the inverse transform (column pass, row IFFT), the
    // quantiser (kRowQuant of the fused row pass), the forward transform, and the
    // intensity accumulation + both MSEs (kAccMetric of the accumulating column
    // pass); seeds and the rest are "other".
    void profile_split(double seconds, double* out) const {
        static constexpr double kRowQuant = 0.05, kAccMetric = 0.10;
        double ci = 0, rw = 0, ca = 0;
        for (int n = 0; n < cfg.subframes && !pev.empty(); ++n) {
            float a = 0.f, b = 0.f, c = 0.f;
            CK(cudaEventElapsedTime(&a, pev[4 * n], pev[4 * n + 1]));
            CK(cudaEventElapsedTime(&b, pev[4 * n + 1], pev[4 * n + 2]));
            CK(cudaEventElapsedTime(&c, pev[4 * n + 2], pev[4 * n + 3]));
            ci += 1e-3 * a;
            rw += 1e-3 * b;
            ca += 1e-3 * c;
        }
        double tr = ci + rw * (1 - kRowQuant) + ca * (1 - kAccMetric), cn = rw * kRowQuant, me = ca * kAccMetric;
        const double dev = tr + cn + me;
        if (dev > seconds && dev > 0) {
            tr *= seconds / dev;
            cn *= seconds / dev;
            me *= seconds / dev;
        }
        out[0] = tr;
        out[1] = cn;
        out[2] = me;
        out[3] = std::max(0.0, seconds - (tr + cn + me));
    }
    DBuf<int> vflags;             // deferred TargetSpec validation flags
    DBuf<uint8_t> roi_rm;

    ~hgc_ospr_plan() {
        if (graph) cudaGraphExecDestroy(graph);
        for (cudaEvent_t e : pev) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_fork, ev_seed, ev_pass[0], ev_pass[1], done, up_ev})
            if (e) cudaEventDestroy(e);
        if (stream2) cudaStreamDestroy(stream2);
        if (stream) cudaStreamDestroy(stream);
    }

    // Pre-seeded mode (plain OSPR, fewer jobs than SMs): all N subframes'
    // draws are one stream of N*npix per job, seeded in one chunked launch
    // (jump-ahead start states) into N field slices; the passes then run
    // frame by frame on their slice.  Otherwise one seed launch per frame,
    // double-buffered against the passes of the previous frame.
    bool preseed = false;
    size_t fstride = 0;  // field elements per job
    bool overlapped() const { return cfg.variant == 0 && field2.p; }
    float2* buf(int n) const {
        if (preseed) return field.p + (size_t)(n - 1) * npix;
        return (overlapped() && (n & 1) == 0) ? field2.p : field.p;
    }
    SeedArgs seed_all_args() const {
        SeedArgs sa{};
        sa.amp = amp_d.p;
        sa.amp_stride = per_job ? npix : 0;
        sa.out = field.p;
        sa.out_stride = fstride;
        sa.npix = (size_t)cfg.subframes * npix;
        sa.quad = 1;
        sa.nx = nx;
        sa.ny = ny;
        return sa;
    }

    float norm() const { return (float)(1.0 / std::sqrt((double)nx * ny)); }

    // Seed of subframe n (1-based): fresh stream at n = 1, continued after.
    SeedArgs seed_args(int n) const {
        SeedArgs sa{};
        sa.states = mt.p;
        sa.seeds = n == 1 ? seeds.p : nullptr;
        sa.amp = amp_d.p;
        sa.amp_stride = per_job ? npix : 0;
        sa.out = buf(n);
        sa.out_stride = npix;
        sa.npix = npix;
        sa.quad = 1;
        sa.nx = nx;
        sa.ny = ny;
        if (cfg.variant == 1 && n > 1) {  // adaptive budget, ospr.hpp:106-116
            sa.S = S.p;
            sa.S_stride = npix;
            sa.n = n;
            sa.gain = cfg.feedback_gain;
        }
        return sa;
    }
    void set_tma(ColArgs& c, int n) const {  // the TMA view of buf(n) (+ the launch's column width)
        c.cw = cw;
        if (preseed) {
            c.tmap = tmap1.d.p;
            c.tma_row0 = (n - 1) * (ny / 2);
            c.tma_brows = cfg.subframes * (ny / 2);
        } else {
            c.tmap = buf(n) == field2.p ? tmap2.d.p : tmap1.d.p;
            c.tma_row0 = 0;
            c.tma_brows = ny / 2;
        }
    }
    ColArgs col_inv_args(int n) const {
        ColArgs ci{};
        ci.tw = tw;
        ci.field = buf(n);
        ci.bstride = fstride;
        ci.nx = nx;
        ci.layout = LAY_QUAD;
        ci.sign = +1;
        set_tma(ci, n);
        return ci;
    }
    RowArgs row_args(int n) const {
        const int N = cfg.subframes;
        RowArgs ra{};
        ra.tw = tw;
        ra.field = buf(n);
        ra.bstride = fstride;
        ra.ny = ny;
        ra.layout = LAY_QUAD;
        ra.norm = norm();
        ra.q = q.p;
        ra.levels8 = wide_levels ? nullptr : lv8.p + (size_t)(n - 1) * npix;
        ra.levels16 = wide_levels ? lv16.p + (size_t)(n - 1) * npix : nullptr;
        ra.lv_bstride = (size_t)N * npix;
        ra.fresnel_q = fresnel ? Q.p : nullptr;  // Fresnel OSPR (extension): f = IFFT(seed) conj(Q), R = FFT(f Q)
        return ra;
    }
    ColArgs col_acc_args(int n) const {
        ColArgs co{};
        co.tw = tw;
        co.field = buf(n);
        co.bstride = fstride;
        co.nx = nx;
        co.layout = LAY_QUAD;
        co.norm = norm();
        co.target = target_f.p;
        co.t_bstride = per_job ? npix : 0;
        co.roi = has_roi ? roi.p : nullptr;
        co.scale_free = cfg.freedom_scale;
        co.partials = partials.p + (size_t)(n - 1) * jobs * tiles * 8;
        co.S = S.p;  // per job, even when the target is shared
        co.S_bstride = npix;
        co.inv_n = 1.0f / (float)n;
        set_tma(co, n);
        return co;
    }

    ColArgs col_mid_args(int n) const {
        ColArgs cm{};
        cm.tw = tw;
        cm.field = field.p;
        cm.bstride = npix;
        cm.nx = nx;
        cm.layout = LAY_QUAD;
        cm.norm = norm();
        cm.q = q.p;
        cm.levels8 = lv8.p + (size_t)(n - 1) * npix;
        cm.lv_bstride = (size_t)cfg.subframes * npix;
        cm.cw = cw;
        cm.tmap = tmap1.d.p;
        cm.tma_row0 = 0;
        cm.tma_brows = ny / 2;
        return cm;
    }
    RowAccArgs row_acc_args(int n) const {
        RowAccArgs ra{};
        ra.field = field.p;
        ra.npix = npix;
        ra.tw = tw;
        ra.norm = norm();
        ra.inv_n = 1.0f / (float)n;
        ra.S = S_rm.p;
        ra.target = target_rm.p;
        ra.t_bstride = per_job ? npix : 0;
        ra.roi = has_roi ? roi_rm.p : nullptr;
        ra.partials = partials.p + (size_t)(n - 1) * jobs * rtiles * 8;
        return ra;
    }
    SeedRowArgs seed_rows_args(int n) const {
        SeedRowArgs sa{};
        sa.ck = ck.p + (size_t)(n & 1) * jobs * rtiles;
        sa.raw = rows_raw ? raw.p + (size_t)(n & 1) * jobs * npix : nullptr;
        sa.amp = amp_d.p;
        sa.amp_stride = per_job ? npix : 0;
        sa.field = field.p;
        sa.npix = npix;
        sa.tw = tw;
        sa.chunks = rtiles;
        return sa;
    }
    WalkArgs walk_args(int n) const {
        WalkArgs wa{};
        wa.states = wst.p;
        wa.seeds = n == 1 ? seeds.p : nullptr;
        wa.ck = ck.p + (size_t)(n & 1) * jobs * rtiles;
        wa.streams = jobs;
        wa.chunks = rtiles;
        wa.len = ospr_rows_len(nx);
        wa.raw = rows_raw ? raw.p + (size_t)(n & 1) * jobs * npix : nullptr;
        return wa;
    }
    // The rows-first subframe loop: the walk of frame n (its own stream of the
    // graph, a few warps) runs beside the passes of frame n-1; then seed + row
    // IFFT, column IFFT + quantiser + column FFT, row FFT + accumulation.
    void record_rows(cudaStream_t st) {
        launches = 0;
        const int N = cfg.subframes;
        CK(cudaMemsetAsync(S_rm.p, 0, sizeof(float) * npix * jobs, st));
        cudaStream_t ss = stream2 ? stream2 : st;
        if (ss != st) {
            CK(cudaEventRecord(ev_fork, st));
            CK(cudaStreamWaitEvent(ss, ev_fork, 0));
        }
        for (int n = 1; n <= N; ++n) {
            if (ss != st && n >= 3) CK(cudaStreamWaitEvent(ss, ev_pass[n & 1], 0));  // checkpoints n%2 read
            ospr_rows_walk(walk_args(n), ss);
            if (ss != st) {
                CK(cudaEventRecord(ev_seed, ss));
                CK(cudaStreamWaitEvent(st, ev_seed, 0));
            }
            pmark(4 * (size_t)(n - 1), st);
            ospr_rows_seed(nx, seed_rows_args(n), jobs, st);
            if (ss != st) CK(cudaEventRecord(ev_pass[n & 1], st));
            pmark(4 * (size_t)(n - 1) + 1, st);
            ospr_rows_mid(ny, col_mid_args(n), qk, jobs, st);
            pmark(4 * (size_t)(n - 1) + 2, st);
            ospr_rows_acc(nx, row_acc_args(n), rtiles, jobs, st);
            pmark(4 * (size_t)(n - 1) + 3, st);
            launches += 4;
        }
        if (ss != st) {
            CK(cudaEventRecord(ev_fork, ss));
            CK(cudaStreamWaitEvent(st, ev_fork, 0));
        }
        to_colpair<float, float>(S_rm.p, S.p, nx, ny, (size_t)jobs, st);  // the plan's S layout (downloads)
        k_finalize<<<jobs, 32, 0, st>>>(partials.p, N, jobs, rtiles, (double)M, cfg.freedom_scale, 1, traces.p);
        launches += 2;
        CK(cudaGetLastError());
    }

    // run_ospr_impl's subframe loop (ospr.hpp:105-147), all jobs at once.
    // Plain OSPR: the seed of frame n+1 (one MT stream per job, its own
    // stream of the graph) overlaps the three passes of frame n on a second
    // field buffer; a seed CTA (512 thr x 56 regs, 40 KiB) co-resides with a
    // pass CTA on an SM.  Adaptive OSPR seeds frame n from S after frame n-1,
    // so it stays sequential.
    void record(cudaStream_t st) {
        if (rows()) {
            record_rows(st);
            return;
        }
        launches = 0;
        const int N = cfg.subframes;
        CK(cudaMemsetAsync(S.p, 0, sizeof(float) * npix * jobs, st));
        if (preseed) {
            launches += chunking.launch(seed_all_args(), seeds.p, mt.p, jobs, st);
            CK(cudaGetLastError());
        }
        const bool ov = overlapped();
        cudaStream_t ss = ov ? stream2 : st;
        if (ov) {  // fork the seed stream into the capture
            CK(cudaEventRecord(ev_fork, st));
            CK(cudaStreamWaitEvent(ss, ev_fork, 0));
        }
        for (int n = 1; n <= N; ++n) {
            if (ov && n >= 3) CK(cudaStreamWaitEvent(ss, ev_pass[n & 1], 0));  // buffer n%2 free again
            if (!preseed) launches += chunking.launch_stream(seed_args(n), seeds.p, mt.p, jobs, n == 1, ss);
            CK(cudaGetLastError());
            if (ov) {
                CK(cudaEventRecord(ev_seed, ss));
                CK(cudaStreamWaitEvent(st, ev_seed, 0));
            }
            pmark(4 * (size_t)(n - 1), st);
            col_plain(ny, col_inv_args(n), jobs, st);
            pmark(4 * (size_t)(n - 1) + 1, st);
            row_fused(nx, row_args(n), jobs, st);
            pmark(4 * (size_t)(n - 1) + 2, st);
            col_ospr(ny, col_acc_args(n), jobs, st);
            pmark(4 * (size_t)(n - 1) + 3, st);
            if (block_mode)  // local running sum after frame n, for hgc_ospr_block_finish
                CK(cudaMemcpyAsync(snaps.p + (size_t)(n - 1) * npix, S.p, sizeof(float) * npix, cudaMemcpyDeviceToDevice,
                                   st));
            if (ov) CK(cudaEventRecord(ev_pass[n & 1], st));
            launches += 3;
        }
        if (ov) {  // join the seed stream
            CK(cudaEventRecord(ev_fork, ss));
            CK(cudaStreamWaitEvent(st, ev_fork, 0));
        }
        k_finalize<<<jobs, 32, 0, st>>>(partials.p, N, jobs, tiles, (double)M, cfg.freedom_scale, 1, traces.p);
        ++launches;
        CK(cudaGetLastError());
    }
};

extern "C" {


static void create_ospr_plan(hgc_ospr_plan** out, const hgc_ospr_cfg* cfg_in, const hgc_slm* slm, int nx, int ny,
                             int jobs, int per_job_target, int first, int count) {
        if (!out) invalid("hgc_ospr_plan_create: null plan pointer");
        *out = nullptr;
        validate_ospr_cfg(cfg_in);
        const bool block = count > 0;
        if (block) {
            if (cfg_in->variant != 0)
                fail(HGC_EUNSUPPORTED, "hgc_ospr_block_plan_create: adaptive OSPR is sequential (replicas only)");
            if (first < 0 || first + count > cfg_in->subframes)
                invalid("hgc_ospr_block_plan_create: subframe block outside [0, subframes)");
        }
        hgc_ospr_cfg cfg_local = *cfg_in;
        if (block) cfg_local.subframes = count;
        const hgc_ospr_cfg* cfg = &cfg_local;
        if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
        validate_slm(slm, (size_t)nx * ny);
        if (jobs < 1) invalid("hgc_ospr_plan_create: jobs must be >= 1");
        check_size(nx, ny);
        const float2* tw = device_twiddles();
        auto p = std::make_unique<hgc_ospr_plan>();
        p->tw = tw;
        CK(cudaGetDevice(&p->device));
        CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        p->cfg = *cfg;
        p->nx = nx;
        p->ny = ny;
        p->jobs = jobs;
        p->per_job = per_job_target ? 1 : 0;
        p->npix = (size_t)nx * ny;
        build_quant(slm, nx, ny, p->q);
        p->wide_levels = slm->levels > 256;
        p->cw = col_width_rt(nx, ny, jobs);
        p->tiles = nx / p->cw;
        const size_t tot = p->npix * jobs;
        const size_t ttot = p->per_job ? tot : p->npix;
        {
            int dev = 0, sms = 148;
            CK(cudaGetDevice(&dev));
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const size_t all = (size_t)cfg->subframes * p->npix;
            // HG_OSPR_ROWS (rows-first subframes, ospr_rows.cuh): unset / 0 off, 1 for plans with a job
            // per SM, 2 also for few jobs (tests), 3 as 2 with the walk storing every raw word
            const char* e = getenv("HG_OSPR_ROWS");
            const bool force_rows = e && atoi(e) >= 2 && ospr_rows_supported(nx, ny);
            p->preseed = cfg->variant == 0 && cfg->subframes > 1 && jobs < sms && all < (1ull << 31) &&
                         all * jobs * sizeof(float2) <= (8ull << 30) && !force_rows;
            p->fstride = p->preseed ? all : p->npix;
        }
        {
            const char* e = getenv("HG_OSPR_ROWS");
            // opt-in (measured slower than the column-first loop)
            p->rows_ok = e && atoi(e) != 0 && cfg->variant == 0 && !p->preseed && !block && !p->wide_levels &&
                         ospr_rows_supported(nx, ny);
        }
        p->field.alloc(p->fstride * jobs);
        if (ny >= 512) p->tmap1.make(p->field.p, nx, p->cw, p->fstride * jobs / (2 * (size_t)nx));
        if (!p->preseed && cfg->variant == 0 && cfg->subframes > 1) {  // second stream (+ buffer) for seed/pass overlap
            if (!p->rows_ok) {  // (a Fresnel plan set later runs the column-first loop without the overlap)
                p->field2.alloc(tot);
                if (ny >= 512) p->tmap2.make(p->field2.p, nx, p->cw, tot / (2 * (size_t)nx));
            }
            CK(cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_seed, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_pass[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_pass[1], cudaEventDisableTiming));
        }
        p->S.alloc(tot);
        p->target_f.alloc(ttot);
        p->amp_d.alloc(ttot);
        const size_t lvtot = tot * cfg->subframes;
        if (p->wide_levels) p->lv16.alloc(lvtot);
        else p->lv8.alloc(lvtot);
        if (p->rows_ok) {
            p->rtiles = ospr_rows_tiles(nx, ny);
            p->qk = quant_kind(p->q.p);
            p->wst.alloc(jobs);
            p->ck.alloc(2 * (size_t)jobs * p->rtiles);
            const char* e = getenv("HG_OSPR_ROWS");
            p->rows_raw = e && atoi(e) == 3;
            if (p->rows_raw) p->raw.alloc(2 * tot);
            p->S_rm.alloc(tot);
            p->target_rm.alloc(ttot);
            ColArgs c0{};
            ospr_rows_seed(nx, SeedRowArgs{}, jobs, nullptr, true);
            ospr_rows_mid(ny, c0, p->qk, jobs, nullptr, true);
            ospr_rows_acc(nx, RowAccArgs{}, p->rtiles, jobs, nullptr, true);
        }
        p->partials.alloc((size_t)cfg->subframes * jobs * std::max(p->tiles, p->rtiles) * 8);
        p->traces.alloc((size_t)cfg->subframes * jobs * 2);
        p->first = block ? first : 0;
        p->total_subframes = cfg_in->subframes;
        p->block_mode = block;
        if (block) {
            p->snaps.alloc((size_t)count * p->npix);
            p->cum_tiles = std::min<int>(148 * 4, (int)((p->npix + 255) / 256));
            p->cum_part.alloc((size_t)count * p->cum_tiles * 8);
            p->cum_tr.alloc((size_t)count * 2);
        }
        if (p->preseed) p->chunking.plan(p->fstride, jobs, (uint64_t)p->first * p->npix);
        else p->chunking.plan_stream(p->npix, jobs, (uint64_t)p->first * p->npix);
        p->mt.alloc((size_t)jobs * p->chunking.chunks);
        p->seeds.alloc(jobs);
        prepare_kernels(nx, ny);
        CK(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->up_ev, cudaEventDisableTiming));
        p->vflags.alloc(1);
        CK(cudaStreamSynchronize(p->stream));
        *out = p.release();
}

int hgc_ospr_plan_create(hgc_ospr_plan** out, const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny, int jobs,
                         int per_job_target) {
    return guarded([&] { create_ospr_plan(out, cfg, slm, nx, ny, jobs, per_job_target, 0, 0); });
}

int hgc_ospr_block_plan_create(hgc_ospr_plan** out, const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny,
                               int first, int count) {
    return guarded([&] {
        if (count < 1) invalid("hgc_ospr_block_plan_create: count must be >= 1");
        create_ospr_plan(out, cfg, slm, nx, ny, 1, 0, first, count);
    });
}

int hgc_ospr_block_sum(hgc_ospr_plan* p, void** dev_ptr, size_t* count) {
    return guarded([&] {
        if (!p || !p->block_mode) invalid("hgc_ospr_block_sum: not a subframe-block plan");
        if (dev_ptr) *dev_ptr = p->S.p;
        if (count) *count = p->npix;
    });
}

int hgc_ospr_block_finish(hgc_ospr_plan* p, const void* gathered, int nblocks, int index, void* stream) {
    return guarded([&] {
        if (!p || !p->block_mode) invalid("hgc_ospr_block_finish: not a subframe-block plan");
        if (!gathered || nblocks < 1 || index < 0 || index >= nblocks)
            invalid("hgc_ospr_block_finish: bad gathered buffer / block index");
        CK(cudaSetDevice(p->device));
        cudaStream_t st = stream ? (cudaStream_t)stream : p->stream;
        CK(cudaStreamWaitEvent(st, p->done, 0));
        const int K = p->cfg.subframes;
        dim3 grid(p->cum_tiles, K);
        k_ospr_block_cum<<<grid, 256, 0, st>>>((const float*)gathered, index, nblocks, p->snaps.p, p->target_f.p,
                                               p->has_roi ? p->roi.p : nullptr, p->npix, p->first, p->S.p,
                                               p->cum_part.p);
        k_finalize<<<1, 32, 0, st>>>(p->cum_part.p, K, 1, p->cum_tiles, (double)p->M, p->cfg.freedom_scale, 1,
                                      p->cum_tr.p);
        // cumulative entries (odd slots) replace the block-local ones
        CK(cudaMemcpy2DAsync(p->traces.p + 1, 2 * sizeof(double), p->cum_tr.p + 1, 2 * sizeof(double), sizeof(double),
                             K, cudaMemcpyDeviceToDevice, st));
        CK(cudaGetLastError());
        CK(cudaEventRecord(p->done, st));
    });
}

int hgc_ospr_plan_upload(hgc_ospr_plan* p, const hgc_ospr_io* io) {
    return guarded([&] {
        if (!p || !io) invalid("hgc_ospr_plan_upload: null argument");
        CK(cudaSetDevice(p->device));
        const size_t ttot = p->per_job ? p->npix * p->jobs : p->npix;
        if (!io->amplitude) invalid("TargetSpec: amplitude image is empty");
        CK(cudaMemcpyAsync(p->amp_d.p, io->amplitude, sizeof(double) * ttot, cudaMemcpyHostToDevice, p->stream));
        p->M = roi_count(io->roi, p->npix);
        launch_validate(p->amp_d.p, nullptr, ttot, p->vflags.p, p->stream);
        to_colpair<double, float>(p->amp_d.p, p->target_f.p, p->nx, p->ny, ttot / p->npix, p->stream);
        if (p->rows_ok) ospr_rows_target(p->amp_d.p, p->target_rm.p, ttot, p->stream);
        CK(cudaGetLastError());
        p->has_roi = io->roi != nullptr;
        if (io->roi) {  // column-pair major
            p->roi.ensure(p->npix);
            p->roi_rm.ensure(p->npix);
            CK(cudaMemcpyAsync(p->roi_rm.p, io->roi, p->npix, cudaMemcpyHostToDevice, p->stream));
            k_to_colpair<uint8_t, uint8_t><<<ew_grid(p->npix), 256, 0, p->stream>>>(p->roi_rm.p, p->roi.p, p->nx,
                                                                                  p->ny, p->npix);
            CK(cudaGetLastError());
            
        }
        std::vector<uint64_t> es(p->jobs);
        for (int j = 0; j < p->jobs; ++j) es[j] = fork_seed(io->seeds ? io->seeds[j] : p->cfg.seed, 0);  // ospr.hpp:89
        CK(cudaMemcpyAsync(p->seeds.p, es.data(), sizeof(uint64_t) * p->jobs, cudaMemcpyHostToDevice, p->stream));
        CK(cudaEventRecord(p->up_ev, p->stream));
        const uint64_t sig = (uint64_t)(uintptr_t)p->roi.p ^ ((uint64_t)p->has_roi << 60) ^ p->M;
        if (p->graph && sig != p->graph_sig) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        p->graph_sig = sig;
        p->uploaded = true;
    });
}

int hgc_ospr_plan_execute(hgc_ospr_plan* p, void* stream) {
    return guarded([&] {
        if (!p) invalid("hgc_ospr_plan_execute: null plan");
        if (!p->uploaded) invalid("hgc_ospr_plan_execute: inputs not uploaded");
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

int hgc_ospr_plan_download(hgc_ospr_plan* p, hgc_ospr_io* io) {
    return guarded([&] {
        if (!p || !io) invalid("hgc_ospr_plan_download: null argument");
        CK(cudaSetDevice(p->device));
        CK(cudaEventSynchronize(p->done));
        {
            int h = 0;
            CK(cudaMemcpy(&h, p->vflags.p, sizeof(int), cudaMemcpyDeviceToHost));
            raise_validation(h);  // deferred from upload
        }
        const int N = p->cfg.subframes;
        const size_t npix = p->npix, tot = npix * p->jobs, lvtot = tot * N;
        std::vector<double> tr((size_t)N * p->jobs * 2);
        CK(cudaMemcpy(tr.data(), p->traces.p, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost));
        for (int j = 0; j < p->jobs; ++j)
            for (int n = 0; n < N; ++n) {
                size_t o = ((size_t)j * N + n);
                if (io->frame_mse) io->frame_mse[o] = tr[o * 2];
                if (io->cumulative_mse) io->cumulative_mse[o] = tr[o * 2 + 1];
            }
        if (io->final_error)
            for (int j = 0; j < p->jobs; ++j) io->final_error[j] = tr[((size_t)j * N + N - 1) * 2 + 1];
        if (io->mean_intensity || io->replay) {  // ospr.hpp:149-156
            std::vector<float> S(tot);
            CK(cudaMemcpy(S.data(), p->S.p, sizeof(float) * tot, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < tot; ++i) {  // S is column-pair major per job
                const size_t j = i / npix, pi = i % npix;
                const int px = (int)(pi % p->nx), py = (int)(pi / p->nx);
                double m = (double)S[j * npix + colpair_index(px, py, p->ny)] / p->total_subframes;
                if (io->mean_intensity) io->mean_intensity[i] = m;
                if (io->replay) {
                    io->replay[2 * i] = (float)std::sqrt(m);
                    io->replay[2 * i + 1] = 0.f;
                }
            }
        }
        if (io->frames_gray8) {
            DBuf<uint8_t> g;
            g.alloc(lvtot);
            levels_gray8_dev(p->wide_levels ? nullptr : p->lv8.p, p->wide_levels ? p->lv16.p : nullptr, lvtot,
                             p->q.p.levels, g.p, p->stream);
            CK(cudaMemcpy(io->frames_gray8, g.p, lvtot, cudaMemcpyDeviceToHost));
        }
        if (io->replay_gray8 || io->replay_peak) {
            const AmpSrc src{1, nullptr, p->S.p, (double)p->total_subframes, p->nx, p->ny, npix};
            DBuf<uint8_t> g;
            DBuf<double> pk;
            g.alloc(tot);
            pk.alloc(p->jobs);
            replay_gray8_dev(src, npix, p->jobs, g.p, pk.p, p->stream);
            if (io->replay_gray8) CK(cudaMemcpy(io->replay_gray8, g.p, tot, cudaMemcpyDeviceToHost));
            if (io->replay_peak) CK(cudaMemcpy(io->replay_peak, pk.p, sizeof(double) * p->jobs, cudaMemcpyDeviceToHost));
        }
        if (io->levels1) levels1_dev(p->lv8.p, lvtot, p->q.p.levels, io->levels1, p->lv1, p->stream);
        if (!p->wide_levels && io->levels8 && !io->levels16 && !io->frames) {
            CK(cudaMemcpy(io->levels8, p->lv8.p, lvtot, cudaMemcpyDeviceToHost));
        } else if (io->levels8 || io->levels16 || io->frames) {
            std::vector<uint8_t> l8;
            std::vector<uint16_t> l16;
            if (p->wide_levels) {
                l16.resize(lvtot);
                CK(cudaMemcpy(l16.data(), p->lv16.p, sizeof(uint16_t) * lvtot, cudaMemcpyDeviceToHost));
                if (io->levels8) invalid("hgc_ospr_io: levels8 requested with more than 256 levels");
                if (io->levels16) std::memcpy(io->levels16, l16.data(), sizeof(uint16_t) * lvtot);
            } else {
                l8.resize(lvtot);
                CK(cudaMemcpy(l8.data(), p->lv8.p, lvtot, cudaMemcpyDeviceToHost));
                if (io->levels8) std::memcpy(io->levels8, l8.data(), lvtot);
                if (io->levels16)
                    for (size_t i = 0; i < lvtot; ++i) io->levels16[i] = l8[i];
            }
            if (io->frames)
                levels_to_states(p->q, p->wide_levels ? l16.data() : nullptr, p->wide_levels ? nullptr : l8.data(), npix,
                                 lvtot, io->frames);
        }
    });
}

int hgc_ospr_plan_device_ptrs(hgc_ospr_plan* p, void** levels, void** traces, void** intensity) {
    return guarded([&] {
        if (!p) invalid("null plan");
        if (levels) *levels = p->wide_levels ? (void*)p->lv16.p : (void*)p->lv8.p;
        if (traces) *traces = p->traces.p;
        if (intensity) *intensity = p->S.p;
    });
}

int hgc_ospr_plan_launches(hgc_ospr_plan* p) { return p ? p->launches : -1; }

// Per-kernel device time of one subframe's four passes (see hgc_ifta_plan_profile).
int hgc_ospr_plan_profile(hgc_ospr_plan* p, int reps, double* ms_seed, double* ms_col_inv, double* ms_row,
                          double* ms_col_acc) {
    return guarded([&] {
        if (!p || !p->uploaded) invalid("hgc_ospr_plan_profile: plan not ready");
        CK(cudaSetDevice(p->device));
        cudaStream_t st = p->stream;
        const int j = p->jobs;
        if (p->rows()) {  // rows-first subframe: walk, seed + row IFFT, column pass, row FFT + accumulation
            if (ms_seed) *ms_seed = time_launches(st, reps, [&] { ospr_rows_walk(p->walk_args(2), st); });
            if (ms_col_inv)
                *ms_col_inv = time_launches(st, reps, [&] { ospr_rows_seed(p->nx, p->seed_rows_args(2), j, st); });
            if (ms_row) *ms_row = time_launches(st, reps, [&] { ospr_rows_mid(p->ny, p->col_mid_args(1), p->qk, j, st); });
            if (ms_col_acc)
                *ms_col_acc = time_launches(st, reps, [&] { ospr_rows_acc(p->nx, p->row_acc_args(1), p->rtiles, j, st); });
            CK(cudaGetLastError());
            return;
        }
        if (ms_seed)
            *ms_seed = p->preseed  // per-frame share of the one all-frames seed
                           ? time_launches(st, reps, [&] {
                                 p->chunking.launch(p->seed_all_args(), p->seeds.p, p->mt.p, j, st);
                             }) / p->cfg.subframes
                           : time_launches(st, reps, [&] {
                                 p->chunking.launch_stream(p->seed_args(1), p->seeds.p, p->mt.p, j, false, st);
                             });
        if (ms_col_inv) *ms_col_inv = time_launches(st, reps, [&] { col_plain(p->ny, p->col_inv_args(1), j, st); });
        if (ms_row) *ms_row = time_launches(st, reps, [&] { row_fused(p->nx, p->row_args(1), j, st); });
        if (ms_col_acc) *ms_col_acc = time_launches(st, reps, [&] { col_ospr(p->ny, p->col_acc_args(1), j, st); });
        CK(cudaGetLastError());
    });
}

int hgc_ospr_plan_destroy(hgc_ospr_plan* p) {
    return guarded([&] {
        if (p) {
            cudaSetDevice(p->device);
            cudaStreamSynchronize(p->stream);
        }
        delete p;
    });
}

// Fresnel OSPR (extension): the reference rejects OSPR with a
// Fresnel propagator (src/config.cpp:443-445) and run_ospr_impl takes a bare
// FftBackend (ospr.hpp:68-69); this composes Propagator<float>::inverse /
// forward (propagation.hpp:81-95) into the subframe loop: f = IFFT(seed)
// conj(Q), quantise, R = FFT(f Q).  Before the plan's first execute.
int hgc_ospr_plan_set_fresnel(hgc_ospr_plan* p, const hgc_fresnel* fresnel) {
    return guarded([&] {
        if (!p) invalid("hgc_ospr_plan_set_fresnel: null plan");
        if (p->graph) invalid("hgc_ospr_plan_set_fresnel: call before the first execute");
        CK(cudaSetDevice(p->device));
        p->fresnel = fresnel != nullptr;
        if (!fresnel) return;
        validate_fresnel(fresnel);
        p->Q.ensure(p->npix);
        const double scale = 3.1415926535897932384626433832795 / (fresnel->wavelength * fresnel->distance);
        k_fresnel_q<<<ew_grid(p->npix), 256, 0, p->stream>>>(p->nx, p->ny, scale, fresnel->pixel_pitch_x,
                                                              fresnel->pixel_pitch_y, p->Q.p);
        CK(cudaGetLastError());
    });
}

int hgc_ospr_run_fresnel(const hgc_ospr_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny,
                         int jobs, hgc_ospr_io* io);

int hgc_ospr_run(const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny, int jobs, hgc_ospr_io* io) {
    return hgc_ospr_run_fresnel(cfg, slm, nullptr, nx, ny, jobs, io);
}

int hgc_ospr_run_fresnel(const hgc_ospr_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny,
                         int jobs, hgc_ospr_io* io) {
    auto t0 = std::chrono::steady_clock::now();
    hgc_ospr_plan* p = nullptr;
    int rc = guarded([] { route_device(); });
    if (rc == HGC_OK) rc = hgc_ospr_plan_create(&p, cfg, slm, nx, ny, jobs, io ? io->per_job_target : 0);
    if (rc == HGC_OK && fresnel) rc = hgc_ospr_plan_set_fresnel(p, fresnel);
    if (rc == HGC_OK && io && io->profile) rc = guarded([&] { p->profile_on(); });
    if (rc == HGC_OK) rc = hgc_ospr_plan_upload(p, io);
    if (rc == HGC_OK) rc = guarded([&] { check_validation(p->vflags.p, p->stream); });  // eager in the one-shot run
    if (rc == HGC_OK) rc = hgc_ospr_plan_execute(p, nullptr);
    if (rc == HGC_OK) rc = hgc_ospr_plan_download(p, io);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc == HGC_OK && io && io->profile) rc = guarded([&] { p->profile_split(secs, io->profile); });
    if (p) {
        std::string keep = g_err;
        hgc_ospr_plan_destroy(p);
        g_err = keep;
    }
    if (rc == HGC_OK && io && io->seconds) *io->seconds = secs;
    return rc;
}

}  // extern "C"
