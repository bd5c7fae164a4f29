// batch.cpp — batch executor with device routing, the B200
// counterpart of the runner's `batch` command (src/runner.cpp:365-421).
//
// The reference runs one job per host thread (up to 64), each job a full
// single-target run.  Here jobs whose configurations differ only in seed and
// target are merged into one batched plan (one launch sequence, one CUDA
// graph, many targets), and the batched groups are spread across the GPUs,
// one host thread per device, largest groups first onto the least-loaded
// device.  Per-job semantics stay those of cmd_batch: every job gets its own
// ok/failed status, message, final_error and seconds, and a job that fails
// (e.g. a non-finite target) fails alone — its group is re-run job by job.
//
// This file is a client of the C ABI only (plan API + hgc_set_device).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hologen_b200.h"

namespace {

bool same_slm(const hgc_slm& a, const hgc_slm& b) {
    return a.mode == b.mode && a.levels == b.levels && a.min_arg == b.min_arg && a.max_arg == b.max_arg &&
           a.full_circle == b.full_circle && a.min_amp == b.min_amp && a.max_amp == b.max_amp &&
           a.illumination == b.illumination;
}

// Jobs that can share one batched plan: everything but the seed and the
// target images (amplitude, phase) must agree.
bool compatible(const hgc_batch_job& a, const hgc_batch_job& b) {
    if (a.kind != b.kind || a.nx != b.nx || a.ny != b.ny || a.roi != b.roi) return false;
    if (!a.slm || !b.slm || !same_slm(*a.slm, *b.slm)) return false;
    if (a.kind == 0) {
        const hgc_ifta_cfg &x = *a.ifta, &y = *b.ifta;
        if (x.variant != y.variant || x.iterations != y.iterations || x.weight_clamp_lo != y.weight_clamp_lo ||
            x.weight_clamp_hi != y.weight_clamp_hi || x.lt_initial_fraction != y.lt_initial_fraction ||
            x.init_phase != y.init_phase || x.freedom_amplitude_outside_roi != y.freedom_amplitude_outside_roi ||
            x.freedom_phase != y.freedom_phase || x.freedom_scale != y.freedom_scale)
            return false;
        if ((a.phase == nullptr) != (b.phase == nullptr)) return false;
        if ((a.fresnel == nullptr) != (b.fresnel == nullptr)) return false;
        if (a.fresnel && std::memcmp(a.fresnel, b.fresnel, sizeof(hgc_fresnel)) != 0) return false;
        return true;
    }
    const hgc_ospr_cfg &x = *a.ospr, &y = *b.ospr;
    return x.variant == y.variant && x.subframes == y.subframes && x.feedback_gain == y.feedback_gain &&
           x.freedom_scale == y.freedom_scale;
}

double work_of(const hgc_batch_job& j) {
    const double px = (double)j.nx * j.ny;
    return j.kind == 0 ? px * (j.ifta ? j.ifta->iterations : 1) : px * (j.ospr ? j.ospr->subframes : 1);
}

void set_result(hgc_batch_job& j, int status, const char* msg, double final_error, double seconds) {
    j.status = status;
    j.final_error = final_error;
    j.seconds = seconds;
    std::snprintf(j.message, sizeof j.message, "%s", msg ? msg : "");
}

// Run a group of compatible jobs as one batched plan on the current device.
int run_group(hgc_batch_job* jobs, const std::vector<int>& idx) {
    const hgc_batch_job& j0 = jobs[idx[0]];
    const int B = (int)idx.size();
    const size_t npix = (size_t)j0.nx * j0.ny;
    std::vector<double> amp(npix * B), phase(j0.phase ? npix * B : 0);
    std::vector<uint64_t> seeds(B);
    for (int b = 0; b < B; ++b) {
        const hgc_batch_job& j = jobs[idx[b]];
        std::memcpy(amp.data() + npix * b, j.amplitude, sizeof(double) * npix);
        if (j0.phase) std::memcpy(phase.data() + npix * b, j.phase, sizeof(double) * npix);
        seeds[b] = j.kind == 0 ? j.ifta->seed : j.ospr->seed;
    }
    const bool wide = j0.slm->levels > 256;
    auto t0 = std::chrono::steady_clock::now();
    int rc = HGC_OK;
    if (j0.kind == 0) {
        const int K = j0.ifta->iterations;
        std::vector<double> trace((size_t)K * B), fe(B);
        std::vector<uint8_t> l8(wide ? 0 : npix * B);
        std::vector<uint16_t> l16(wide ? npix * B : 0);
        hgc_ifta_plan* p = nullptr;
        rc = hgc_ifta_plan_create(&p, j0.ifta, j0.slm, j0.fresnel, j0.nx, j0.ny, B);
        hgc_ifta_io io{};
        io.amplitude = amp.data();
        io.phase = j0.phase ? phase.data() : nullptr;
        io.roi = j0.roi;
        io.seeds = seeds.data();
        io.levels8 = wide ? nullptr : l8.data();
        io.levels16 = wide ? l16.data() : nullptr;
        io.trace = trace.data();
        io.final_error = fe.data();
        if (rc == HGC_OK) rc = hgc_ifta_plan_upload(p, &io);
        if (rc == HGC_OK) rc = hgc_ifta_plan_execute(p, nullptr);
        if (rc == HGC_OK) rc = hgc_ifta_plan_download(p, &io);
        const std::string msg = rc == HGC_OK ? "" : hgc_last_error();
        if (p) hgc_ifta_plan_destroy(p);
        if (rc != HGC_OK) return rc;
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int b = 0; b < B; ++b) {
            hgc_batch_job& j = jobs[idx[b]];
            if (j.levels8 && !wide) std::memcpy(j.levels8, l8.data() + npix * b, npix);
            if (j.levels16) {
                for (size_t i = 0; i < npix; ++i) j.levels16[i] = wide ? l16[npix * b + i] : l8[npix * b + i];
            }
            if (j.trace) std::memcpy(j.trace, trace.data() + (size_t)K * b, sizeof(double) * K);
            set_result(j, HGC_OK, "", fe[b], secs);
        }
        return HGC_OK;
    }
    const int N = j0.ospr->subframes;
    std::vector<double> fm((size_t)N * B), cm((size_t)N * B), fe(B);
    std::vector<uint8_t> l8(wide ? 0 : npix * N * B);
    std::vector<uint16_t> l16(wide ? npix * N * B : 0);
    hgc_ospr_plan* p = nullptr;
    rc = hgc_ospr_plan_create(&p, j0.ospr, j0.slm, j0.nx, j0.ny, B, 1);
    hgc_ospr_io io{};
    io.amplitude = amp.data();
    io.per_job_target = 1;
    io.roi = j0.roi;
    io.seeds = seeds.data();
    io.levels8 = wide ? nullptr : l8.data();
    io.levels16 = wide ? l16.data() : nullptr;
    io.frame_mse = fm.data();
    io.cumulative_mse = cm.data();
    io.final_error = fe.data();
    if (rc == HGC_OK) rc = hgc_ospr_plan_upload(p, &io);
    if (rc == HGC_OK) rc = hgc_ospr_plan_execute(p, nullptr);
    if (rc == HGC_OK) rc = hgc_ospr_plan_download(p, &io);
    if (p) hgc_ospr_plan_destroy(p);
    if (rc != HGC_OK) return rc;
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const size_t fr = npix * N;
    for (int b = 0; b < B; ++b) {
        hgc_batch_job& j = jobs[idx[b]];
        if (j.levels8 && !wide) std::memcpy(j.levels8, l8.data() + fr * b, fr);
        if (j.levels16) {
            for (size_t i = 0; i < fr; ++i) j.levels16[i] = wide ? l16[fr * b + i] : l8[fr * b + i];
        }
        if (j.trace) std::memcpy(j.trace, cm.data() + (size_t)N * b, sizeof(double) * N);
        set_result(j, HGC_OK, "", fe[b], secs);
    }
    return HGC_OK;
}

}  // namespace

extern "C" int hgc_batch_run(hgc_batch_job* jobs, int njobs, int max_devices, size_t max_group_bytes) {
    if (!jobs || njobs < 0) return HGC_EINVAL;
    // structural checks per job (the rest is the plan API's own validation)
    std::vector<int> runnable;
    for (int i = 0; i < njobs; ++i) {
        hgc_batch_job& j = jobs[i];
        set_result(j, HGC_EINVAL, "", 0.0, 0.0);
        if ((j.kind != 0 && j.kind != 1) || !j.slm || !j.amplitude || (j.kind == 0 && !j.ifta) ||
            (j.kind == 1 && !j.ospr)) {
            set_result(j, HGC_EINVAL, "hgc_batch_run: malformed job", 0.0, 0.0);
            continue;
        }
        runnable.push_back(i);
    }
    // greedy grouping in job order (cmd_batch processes jobs in sorted order)
    const size_t cap = max_group_bytes ? max_group_bytes : (size_t)16 << 30;
    std::vector<std::vector<int>> groups;
    for (int i : runnable) {
        const size_t bytes = (size_t)jobs[i].nx * jobs[i].ny * 48;  // resident bytes per target, roughly
        bool placed = false;
        for (auto& g : groups)
            if (compatible(jobs[g[0]], jobs[i]) && (g.size() + 1) * bytes <= cap) {
                g.push_back(i);
                placed = true;
                break;
            }
        if (!placed) groups.push_back({i});
    }
    int ndev = 0;
    if (hgc_device_count(&ndev) != HGC_OK || ndev < 1) {
        for (int i : runnable) set_result(jobs[i], HGC_ECUDA, "hgc_batch_run: no CUDA device", 0.0, 0.0);
        return HGC_ECUDA;
    }
    if (max_devices > 0) ndev = std::min(ndev, max_devices);
    // largest groups first onto the least-loaded device (LPT)
    std::vector<int> order(groups.size());
    for (size_t g = 0; g < groups.size(); ++g) order[g] = (int)g;
    auto gwork = [&](int g) { return work_of(jobs[groups[g][0]]) * groups[g].size(); };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return gwork(a) > gwork(b); });
    std::vector<std::vector<int>> per_dev(ndev);
    std::vector<double> load(ndev, 0.0);
    for (int g : order) {
        const int d = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        per_dev[d].push_back(g);
        load[d] += gwork(g);
    }
    std::vector<std::thread> pool;
    for (int d = 0; d < ndev; ++d) {
        if (per_dev[d].empty()) continue;
        pool.emplace_back([&, d] {
            hgc_set_device(d);
            for (int g : per_dev[d]) {
                if (run_group(jobs, groups[g]) == HGC_OK) continue;
                // isolate the failure: each job of the group alone (cmd_batch semantics)
                for (int i : groups[g]) {
                    const int rc = run_group(jobs, {i});
                    if (rc != HGC_OK) set_result(jobs[i], rc, hgc_last_error(), 0.0, 0.0);
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int i = 0; i < njobs; ++i)
        if (jobs[i].status != HGC_OK) return jobs[i].status;
    return HGC_OK;
}
