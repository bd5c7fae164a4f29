// capi.cu — library-level part of the C ABI in include/hologen_b200.h:
// version and error state, device selection and routing, the per-device
// twiddle tables, and the configuration validation shared by the plans.
// The plans and primitives live in ifta_plan.cu (run_ifta), ospr_plan.cu
// (run_ospr_impl), f64.cu (the double loops), primitives.cu (FftBackend,
// Propagator, Quantiser, seed_random_phase, mse, output encodings).
#include "capi_impl.cuh"

namespace hg {
thread_local std::string g_err;

// ------------------------------------------------------- twiddle tables
static __global__ void k_init_twiddles(float2* tw) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 1 || idx >= kTwEntries) return;
    double s, c;
    if (idx >= 2 * kMaxLine) {  // the radix-16 span-256 pass: W_256^(r k), r, k < 16 (fft.cuh kTw256)
        const int rk = idx - 2 * kMaxLine, r = rk >> 4, k = rk & 15;
        sincospi(-2.0 * (double)(r * k) / 256.0, &s, &c);
    } else {
        int N = 1;
        while (N * 2 <= idx) N *= 2;
        int m = idx - N;
        sincospi(-2.0 * (double)m / (double)N, &s, &c);
    }
    tw[idx] = make_float2((float)c, (float)s);
}

static std::mutex g_init_mu;
static std::map<int, float2*> g_tw_tables;

// Per-device one-time setup; returns the device's twiddle table.
const float2* device_twiddles() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_init_mu);
    auto it = g_tw_tables.find(dev);
    if (it != g_tw_tables.end()) return it->second;
    float2* tw = nullptr;
    CK(cudaMalloc(&tw, sizeof(float2) * kTwEntries));
    k_init_twiddles<<<(kTwEntries + 255) / 256, 256>>>(tw);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    g_tw_tables[dev] = tw;
    return tw;
}

// ---------------------------------------------------- size dispatch
}  // namespace hg

extern "C" {

int hgc_abi_version(void) { return HGC_ABI_VERSION; }
const char* hgc_last_error(void) { return g_err.c_str(); }
int hgc_max_side(void) { return kMaxLine; }

int hgc_device_count(int* count) {
    return guarded([&] { CK(cudaGetDeviceCount(count)); });
}
int hgc_set_device(int device) {
    return guarded([&] { CK(cudaSetDevice(device)); });
}

// Device routing for callers that run jobs on their own threads (the
// runner's batch pool, runner.cpp:387-421, through the C++ drop-in):
// policy 1 binds each host thread, on its first run, to the next device
// round-robin; policy 0 leaves the thread's current device alone.
static std::atomic<int> g_dev_policy{0};
static std::atomic<int> g_dev_next{0};
int hgc_set_device_policy(int policy) {
    return guarded([&] {
        if (policy != 0 && policy != 1) invalid("hgc_set_device_policy: policy must be 0 or 1");
        g_dev_policy = policy;
    });
}
extern "C++" void route_device() {
    thread_local int bound = -1;
    if (g_dev_policy.load() != 1 || bound >= 0) return;
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 1) fail(HGC_ECUDA, "no CUDA device");
    bound = g_dev_next.fetch_add(1) % n;
    CK(cudaSetDevice(bound));
}
uint64_t hgc_fork_seed(uint64_t seed, uint64_t stream) { return fork_seed(seed, stream); }

double hgc_subframe_mse_statistic(const double* v, int n) {  // ospr.hpp:58-64
    if (!v || n <= 0) {
        g_err = "subframe_mse_statistic: empty list";
        return std::nan("");
    }
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i];
    return s / std::sqrt((double)n);
}

extern "C++" void validate_ifta_cfg(const hgc_ifta_cfg* c) {  // IftaConfig::validate, ifta.hpp:41-50
    if (!c) invalid("IftaConfig: missing");
    if (c->iterations < 1) invalid("IftaConfig: iterations must be >= 1");
    if (!(c->weight_clamp_lo > 0) || !(c->weight_clamp_hi >= c->weight_clamp_lo))
        invalid("IftaConfig: weight clamp bounds invalid");
    if (!(c->lt_initial_fraction > 0) || !(c->lt_initial_fraction <= 1))
        invalid("IftaConfig: lt_initial_fraction must be in (0,1]");
    if (c->variant < 0 || c->variant > 2) invalid("IftaConfig: unknown variant");
    if (c->init_phase < 0 || c->init_phase > 3) invalid("IftaConfig: unknown init phase");
}

extern "C++" void validate_fresnel(const hgc_fresnel* p) {  // FresnelParams::validate, propagation.hpp:21-29
    if (!(p->wavelength > 0) || !std::isfinite(p->wavelength)) invalid("FresnelParams: wavelength must be positive");
    if (p->distance == 0 || !std::isfinite(p->distance)) invalid("FresnelParams: distance must be non-zero");
    if (!(p->pixel_pitch_x > 0) || !(p->pixel_pitch_y > 0) || !std::isfinite(p->pixel_pitch_x) ||
        !std::isfinite(p->pixel_pitch_y))
        invalid("FresnelParams: pixel pitches must be positive");
}

extern "C++" void validate_ospr_cfg(const hgc_ospr_cfg* c) {  // OsprConfig::validate, ospr.hpp:30-37
    if (!c) invalid("OsprConfig: missing");
    if (c->subframes < 1) invalid("OsprConfig: subframes must be >= 1");
    if (!(c->feedback_gain >= 0.0 && c->feedback_gain <= 1.0)) invalid("OsprConfig: feedback_gain must be in [0,1]");
    if (c->variant < 0 || c->variant > 1) invalid("OsprConfig: unknown variant");
}

}  // extern "C"
