// capi.cu — host side of the B200 HoloGen hot path behind the C ABI in
// include/hologen_b200.h.  Owns device memory, builds the fused pass
// sequence of run_ifta / run_ospr_impl as one CUDA graph per plan, and maps
// errors to the reference's exception semantics (status + message).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hologen_b200.h"
#include "errors.h"
#include "launch.h"
#include "mt64.cuh"
#include "f64path.cuh"
#include "mtjump.h"
#include "passes.cuh"

namespace hg {


// ------------------------------------------------------------------ errors
thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return HGC_OK;
    } catch (const Failure& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return HGC_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HGC_ECUDA;
    }
}

// ---------------------------------------------------------- device memory
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { reset(); }
    void alloc(size_t count) {
        reset();
        if (count == 0) return;
        CK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // Allocate unless already holding exactly `count` elements (keeps device
    // pointers stable across uploads so a captured graph stays valid).
    void ensure(size_t count) {
        if (n != count) alloc(count);
    }
};

// ------------------------------------------------------- twiddle tables
// tw[N + m] = exp(-2*pi*i*m/N) for N = 1..4096 (fft.cuh), in double then
// rounded to float, one table per device.
__global__ void k_init_twiddles(float2* tw) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 1 || idx >= 2 * kMaxLine) return;
    int N = 1;
    while (N * 2 <= idx) N *= 2;
    int m = idx - N;
    double s, c;
    sincospi(-2.0 * (double)m / (double)N, &s, &c);
    tw[idx] = make_float2((float)c, (float)s);
}

static std::mutex g_init_mu;
static std::map<int, float2*> g_tw_tables;

// Per-device one-time setup; returns the device's twiddle table.
static const float2* device_twiddles() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_init_mu);
    auto it = g_tw_tables.find(dev);
    if (it != g_tw_tables.end()) return it->second;
    float2* tw = nullptr;
    CK(cudaMalloc(&tw, sizeof(float2) * 2 * kMaxLine));
    k_init_twiddles<<<(2 * kMaxLine + 255) / 256, 256>>>(tw);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    g_tw_tables[dev] = tw;
    return tw;
}

// ---------------------------------------------------- size dispatch
static bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
static void check_size(int nx, int ny) {
    if (nx <= 0 || ny <= 0) invalid("ComplexField: dimensions must be positive");
    if (!is_pow2(nx) || !is_pow2(ny) || nx > kMaxLine || ny > kMaxLine || nx < 2 || ny < 2)
        fail(HGC_EUNSUPPORTED, "hologen_b200: field " + std::to_string(nx) + "x" + std::to_string(ny) +
                                   " unsupported (GPU path: powers of two, 2..4096 per side)");
}

static void prepare_kernels(int nx, int ny) {
    RowArgs ra{};
    ColArgs ca{};
    ca.nx = nx;
    ra.layout = LAY_QUAD;
    row_fused(nx, ra, 1, nullptr, true);
    ra.layout = LAY_ROW;
    row_plain(nx, ra, 1, nullptr, true);
    col_plain(ny, ca, 1, nullptr, true);
    ca.layout = LAY_QUAD;
    col_gs(ny, ca, 1, nullptr, true);
    col_ospr(ny, ca, 1, nullptr, true);
    CK(cudaFuncSetAttribute(k_seed_random_phase<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSeedSmem));
    CK(cudaFuncSetAttribute(k_seed_random_phase<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSeedSmem));
}

// ------------------------------------------------ TMA tensor maps
// A quad-layout complex64 region seen as a 2-D float tensor: inner = one quad
// row (4*nx floats = two field rows), outer = `rows` quad rows; box = one
// column pair (8 floats = 32 B) x 256 quad rows.  The map lives in device
// memory (ColArgs::tmap).  cuTensorMapEncodeTiled comes from the driver entry
// point so cudart stays statically linked.
struct DevTensorMap {
    DBuf<CUtensorMap> d;
    void make(float2* base, int nx, int C, size_t rows) {  // C: columns per column-pass tile
        static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) fail(HGC_ECUDA, "cuTensorMapEncodeTiled unavailable");
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }();
        CUtensorMap m;
        const cuuint64_t dims[2] = {(cuuint64_t)4 * nx, (cuuint64_t)rows};
        const cuuint64_t strides[1] = {(cuuint64_t)4 * nx * sizeof(float)};
        const cuuint32_t box[2] = {(cuuint32_t)(4 * C), 256};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(HGC_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        d.alloc(1);
        CK(cudaMemcpy(d.p, &m, sizeof m, cudaMemcpyHostToDevice));
    }
};

// ------------------------------------------ RNG chunking (jump-ahead)
// One reference stream split across several CTAs: CTA (stream s, chunk c)
// starts at draw offset0 + c*len, its state set by k_mt_jump from the
// polynomials of mtjump.cpp (computed once per process per shape).  Enough
// chunks that streams*chunks fills the GPU twice, none shorter than
// kMinChunkDraws (the jump costs about as much as ~30k draws).
constexpr size_t kMinChunkDraws = 32768;
constexpr int kMaxChunks = 512;
// The seed kernel instantiation for a launch: the fast consumer loop when the
// output is the plans' float quad layout with a plain amplitude.
#ifndef HG_SEED_FAST
#define HG_SEED_FAST 1
#endif
static void seed_launch(int grid, const SeedArgs& sa, cudaStream_t st) {
    if (HG_SEED_FAST && sa.quad && sa.out && !sa.out64 && !sa.S && sa.nx >= 2)
        k_seed_random_phase<true><<<grid, kSeedThreads, kSeedSmem, st>>>(sa);
    else
        k_seed_random_phase<false><<<grid, kSeedThreads, kSeedSmem, st>>>(sa);
    CK(cudaGetLastError());
}

struct SeedChunks {
    int chunks = 1;
    size_t len = 0;
    uint64_t offset0 = 0;
    DBuf<int> starts;       // jump polynomials as set-bit offsets (mt_poly_offsets)
    DBuf<uint16_t> pool;

    static void upload_offsets(const uint64_t* polys, int n, DBuf<int>& st, DBuf<uint16_t>& pl) {
        std::vector<int> s;
        std::vector<uint16_t> p;
        mt_poly_offsets(polys, n, s, p);
        st.alloc(s.size());
        pl.alloc(std::max<size_t>(p.size(), 1));
        CK(cudaMemcpy(st.p, s.data(), sizeof(int) * s.size(), cudaMemcpyHostToDevice));
        if (!p.empty()) CK(cudaMemcpy(pl.p, p.data(), sizeof(uint16_t) * p.size(), cudaMemcpyHostToDevice));
    }

    void plan(size_t npix, int streams, uint64_t offset = 0, int ctas_per_sm = 2) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // enough chunks to fill every slot; among up to 4x that, the count
        // whose last wave is fullest (ties: fewer chunks, fewer jumps)
        const long long slots = (long long)ctas_per_sm * sms, S = std::max(1, streams);
        const long long cmax = std::max<long long>(1, (long long)(npix / kMinChunkDraws));
        long long c = std::min((slots + S - 1) / S, cmax);
        double best = 0.0;
        for (long long k = c, hi = std::min(4 * c, cmax); k <= hi; ++k) {
            const long long ctas = S * k, waves = (ctas + slots - 1) / slots;
            const double eff = (double)ctas / (double)(waves * slots);
            if (eff > best + 0.02) best = eff, c = k;
        }
        if (const char* ev = getenv("HG_SEED_CHUNKS")) c = std::max(1, atoi(ev));  // tuning / tests
        c = std::min<long long>(c, (long long)std::max<size_t>(1, npix));
        c = std::max<long long>(1, std::min<long long>(c, kMaxChunks));
        len = (npix + c - 1) / c;
        chunks = (int)((npix + len - 1) / len);
        offset0 = offset;
        starts.reset();
        pool.reset();
        if (jumps()) {
            const std::vector<uint64_t>& v = mt_chunk_polys(offset0, len, chunks);
            upload_offsets(v.data(), (int)(v.size() / kMtPolyWords), starts, pool);
        }
    }
    int c_first() const { return offset0 == 0 ? 1 : 0; }
    bool jumps() const { return chunks > c_first(); }
    // One-shot stream (IFTA init, seed_random_phase, pre-seeded OSPR): jump
    // (when needed) + chunked seed; `seeds` are engine seeds (already
    // forked), `states` holds streams*chunks entries.  Returns the number of
    // launches.
    int launch(SeedArgs sa, const uint64_t* seeds, MtState* states, int streams, cudaStream_t st) const {
        int n = 0;
        if (jumps()) {
            JumpArgs ja{seeds, nullptr, starts.p, pool.p, 1, states, chunks, c_first(), c_first()};
            k_mt_jump<<<streams * (chunks - c_first()), kJumpThreads, 0, st>>>(ja);
            ++n;
        }
        sa.states = states;
        sa.seeds = offset0 == 0 ? seeds : nullptr;
        sa.chunks = chunks;
        sa.chunk_len = len;
        seed_launch(streams * chunks, sa, st);
        return n + 1;
    }

    // Continued stream (adaptive OSPR: subframe n draws [(n-1)*npix, n*npix)).
    // With chunks > 1, states[] holds each chunk's start window; subframe 1
    // jumps from the seeds, later subframes move every start window by npix
    // draws in place (one polynomial, x^(npix-1)).
    DBuf<int> step_starts;
    DBuf<uint16_t> step_pool;
    void plan_stream(size_t npix, int streams, uint64_t offset = 0) {
        plan(npix, streams, offset, 1);  // a per-frame jump per chunk: split only below one CTA per SM
        step_starts.reset();
        step_pool.reset();
        if (chunks > 1) {
            std::vector<uint64_t> g(kMtPolyWords);
            mt_jump_poly(npix - 1, g.data());
            upload_offsets(g.data(), 1, step_starts, step_pool);
        }
    }
    int launch_stream(SeedArgs sa, const uint64_t* seeds, MtState* states, int streams, bool first,
                      cudaStream_t st) const {
        sa.states = states;
        if (chunks == 1) {
            int n = 0;
            if (first && offset0 > 0) {  // stream starts offset0 draws in (subframe block)
                JumpArgs ja{seeds, nullptr, starts.p, pool.p, 1, states, 1, 0, 0};
                k_mt_jump<<<streams, kJumpThreads, 0, st>>>(ja);
                ++n;
            }
            sa.seeds = first && offset0 == 0 ? seeds : nullptr;
            seed_launch(streams, sa, st);
            return n + 1;
        }
        JumpArgs ja = first ? JumpArgs{seeds, nullptr, starts.p, pool.p, 1, states, chunks, 0, c_first()}
                            : JumpArgs{nullptr, states, step_starts.p, step_pool.p, 0, states, chunks, 0, 0};
        k_mt_jump<<<streams * chunks, kJumpThreads, 0, st>>>(ja);
        sa.seeds = nullptr;
        sa.chunks = chunks;
        sa.chunk_len = len;
        sa.no_save = 1;
        seed_launch(streams * chunks, sa, st);
        return 2;
    }
};

// ------------------------------------------------------- small kernels
__global__ void k_fill_c(float2* p, size_t n, float2 v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_f(float* p, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_d2f(const double* a, float* o, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        o[i] = (float)a[i];
}
// Row-major (host order) <-> resident layouts (passes.cuh): one thread per
// element of a batch of nx x ny images.
struct Pix {
    size_t b, i;  // batch index, row-major pixel index
    int x, y;
};
__device__ __forceinline__ Pix pix_of(size_t g, int nx, size_t npix) {
    Pix p;
    p.b = g / npix;
    p.i = g % npix;
    p.y = (int)(p.i / nx);
    p.x = (int)(p.i % nx);
    return p;
}
#define HG_GRID_LOOP(g, n) \
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < (n); g += (size_t)gridDim.x * blockDim.x)

template <class TI, class TO>
__global__ void k_to_colpair(const TI* in, TO* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[p.b * npix + colpair_index(p.x, p.y, ny)] = (TO)in[g];
    }
}
template <class T>
__global__ void k_from_colpair(const T* in, T* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[g] = in[p.b * npix + colpair_index(p.x, p.y, ny)];
    }
}
// Row-major -> column-pair major through a 32-row x 64-column smem tile, so
// both the reads (rows) and the writes (64 contiguous outputs per column pair)
// are coalesced.  Requires nx % 64 == 0 and ny % 32 == 0.
template <class TI, class TO>
__global__ void __launch_bounds__(256) k_to_colpair_tiled(const TI* in, TO* out, int nx, int ny) {
    __shared__ TO tile[32][65];
    const int x0 = blockIdx.x * 64, y0 = blockIdx.y * 32;
    const size_t base = (size_t)blockIdx.z * nx * ny;
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int r = tid / 64 + 4 * k, c = tid % 64;
        tile[r][c] = (TO)in[base + (size_t)(y0 + r) * nx + x0 + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int idx = tid + 256 * k, pair = idx / 64, w = idx % 64;
        const int y = w >> 1, xl = 2 * pair + (w & 1);
        out[base + colpair_index(x0 + xl, y0 + y, ny)] = tile[y][xl];
    }
}

__global__ void k_to_quad(const float2* in, float2* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[p.b * npix + quad_index(p.x, p.y, nx)] = in[g];
    }
}
__global__ void k_from_quad(const float2* in, float2* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[g] = in[p.b * npix + quad_index(p.x, p.y, nx)];
    }
}
// InitPhase::Flat, ifta.hpp:128-130 (quad output)
__global__ void k_init_flat(const double* a, float2* f, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        f[p.b * npix + quad_index(p.x, p.y, nx)] = make_float2((float)a[g], 0.f);
    }
}
// target-phase init, ifta.hpp:131-136 (tphase = 2*pi*turns, ifta.hpp:107-111) (quad output)
__global__ void k_init_target_phase(const double* a, const double* turns, float2* f, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        double ph = __dmul_rn(HG_TWO_PI, turns[g]);
        double s, c;
        sincos(ph, &s, &c);
        f[p.b * npix + quad_index(p.x, p.y, nx)] =
            make_float2((float)__dmul_rn(a[g], c), (float)__dmul_rn(a[g], s));
    }
}
// (cos, sin) of the target phase for the no-phase-freedom constraint
// (ifta.hpp:215-219), column-pair major
__global__ void k_phase_cs(const double* turns, float2* cs, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        double s, c;
        sincos(__dmul_rn(HG_TWO_PI, turns[g]), &s, &c);
        cs[p.b * npix + colpair_index(p.x, p.y, ny)] = make_float2((float)c, (float)s);
    }
}
// make_fresnel_phase<float>, propagation.hpp:36-54 (no FMA contraction)
__global__ void k_fresnel_q(int nx, int ny, double scale, double px, double py, float2* q) {
    size_t n = (size_t)nx * ny;
    const double cx = nx / 2.0, cy = ny / 2.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        int y = (int)(i / nx), x = (int)(i % nx);
        double dy = __dmul_rn(__dsub_rn((double)y, cy), py);
        double ty = __dmul_rn(dy, dy);
        double dx = __dmul_rn(__dsub_rn((double)x, cx), px);
        double ph = __dmul_rn(scale, __dadd_rn(__dmul_rn(dx, dx), ty));
        double s, c;
        sincos(ph, &s, &c);
        q[i] = make_float2((float)c, (float)s);
    }
}
// Quantiser::apply over a batch (primitive entry point)
__global__ void k_quantise(float2* f, int32_t* lv, size_t npix, size_t total, QuantParams q) {
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        size_t i = g % npix;
        float2 v = f[g];
        int k = quant_decide(q, v.x, v.y, i);
        f[g] = quant_state(q, k, i);
        if (lv) lv[g] = k;
    }
}
// mse partials in double (primitive): sum (T-r)^2, T r, r^2, T^2, count
__global__ void k_mse_partials(const double* t, const float2* r, const uint8_t* m, size_t n, double* out) {
    double acc[5] = {0, 0, 0, 0, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (m && m[i] == 0) continue;
        double re = r[i].x, im = r[i].y;
        double rr = __dsqrt_rn(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
        double d = __dsub_rn(t[i], rr);
        acc[0] += d * d;
        acc[1] += t[i] * rr;
        acc[2] += rr * rr;
        acc[3] += t[i] * t[i];
        acc[4] += 1.0;
    }
    block_sum_store<5>(acc, out + blockIdx.x * 5);
}

// Deterministic per-(target, iteration) reduction of the column-pass
// partials into MSE values (metrics.hpp:70-124; scale-free gain :213-225).
// partials: [slots][targets][tiles][8]; out: [targets][slots][nout]
// Per-target traces from the column-pass partial sums.  GS (ospr == 0): the
// mse (metrics.hpp:70-97, :123) with sum T^2 from stt[target] (scale-free
// only), and, when eff != nullptr, the diffraction efficiency of the last
// iteration's replay: power on the target's support (slot 3) over the total
// replay power (slot 4).  OSPR: frame and cumulative mse.
__global__ void k_finalize(const double* part, int slots, int targets, int tiles, double M, int scale_free,
                           int ospr, double* out, const double* stt = nullptr, double* eff = nullptr) {
    const int b = blockIdx.x, lane = threadIdx.x;
    for (int k = 0; k < slots; ++k) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const double* p = part + ((size_t)k * targets + b) * (size_t)tiles * 8;
        for (int j = lane; j < tiles; j += 32)
#pragma unroll
            for (int v = 0; v < 8; ++v) acc[v] += p[(size_t)j * 8 + v];
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[v] = warp_sum(acc[v]);
        if (lane == 0) {
            auto mse_of = [&](double sdd, double str, double srr, double stt) {
                if (!scale_free) return sdd / M;
                double g = srr > 0.0 ? str / srr : 0.0;
                if (g < 0.0) g = 0.0;
                double v = stt - 2.0 * g * str + g * g * srr;
                return (v < 0.0 ? 0.0 : v) / M;
            };
            if (!ospr) {
                out[(size_t)b * slots + k] = mse_of(acc[0], acc[1], acc[2], stt ? stt[b] : 0.0);
                if (eff && k == slots - 1) eff[b] = acc[4] > 0.0 ? acc[3] / acc[4] : 0.0;  // the last iteration
            } else {
                out[((size_t)b * slots + k) * 2 + 0] = mse_of(acc[0], acc[1], acc[2], acc[3]);
                out[((size_t)b * slots + k) * 2 + 1] = mse_of(acc[4], acc[5], acc[6], acc[3]);
            }
        }
    }
}

// Subframe-block OSPR, after the all-gather of every block's
// intensity sum: cumulative-MSE partials of local frame n (global frame
// first+n+1) from S = (sum of the earlier blocks) + local snapshot n, with the
// per-pixel float math of COL_OSPR (passes.cuh; ospr.hpp:134-145).  Frame-0
// CTAs also store the job total into S (mean intensity, ospr.hpp:149-156).
__global__ void __launch_bounds__(256) k_ospr_block_cum(const float* gathered, int index, int nblocks,
                                                        const float* snaps, const float* target, const uint8_t* roi,
                                                        size_t npix, int first, float* S, double* partials) {
    const int n = blockIdx.y;
    const float inv_n = 1.0f / (float)(first + n + 1);
    float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float* sn = snaps + (size_t)n * npix;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x) {
        float pre = 0.f;
        for (int h = 0; h < index; ++h) pre += gathered[(size_t)h * npix + i];
        const float sv = pre + sn[i];
        const float m = (!roi || roi[i]) ? 1.f : 0.f;
        const float amp = target[i] * m;
        const float rc = sqrtf(sv * inv_n) * m;
        const float dc = amp - rc;
        acc[3] = fmaf(amp, amp, acc[3]);
        acc[4] = fmaf(dc, dc, acc[4]);
        acc[5] = fmaf(amp, rc, acc[5]);
        acc[6] = fmaf(rc, rc, acc[6]);
        if (n == 0) {
            float tot = pre;
            for (int h = index; h < nblocks; ++h) tot += gathered[(size_t)h * npix + i];
            S[i] = tot;
        }
    }
    block_sum_float_store<7>(acc, partials + ((size_t)n * gridDim.x + blockIdx.x) * 8);
}

// ------------------------------------- output encodings
// write_hologram_png's pixels (io.cpp:272-287) from the resident levels via
// a host-built table lround(255 k / (L-1)).
__global__ void k_levels_gray8(const uint8_t* lv8, const uint16_t* lv16, size_t n, const uint8_t* table,
                               uint8_t* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = table[lv8 ? lv8[i] : lv16[i]];
}

// 2-level SLMs: levels as bit-planes (bit i & 7 of byte i >> 3), 8 pixels per byte.
__global__ void k_pack_levels1(const uint8_t* lv8, size_t nbytes, uint8_t* out) {
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < nbytes; j += (size_t)gridDim.x * blockDim.x) {
        const uint2 w = *reinterpret_cast<const uint2*>(lv8 + 8 * j);  // 8 levels, each 0 or 1
        const uint64_t v = ((uint64_t)w.y << 32) | w.x;
        uint8_t b = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) b |= (uint8_t)(((v >> (8 * k)) & 1) << k);
        out[j] = b;
    }
}

// |z| in double exactly as std::abs(std::complex<double>) (io.cpp:193-195)
// computes it on the reference's host: glibc's hypot, i.e. Borges' corrected
// algorithm ("An Improved Algorithm for hypot(a,b)", arXiv:1904.09481;
// glibc >= 2.35, non-FMA build).  It is not always correctly rounded
// (~0.6% of float pairs are 1 ulp off), so the same operation sequence is
// replayed here, without FMA contraction; checked bit-for-bit against this
// image's glibc on 3e7 float pairs.
__device__ __forceinline__ double ref_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

// Source of the replay amplitude of target/job b at row-major pixel i.
struct AmpSrc {
    int kind;             // 0: complex field, quad layout; 1: OSPR replay (T)sqrt(S/N), S column-pair major;
                          // 2: complex field, row-major
    const float2* f;
    const float* S;
    double N;
    int nx, ny;
    size_t bstride;
    __device__ __forceinline__ double amp(int b, size_t i) const {
        const int x = (int)(i % nx), y = (int)(i / nx);
        if (kind == 1) {  // ospr.hpp:149-156: replay = (T)sqrt(S/N) + 0i
            const float re = (float)sqrt((double)S[bstride * b + colpair_index(x, y, ny)] / N);
            return fabs((double)re);
        }
        const float2 z = f[bstride * b + (kind == 0 ? quad_index(x, y, nx) : i)];
        return ref_hypot((double)z.x, (double)z.y);
    }
};

// write_replay_png (io.cpp:189-205): peak = max |z| per target (block maxima,
// then one warp per target), px = clamp(lround(amp * 255/peak)), 0 when peak == 0.
__global__ void k_amp_peak(AmpSrc src, size_t npix, double* block_max) {
    const int b = blockIdx.y;
    double m = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x)
        m = fmax(m, src.amp(b, i));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) block_max[(size_t)b * gridDim.x + blockIdx.x] = m;
    }
}
__global__ void k_peak_final(const double* block_max, int nblk, double* peak) {
    const int b = blockIdx.x;
    double m = 0.0;
    for (int j = threadIdx.x; j < nblk; j += 32) m = fmax(m, block_max[(size_t)b * nblk + j]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) peak[b] = m;
}
__global__ void k_amp_gray8(AmpSrc src, size_t npix, const double* peak, uint8_t* out) {
    const int b = blockIdx.y;
    const double pk = peak[b];
    const double s = pk > 0.0 ? 255.0 / pk : 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x) {
        uint8_t v = 0;
        if (pk > 0.0) {
            const long long g = llround(src.amp(b, i) * s);
            v = (uint8_t)(g < 0 ? 0 : g > 255 ? 255 : g);
        }
        out[(size_t)b * npix + i] = v;
    }
}

// TargetSpec::validate on the device (target.hpp:52-73): bit 0 = non-finite
// amplitude, bit 1 = negative amplitude, bit 2 = non-finite phase.
// sum T^2 over the mask per target (metrics.hpp:91-97, the scale-free MSE's
// target energy), once per upload: [targets] doubles, fixed-order tree.
__global__ void __launch_bounds__(256) k_target_energy(const double* amp, const uint8_t* roi_rm, size_t npix,
                                                      double* stt) {
    const double* a = amp + npix * blockIdx.x;
    double s = 0.0;
    for (size_t i = threadIdx.x; i < npix; i += blockDim.x)
        if (!roi_rm || roi_rm[i]) s += a[i] * a[i];
    __shared__ double red[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
        x = warp_sum(x);
        if (threadIdx.x == 0) stt[blockIdx.x] = x;
    }
}

__global__ void k_validate(const double* amp, const double* phase, size_t n, int* flags) {
    int f = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double a = amp[i];
        if (!isfinite(a)) f |= 1;
        else if (a < 0) f |= 2;
        if (phase && !isfinite(phase[i])) f |= 4;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

static dim3 ew_grid(size_t n) {
    size_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return dim3((unsigned)b);
}

// (b: the plan's persistent buffer — a per-call cudaFree would synchronise the
// whole device and stall other plans running concurrently)
static void levels1_dev(const uint8_t* lv8, size_t n, int levels, uint8_t* host_out, DBuf<uint8_t>& b,
                        cudaStream_t st) {
    if (levels != 2) invalid("levels1: bit-planes need a 2-level SLM");
    if (n % 8) invalid("levels1: pixel count must be a multiple of 8");
    b.ensure(n / 8);
    k_pack_levels1<<<ew_grid(n / 8), 256, 0, st>>>(lv8, n / 8, b.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(host_out, b.p, n / 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

template <class TI, class TO>
static void to_colpair(const TI* in, TO* out, int nx, int ny, size_t batch, cudaStream_t st) {
    if (nx % 64 == 0 && ny % 32 == 0 && batch <= 65535) {
        k_to_colpair_tiled<TI, TO><<<dim3(nx / 64, ny / 32, (unsigned)batch), 256, 0, st>>>(in, out, nx, ny);
    } else {
        const size_t tot = (size_t)nx * ny * batch;
        k_to_colpair<TI, TO><<<ew_grid(tot), 256, 0, st>>>(in, out, nx, ny, tot);
    }
    CK(cudaGetLastError());
}

// ---------------------------------------------------------- validation
static const double kTwoPi = 6.283185307179586476925286766559;

static void require_finite_img(const double* p, size_t n, const char* what) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) invalid(std::string(what) + ": image contains non-finite values");
}

// SlmSpec::validate, quantise.hpp:71-96
static void validate_slm(const hgc_slm* s, size_t npix) {
    if (!s) invalid("SlmSpec: missing");
    if (s->levels < 2) invalid("SlmSpec: levels must be >= 2");
    if (s->mode == 1) {
        if (!std::isfinite(s->min_arg) || !std::isfinite(s->max_arg)) invalid("SlmSpec: phase range must be finite");
        if (!(s->min_arg < s->max_arg) || s->max_arg - s->min_arg > kTwoPi * (1 + 1e-12))
            invalid("SlmSpec: phase range must satisfy min_arg < max_arg <= min_arg + 2*pi");
        if (s->full_circle && std::abs((s->max_arg - s->min_arg) - kTwoPi) > 1e-9)
            invalid("SlmSpec: full_circle requires a 2*pi range");
    } else if (s->mode == 0) {
        if (!std::isfinite(s->min_amp) || !std::isfinite(s->max_amp)) invalid("SlmSpec: amplitude range must be finite");
        if (!(s->min_amp >= 0) || !(s->min_amp < s->max_amp)) invalid("SlmSpec: need 0 <= min_amp < max_amp");
    } else {
        invalid("SlmSpec: unknown mode");
    }
    if (s->illumination)
        for (size_t i = 0; i < npix; ++i) {
            double re = s->illumination[2 * i], im = s->illumination[2 * i + 1];
            if (!std::isfinite(re) || !std::isfinite(im)) invalid("SlmSpec: illumination must be finite");
            if (re == 0.0 && im == 0.0) invalid("SlmSpec: illumination must be nowhere zero");
        }
    if (s->levels > 65536) fail(HGC_EUNSUPPORTED, "SlmSpec: more than 65536 levels unsupported on the GPU path");
}

// TargetSpec::validate, target.hpp:52-73, for a batch already copied to the
// device (amplitude + optional phase), and the shared roi on the host.
// Returns the roi coverage M (npix without roi).
// TargetSpec::validate (target.hpp:52-73) for the plan API, asynchronous: the
// amplitude / phase scan runs on the device at upload and its flags are
// raised by the next download (or right away by the one-shot hgc_*_run).
static void launch_validate(const double* d_amp, const double* d_phase, size_t total, int* flags, cudaStream_t st) {
    CK(cudaMemsetAsync(flags, 0, sizeof(int), st));
    k_validate<<<ew_grid(total), 256, 0, st>>>(d_amp, d_phase, total, flags);
    CK(cudaGetLastError());
}
static void raise_validation(int h) {
    if (h & 1) invalid("TargetSpec.amplitude: image contains non-finite values");
    if (h & 2) invalid("TargetSpec: amplitude must be non-negative");
    if (h & 4) invalid("TargetSpec.phase: image contains non-finite values");
}
static void check_validation(const int* flags, cudaStream_t st) {
    int h = 0;
    CK(cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    raise_validation(h);
}
static size_t roi_count(const uint8_t* roi, size_t npix) {
    if (!roi) return npix;
    size_t m = 0;
    for (size_t i = 0; i < npix; ++i) m += roi[i] != 0;
    if (m == 0) invalid("TargetSpec: roi covers no pixels");
    return m;
}

// Device encodings of resident results, enqueued on `st`;
// the caller copies `d_out` / `d_peak` back.
static void replay_gray8_dev(const AmpSrc& src, size_t npix, int batch, uint8_t* d_out, double* d_peak,
                             cudaStream_t st) {
    const int nblk = (int)std::min<size_t>(148 * 2, (npix + 255) / 256);
    DBuf<double> bm;
    bm.alloc((size_t)nblk * batch);
    k_amp_peak<<<dim3(nblk, batch), 256, 0, st>>>(src, npix, bm.p);
    k_peak_final<<<batch, 32, 0, st>>>(bm.p, nblk, d_peak);
    k_amp_gray8<<<dim3(nblk, batch), 256, 0, st>>>(src, npix, d_peak, d_out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));  // bm is freed on return
}
static void levels_gray8_dev(const uint8_t* lv8, const uint16_t* lv16, size_t n, int levels, uint8_t* d_out,
                             cudaStream_t st) {
    if (levels < 2 || levels > 256)
        invalid("write_hologram_png: level count must be in [2, 256] for a lossless 8-bit encoding");
    uint8_t table[256];
    for (int k = 0; k < levels; ++k) table[k] = (uint8_t)std::lround(255.0 * k / (levels - 1));
    DBuf<uint8_t> t;
    t.alloc(256);
    CK(cudaMemcpyAsync(t.p, table, 256, cudaMemcpyHostToDevice, st));
    k_levels_gray8<<<ew_grid(n), 256, 0, st>>>(lv8, lv16, n, t.p, d_out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

// --------------------------------------------------------- quantiser state
struct QuantDev {
    QuantParams p{};
    DBuf<float2> states, illum, illum_unit;
    DBuf<double> illum_arg;
    std::vector<float2> h_states, h_illum, h_illum_unit;  // for host-side state_value
    int mode = 1;
};

// Quantiser ctor, quantise.hpp:139-166 (host arithmetic identical to the reference)
static void build_quant(const hgc_slm* s, int nx, int ny, QuantDev& q) {
    const size_t npix = (size_t)nx * ny;
    const int L = s->levels;
    double spac = s->mode == 1 ? (s->full_circle ? kTwoPi / L : (s->max_arg - s->min_arg) / (L - 1))
                               : (s->max_amp - s->min_amp) / (L - 1);
    double inv = 1.0 / spac;
    double range = s->mode == 1 ? s->max_arg - s->min_arg : 0.0;
    q.mode = s->mode;
    q.h_states.resize(L);
    for (int k = 0; k < L; ++k) {
        if (s->mode == 1) {
            double a = s->min_arg + k * spac;
            q.h_states[k] = make_float2((float)std::cos(a), (float)std::sin(a));
        } else {
            q.h_states[k] = make_float2((float)(s->min_amp + k * spac), 0.f);
        }
    }
    q.states.alloc(L);
    CK(cudaMemcpy(q.states.p, q.h_states.data(), sizeof(float2) * L, cudaMemcpyHostToDevice));
    QuantParams& p = q.p;
    p.mode = s->mode;
    p.levels = L;
    p.full_circle = s->full_circle ? 1 : 0;
    p.min_arg = s->min_arg;
    p.inv_spac = inv;
    p.range = range;
    p.min_amp = s->min_amp;
    p.min_arg_f = (float)s->min_arg;
    p.inv_spac_f = (float)inv;
    p.range_f = (float)range;
    p.min_amp_f = (float)s->min_amp;
    p.wshed_f = (float)(3.1415926535897932384626433832795 + range / 2.0);
    p.margin_rad = 1e-5f;
    p.margin_u = (float)(1e-5 * inv + L * 4e-7 + 1e-6);
    p.states = q.states.p;
    p.s0 = q.h_states[0];
    p.s1 = q.h_states[L > 1 ? 1 : 0];
    if (s->illumination) {
        std::vector<double> arg(npix);
        q.h_illum.resize(npix);
        q.h_illum_unit.resize(npix);
        for (size_t i = 0; i < npix; ++i) {
            double re = s->illumination[2 * i], im = s->illumination[2 * i + 1];
            double a = std::hypot(re, im);  // std::abs(complex<double>)
            arg[i] = std::atan2(im, re);
            q.h_illum_unit[i] = make_float2((float)(re / a), (float)(im / a));
            q.h_illum[i] = make_float2((float)re, (float)im);
        }
        q.illum_arg.alloc(npix);
        CK(cudaMemcpy(q.illum_arg.p, arg.data(), sizeof(double) * npix, cudaMemcpyHostToDevice));
        p.illum_arg = q.illum_arg.p;
        if (s->mode == 1) {
            q.illum.alloc(npix);
            CK(cudaMemcpy(q.illum.p, q.h_illum.data(), sizeof(float2) * npix, cudaMemcpyHostToDevice));
            p.illum = q.illum.p;
        } else {
            q.illum_unit.alloc(npix);
            CK(cudaMemcpy(q.illum_unit.p, q.h_illum_unit.data(), sizeof(float2) * npix, cudaMemcpyHostToDevice));
            p.illum_unit = q.illum_unit.p;
            p.illum_arg = nullptr;  // amplitude mode ignores the illumination phase in decide()
        }
    }
}

// complex<float> product as GCC evaluates it (host, no FMA): reference state_value
static inline float2 hcmul(float2 a, float2 b) {
    volatile float ac = a.x * b.x, bd = a.y * b.y, ad = a.x * b.y, bc = a.y * b.x;
    return make_float2(ac - bd, ad + bc);
}
static void levels_to_states(const QuantDev& q, const uint16_t* lv16, const uint8_t* lv8, size_t npix, size_t total,
                             float* out) {
    for (size_t g = 0; g < total; ++g) {
        int k = lv16 ? lv16[g] : lv8[g];
        size_t i = g % npix;
        float2 s = q.h_states[k];
        if (q.mode == 1 && !q.h_illum.empty()) s = hcmul(q.h_illum[i], s);
        if (q.mode == 0 && !q.h_illum_unit.empty()) s = hcmul(q.h_illum_unit[i], s);
        out[2 * g] = s.x;
        out[2 * g + 1] = s.y;
    }
}

}  // namespace hg

using namespace hg;

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
    DBuf<double> amp_d, phase_d, partials, trace, stt, eff;  // stt: sum T^2 per target; eff: efficiency trace
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
struct PhaseClock {
    cudaStream_t st = nullptr;
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> ph;
    PhaseClock(cudaStream_t s, bool enable) : st(s), on(enable) {
        if (on) mark(3);
    }
    ~PhaseClock() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    void mark(int phase) {  // closes the interval since the previous mark
        if (!on) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, st));
        ev.push_back(e);
        ph.push_back(phase);
    }
    // (after the stream is synchronised) out = {transform, constraint, metric,
    // other} with other = seconds - the rest, as ifta.hpp:231-233 does.
    void report(double seconds, double* out) const {
        double t[4] = {0, 0, 0, 0};
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
            t[ph[i]] += 1e-3 * ms;
        }
        const double counted = t[0] + t[1] + t[2];
        const double sc = counted > seconds && counted > 0 ? seconds / counted : 1.0;
        for (int i = 0; i < 3; ++i) out[i] = t[i] * sc;
        out[3] = std::max(0.0, seconds - counted * sc);
    }
};

// Average device time (ms) of `reps` launches of f on stream st.
template <class F>
static double time_launches(cudaStream_t st, int reps, F&& f) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();  // warm
    CK(cudaEventRecord(a, st));
    for (int r = 0; r < reps; ++r) f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / reps;
}

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
static void route_device() {
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

static void validate_ifta_cfg(const hgc_ifta_cfg* c) {  // IftaConfig::validate, ifta.hpp:41-50
    if (!c) invalid("IftaConfig: missing");
    if (c->iterations < 1) invalid("IftaConfig: iterations must be >= 1");
    if (!(c->weight_clamp_lo > 0) || !(c->weight_clamp_hi >= c->weight_clamp_lo))
        invalid("IftaConfig: weight clamp bounds invalid");
    if (!(c->lt_initial_fraction > 0) || !(c->lt_initial_fraction <= 1))
        invalid("IftaConfig: lt_initial_fraction must be in (0,1]");
    if (c->variant < 0 || c->variant > 2) invalid("IftaConfig: unknown variant");
    if (c->init_phase < 0 || c->init_phase > 3) invalid("IftaConfig: unknown init phase");
}

static void validate_fresnel(const hgc_fresnel* p) {  // FresnelParams::validate, propagation.hpp:21-29
    if (!(p->wavelength > 0) || !std::isfinite(p->wavelength)) invalid("FresnelParams: wavelength must be positive");
    if (p->distance == 0 || !std::isfinite(p->distance)) invalid("FresnelParams: distance must be non-zero");
    if (!(p->pixel_pitch_x > 0) || !(p->pixel_pitch_y > 0) || !std::isfinite(p->pixel_pitch_x) ||
        !std::isfinite(p->pixel_pitch_y))
        invalid("FresnelParams: pixel pitches must be positive");
}

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
        k_target_energy<<<p->batch, 256, 0, p->stream>>>(p->amp_d.p, io->roi ? p->roi_rm.p : nullptr, npix, p->stt.p);
        CK(cudaGetLastError());
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

    // run_ospr_impl's subframe loop (ospr.hpp:105-147), all jobs at once.
    // Plain OSPR: the seed of frame n+1 (one MT stream per job, its own
    // stream of the graph) overlaps the three passes of frame n on a second
    // field buffer; a seed CTA (512 thr x 56 regs, 40 KiB) co-resides with a
    // pass CTA on an SM.  Adaptive OSPR seeds frame n from S after frame n-1,
    // so it stays sequential.
    void record(cudaStream_t st) {
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

static void validate_ospr_cfg(const hgc_ospr_cfg* c) {  // OsprConfig::validate, ospr.hpp:30-37
    if (!c) invalid("OsprConfig: missing");
    if (c->subframes < 1) invalid("OsprConfig: subframes must be >= 1");
    if (!(c->feedback_gain >= 0.0 && c->feedback_gain <= 1.0)) invalid("OsprConfig: feedback_gain must be in [0,1]");
    if (c->variant < 0 || c->variant > 1) invalid("OsprConfig: unknown variant");
}

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
            p->preseed = cfg->variant == 0 && cfg->subframes > 1 && jobs < sms && all < (1ull << 31) &&
                         all * jobs * sizeof(float2) <= (8ull << 30);
            p->fstride = p->preseed ? all : p->npix;
        }
        p->field.alloc(p->fstride * jobs);
        if (ny >= 512) p->tmap1.make(p->field.p, nx, p->cw, p->fstride * jobs / (2 * (size_t)nx));
        if (!p->preseed && cfg->variant == 0 && cfg->subframes > 1) {  // second buffer + stream for seed/pass overlap
            p->field2.alloc(tot);
            if (ny >= 512) p->tmap2.make(p->field2.p, nx, p->cw, tot / (2 * (size_t)nx));
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
        p->partials.alloc((size_t)cfg->subframes * jobs * p->tiles * 8);
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
