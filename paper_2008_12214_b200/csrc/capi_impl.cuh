// capi_impl.cuh — internals shared by the C-ABI translation units (capi.cu:
// library state, device routing and validation; ifta_plan.cu; ospr_plan.cu;
// f64.cu; primitives.cu): device buffers, layout conversions, the quantiser
// tables, TMA tensor maps and the seed chunking.  Its kernels and helpers are
// static: each translation unit gets the ones it uses.
#pragma once
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
extern thread_local std::string g_err;  // capi.cu

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
// Per-device one-time setup; returns the device's twiddle table (capi.cu).
const float2* device_twiddles();

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
constexpr size_t kMinChunkDraws = 4096;
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
        // Chunk count from a cost model measured on B200: a chunk's draws cost
        // ~1.2 ns each on its CTA; a jump ~240 us on one CTA (64 sequential
        // 312-word XOR blocks), split over up to 16 CTAs when the jumps do not
        // fill the GPU (launch()), plus ~15 us of block prefix per split.
        const long long cmax = std::max<long long>(1, std::min<long long>(kMaxChunks, (long long)(npix / kMinChunkDraws)));
        auto cost = [&](long long k) {
            const double draws = (double)((npix + k - 1) / k);
            const long long seed_waves = (S * k + slots - 1) / slots;
            double t = (double)seed_waves * draws * 1.2e-3;  // us
            if (k > 1 || offset > 0) {
                const long long nj = S * (offset > 0 ? k : k - 1);
                const long long jslots = 2LL * sms;
                const long long sp = std::max<long long>(1, std::min<long long>(16, jslots / std::max<long long>(1, nj)));
                const long long jwaves = (nj * sp + jslots - 1) / jslots;
                t += (double)jwaves * (15.0 + 240.0 / (double)sp);
            }
            return t;
        };
        long long c = 1;
        double best = cost(1);
        for (long long k = 2; k <= cmax; ++k) {
            const double t = cost(k);
            if (t < best * 0.98) best = t, c = k;
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
            // a jump costs ~240 us on one CTA (64 blocks of 312-word XOR windows,
            // shared-memory bound): when there are fewer jumps than SM slots, each
            // is split over several CTAs (their partial XORs combined atomically)
            const int nj = streams * (chunks - c_first());
            int sms = 148, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            int splits = std::max(1, std::min(16, 2 * sms / std::max(1, nj)));
            if (const char* ev = getenv("HG_JUMP_SPLITS")) splits = std::max(1, atoi(ev));  // tuning
            if (splits > 1) CK(cudaMemsetAsync(states, 0, sizeof(MtState) * (size_t)streams * chunks, st));
            JumpArgs ja{seeds, nullptr, starts.p, pool.p, 1, states, chunks, c_first(), c_first(), splits};
            k_mt_jump<<<nj * splits, kJumpThreads, 0, st>>>(ja);
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
                JumpArgs ja{seeds, nullptr, starts.p, pool.p, 1, states, 1, 0, 0, 1};
                k_mt_jump<<<streams, kJumpThreads, 0, st>>>(ja);
                ++n;
            }
            sa.seeds = first && offset0 == 0 ? seeds : nullptr;
            seed_launch(streams, sa, st);
            return n + 1;
        }
        JumpArgs ja = first ? JumpArgs{seeds, nullptr, starts.p, pool.p, 1, states, chunks, 0, c_first(), 1}
                            : JumpArgs{nullptr, states, step_starts.p, step_pool.p, 0, states, chunks, 0, 0, 1};
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
static __global__ void k_fill_c(float2* p, size_t n, float2 v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
static __global__ void k_fill_f(float* p, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
static __global__ void k_d2f(const double* a, float* o, size_t n) {
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
static __global__ void k_to_colpair(const TI* in, TO* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[p.b * npix + colpair_index(p.x, p.y, ny)] = (TO)in[g];
    }
}
template <class T>
static __global__ void k_from_colpair(const T* in, T* out, int nx, int ny, size_t total) {
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
static __global__ void __launch_bounds__(256) k_to_colpair_tiled(const TI* in, TO* out, int nx, int ny) {
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

static __global__ void k_to_quad(const float2* in, float2* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[p.b * npix + quad_index(p.x, p.y, nx)] = in[g];
    }
}
static __global__ void k_from_quad(const float2* in, float2* out, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        out[g] = in[p.b * npix + quad_index(p.x, p.y, nx)];
    }
}
// InitPhase::Flat, ifta.hpp:128-130 (quad output)
static __global__ void k_init_flat(const double* a, float2* f, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        f[p.b * npix + quad_index(p.x, p.y, nx)] = make_float2((float)a[g], 0.f);
    }
}
// target-phase init, ifta.hpp:131-136 (tphase = 2*pi*turns, ifta.hpp:107-111) (quad output)
static __global__ void k_init_target_phase(const double* a, const double* turns, float2* f, int nx, int ny, size_t total) {
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
static __global__ void k_phase_cs(const double* turns, float2* cs, int nx, int ny, size_t total) {
    const size_t npix = (size_t)nx * ny;
    HG_GRID_LOOP(g, total) {
        Pix p = pix_of(g, nx, npix);
        double s, c;
        sincos(__dmul_rn(HG_TWO_PI, turns[g]), &s, &c);
        cs[p.b * npix + colpair_index(p.x, p.y, ny)] = make_float2((float)c, (float)s);
    }
}
// make_fresnel_phase<float>, propagation.hpp:36-54 (no FMA contraction)
static __global__ void k_fresnel_q(int nx, int ny, double scale, double px, double py, float2* q) {
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
static __global__ void k_quantise(float2* f, int32_t* lv, size_t npix, size_t total, QuantParams q) {
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        size_t i = g % npix;
        float2 v = f[g];
        int k = quant_decide(q, v.x, v.y, i);
        f[g] = quant_state(q, k, i);
        if (lv) lv[g] = k;
    }
}
// mse partials in double (primitive): sum (T-r)^2, T r, r^2, T^2, count
static __global__ void k_mse_partials(const double* t, const float2* r, const uint8_t* m, size_t n, double* out) {
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
static __global__ void k_finalize(const double* part, int slots, int targets, int tiles, double M, int scale_free,
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
static __global__ void __launch_bounds__(256) k_ospr_block_cum(const float* gathered, int index, int nblocks,
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
static __global__ void k_levels_gray8(const uint8_t* lv8, const uint16_t* lv16, size_t n, const uint8_t* table,
                               uint8_t* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = table[lv8 ? lv8[i] : lv16[i]];
}

// 2-level SLMs: levels as bit-planes (bit i & 7 of byte i >> 3), 8 pixels per byte.
static __global__ void k_pack_levels1(const uint8_t* lv8, size_t nbytes, uint8_t* out) {
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
static __global__ void k_amp_peak(AmpSrc src, size_t npix, double* block_max) {
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
static __global__ void k_peak_final(const double* block_max, int nblk, double* peak) {
    const int b = blockIdx.x;
    double m = 0.0;
    for (int j = threadIdx.x; j < nblk; j += 32) m = fmax(m, block_max[(size_t)b * nblk + j]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) peak[b] = m;
}
static __global__ void k_amp_gray8(AmpSrc src, size_t npix, const double* peak, uint8_t* out) {
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
// target energy), once per upload of a scale-free plan: kTeBlocks partial
// sums per target (grid-strided), then a fixed-order sum per target.
constexpr int kTeBlocks = 128;
static __global__ void __launch_bounds__(256) k_target_energy_part(const double* amp, const uint8_t* roi_rm,
                                                                   size_t npix, double* part) {
    const double* a = amp + npix * blockIdx.y;
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x)
        if (!roi_rm || roi_rm[i]) s += a[i] * a[i];
    __shared__ double red[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
        x = warp_sum(x);
        if (threadIdx.x == 0) part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = x;
    }
}
static __global__ void k_target_energy_fin(const double* part, int nb, double* stt) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) s += part[(size_t)blockIdx.x * nb + i];
    s = warp_sum(s);
    if (threadIdx.x == 0) stt[blockIdx.x] = s;
}

static __global__ void k_validate(const double* amp, const double* phase, size_t n, int* flags) {
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
    p.min_u_f = (float)(s->min_arg * inv);
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

// ---- shared between the translation units (defined in capi.cu) -----------
void route_device();
void validate_ifta_cfg(const hgc_ifta_cfg* c);
void validate_fresnel(const hgc_fresnel* p);
void validate_ospr_cfg(const hgc_ospr_cfg* c);

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
inline double time_launches(cudaStream_t st, int reps, F&& f) {
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

