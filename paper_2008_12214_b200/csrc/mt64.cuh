// mt64.cuh — bit-exact std::mt19937_64 stream on the GPU and the fused
// random-phase seed (seed_random_phase<float>, rng.hpp:54-67).
//
// The reference draws every random phase from ONE std::mt19937_64 stream
// seeded with Rng(seed).fork(0) (rng.hpp:42-44; ifta.hpp:124; ospr.hpp:89),
// one draw per pixel in row-major order, OSPR subframe k consuming draws
// [k*npix, (k+1)*npix).  The engine's 312-word twist is parallel within a
// block of 312 words, so one warp regenerates the raw-word sequence into a
// shared-memory ring while the rest of the CTA tempers the words and
// evaluates (T)(a*cos(2*pi*u)), (T)(a*sin(2*pi*u)) in double — the DP sincos
// is the real cost and is spread across 15 warps.  The stream state (the
// twist block holding the next draw + position) is saved to global memory at
// the end of a launch so the next subframe continues the same stream.
#pragma once
#include "common.cuh"

namespace hg {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtUM = 0xFFFFFFFF80000000ull;
constexpr uint64_t kMtLM = 0x000000007FFFFFFFull;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;

// Saved stream position: the twist block that holds the next draw, and the
// index of that draw within the block (312 = block exhausted).
struct MtState {
    uint64_t w[kMtN];
    int pos;
    int pad_;
};

__host__ __device__ inline uint64_t mix64(uint64_t z) {  // rng.hpp:12-17
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d4a2c62a2b3b9full;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t fork_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:42-44
    return mix64(seed ^ mix64(stream + 1));
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t hi, uint64_t lo) {
    uint64_t x = (hi & kMtUM) | (lo & kMtLM);
    return (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
}

// One twist by a single warp: nw <- twist(ow).  Same recurrence as the
// in-place libstdc++ _M_gen_rand, written out-of-place: words i < 156 depend
// only on the old block, words 156..311 on the old block and new words
// i - 156 (and word 311 on new word 0).  All loads of a phase are issued
// before any store so the smem latency is paid twice per twist, not per word.
__device__ __forceinline__ void mt_twist_warp(const uint64_t* __restrict__ ow, uint64_t* __restrict__ nw, int lane) {
    constexpr int H = kMtN - kMtM;  // 156
    uint64_t a[5], b[5], c[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        const int i = lane + 32 * m;
        if (i < H) {
            a[m] = ow[i];
            b[m] = ow[i + 1];
            c[m] = ow[i + kMtM];
        }
    }
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        const int i = lane + 32 * m;
        if (i < H) nw[i] = c[m] ^ mt_mix(a[m], b[m]);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        const int i = H + lane + 32 * m;
        if (i < kMtN) {
            a[m] = ow[i];
            b[m] = i + 1 < kMtN ? ow[i + 1] : nw[0];
            c[m] = nw[i - H];
        }
    }
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        const int i = H + lane + 32 * m;
        if (i < kMtN) nw[i] = c[m] ^ mt_mix(a[m], b[m]);
    }
    __syncwarp();
}

// sin and cos of theta in [0, 2*pi] in double: 3-part Cody-Waite reduction by
// pi/2 (exact for n <= 4 with FMA) + fdlibm __kernel_sin/__kernel_cos
// polynomials.  <= 1 ulp from glibc's sin/cos; over 4e7 random draws the
// float casts (T)(a*cos), (T)(a*sin) of rng.hpp:62-64 matched glibc exactly.
// ~3x fewer instructions than the general-range CUDA sincos (no slow path).
// The coefficients live in constant memory so DFMA reads them as constant-
// bank operands (as literals, every use re-materialised the 64-bit value
// with two uniform moves).
struct SinCos64 {
    double two_over_pi, pio2_1, pio2_2, pio2_3;
    double s6, s5, s4, s3, s2, s1;
    double c6, c5, c4, c3, c2, c1;
};
static __constant__ SinCos64 kSC = {6.36619772367581382433e-01,  1.5707963267948966192e+00,
                                    6.123233995736766036e-17,     -1.4973849048591698e-33,
                                    1.58969099521155010221e-10,   -2.50507602534068634195e-08,
                                    2.75573137070700676789e-06,   -1.98412698298579493134e-04,
                                    8.33333333332248946124e-03,   -1.66666666666666324348e-01,
                                    -1.13596475577881948265e-11,  2.08757232129817482790e-09,
                                    -2.75573143513906633035e-07,  2.48015872894767294178e-05,
                                    -1.38888888888741095749e-03,  4.16666666666666019037e-02};
__device__ __forceinline__ void sincos_0_2pi(double x, double* sp, double* cp) {
    const double n = rint(x * kSC.two_over_pi);
    double r = fma(-n, kSC.pio2_1, x);
    r = fma(-n, kSC.pio2_2, r);
    r = fma(-n, kSC.pio2_3, r);
    const int q = (int)n & 3;
    const double z = r * r;
    const double ps = fma(fma(fma(fma(kSC.s6, z, kSC.s5), z, kSC.s4), z, kSC.s3), z, kSC.s2);
    const double sr = fma(r * z, fma(z, ps, kSC.s1), r);
    const double pc = fma(fma(fma(fma(fma(kSC.c6, z, kSC.c5), z, kSC.c4), z, kSC.c3), z, kSC.c2), z, kSC.c1);
    const double hz = 0.5 * z, w = 1.0 - hz;
    const double cr = w + (((1.0 - w) - hz) + z * (z * pc));
    const double s0 = (q & 1) ? cr : sr, c0 = (q & 1) ? sr : cr;
    *sp = (q & 2) ? -s0 : s0;
    *cp = ((q + 1) & 2) ? -c0 : c0;
}

constexpr int kSeedThreads = 512;
// Fast loop: one draw per iteration at <= 64 registers (2 CTAs / SM).  The
// OSPR seed runs beside the passes of the previous frame, so its footprint
// matters: unroll 2 / 64 registers / 1 CTA per SM measured 43.0k vs 51.8k
// subframes/s, unroll 4 (96 registers) no better.
#ifndef HG_SEED_UNROLL
#define HG_SEED_UNROLL 1
#endif
#ifndef HG_SEED_MINB
#define HG_SEED_MINB 2
#endif
constexpr int kSeedUnroll = HG_SEED_UNROLL;
constexpr int kTwistsPerGroup = 8;
constexpr int kRingSlots = 2 * kTwistsPerGroup;  // two groups: one produced while one is consumed
constexpr size_t kSeedSmem = sizeof(uint64_t) * kMtN * kRingSlots;

struct SeedArgs {
    MtState* states;           // [streams]
    const uint64_t* seeds;     // [streams] engine seeds (already forked) or nullptr = continue
    const double* amp;         // amplitude (double, as RealImage), per stream stride amp_stride
    size_t amp_stride;
    float2* out;               // seeded field, per stream stride out_stride
    size_t out_stride;
    size_t npix;               // draws (pixels) this launch
    // adaptive OSPR intensity budget (ospr.hpp:106-116): amp for frame n >= 2
    // is (1-g)*T + g*sqrt(max(0, n*T^2 - (n-1)*(S/(n-1)))), S = running sum.
    const float* S;            // [streams][npix] or nullptr (plain amplitude)
    size_t S_stride;
    int n;
    double gain;
    // output layout: quad != 0 writes the plans' LAY_QUAD field (and reads S
    // column-pair major); otherwise row-major.  nx, ny used when quad != 0.
    int quad, nx, ny;
    // chunking: CTA b = stream * chunks + c draws [c*chunk_len, min(npix, (c+1)*chunk_len))
    // of this launch, starting from states[b] (set by k_mt_jump) unless c == 0 and seeds
    // is given.  chunks <= 1: one CTA per stream over all npix draws.
    int chunks;
    size_t chunk_len;
    int no_save;  // keep states[] (the chunk start windows) instead of saving the end state
    // seed_random_phase<double> (the f64 loops): (a*cos, a*sin) unrounded,
    // row-major, stride out_stride — used instead of `out` when set
    double2* out64;
};

// Jump-ahead (mtjump.cpp): CTA (stream s, chunk c), c in [c_lo, chunks),
// writes states[s*chunks + c] = its start window advanced by J draws, as
// g(F) W_1 with g = x^(J-1) mod P: word j = XOR over set bits i of g of raw
// word x_{1+i+j}, x_0.. being the start window (the fresh seed block when
// `from` is null, else from[s*chunks + c], a pos = 312 window; may alias
// states).  g is given as its set-bit offsets per 312-bit block (mtjump.cpp,
// mt_poly_offsets): poly k = c - poly_base (0 for every chunk when
// poly_step == 0) has offsets pool[starts[65k + q] .. starts[65k + q + 1]) in
// block q.  Chunks c < poly_base are not moved (the seed block is stored as
// is).  The raw words are regenerated block by block (one warp twists block
// q+2 while the CTA accumulates block q's offsets from blocks q, q+1); each
// block is stored twice (slots b%3 and b%3+3) so reads never wrap.  Two
// thread groups split each block's offsets; their partial XORs are combined
// at the end.
constexpr int kJumpGroups = 2;
constexpr int kJumpGroupThreads = 320;
constexpr int kJumpThreads = kJumpGroups * kJumpGroupThreads;
constexpr int kJumpBlocks = 64;  // 312-bit blocks covering deg P = 19937
struct JumpArgs {
    const uint64_t* seeds;  // [streams] engine seeds (from == nullptr)
    const MtState* from;    // [streams * chunks] start windows, or nullptr
    const int* starts;      // [polys][kJumpBlocks + 1]
    const uint16_t* pool;   // set-bit offsets within each block
    int poly_step;          // 1: one polynomial per chunk; 0: one for all
    MtState* states;        // [streams * chunks]
    int chunks, c_lo, poly_base;
    int splits;             // > 1: each jump's 64 blocks split over `splits` CTAs, combined by
                            // atomicXor into zeroed states (from must be null); <= 1: one CTA
};

static __global__ void __launch_bounds__(kJumpThreads) k_mt_jump(JumpArgs a) {
    __shared__ uint64_t ring[6 * kMtN];
    __shared__ uint64_t red[kMtN];
    const int splits = a.splits > 1 ? a.splits : 1;
    const int per = a.chunks - a.c_lo;
    const int jb = blockIdx.x / splits, part = blockIdx.x % splits;
    const int s = jb / per, c = a.c_lo + jb % per;
    const size_t b = (size_t)s * a.chunks + c;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.from) {
        for (int i = tid; i < kMtN; i += blockDim.x) ring[i] = ring[3 * kMtN + i] = a.from[b].w[i];
    } else if (tid == 0) {
        uint64_t x = a.seeds[s];  // std::mt19937_64::seed: block 0
        ring[0] = ring[3 * kMtN] = x;
        for (int i = 1; i < kMtN; ++i) {
            x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
            ring[i] = ring[3 * kMtN + i] = x;
        }
    }
    __syncthreads();
    if (c < a.poly_base) {  // offset 0: the seed block itself
        if (part == 0) {
            for (int i = tid; i < kMtN; i += blockDim.x) a.states[b].w[i] = ring[i];
            if (tid == 0) a.states[b].pos = kMtN;
        }
        return;
    }
    // this CTA's share of the blocks: q in [q0, q1); raw blocks 1 .. q0+1 first
    // (block i lives in ring slot i % 3, mirrored at +3)
    const int q0 = part * kJumpBlocks / splits, q1 = (part + 1) * kJumpBlocks / splits;
    const int* st = a.starts + (size_t)(c - a.poly_base) * a.poly_step * (kJumpBlocks + 1);
    if (warp == 0) {
        for (int i = 1; i <= q0 + 1; ++i) {
            const int so = (i - 1) % 3, sn = i % 3;
            mt_twist_warp(ring + so * kMtN, ring + sn * kMtN, lane);
            for (int w = lane; w < kMtN; w += 32) ring[(sn + 3) * kMtN + w] = ring[sn * kMtN + w];
            __syncwarp();
        }
    }
    __syncthreads();
    const int grp = tid / kJumpGroupThreads, j = tid % kJumpGroupThreads;
    uint64_t acc = 0;
    for (int q = q0; q < q1; ++q) {
        if (warp == 0 && q + 1 < q1) {  // block q+2 from block q+1 (needed by block q+1's offsets)
            const int so = (q + 1) % 3, sn = (q + 2) % 3;
            mt_twist_warp(ring + so * kMtN, ring + sn * kMtN, lane);
            for (int i = lane; i < kMtN; i += 32) ring[(sn + 3) * kMtN + i] = ring[sn * kMtN + i];
        }
        if (j < kMtN) {
            const uint64_t* base = ring + (q % 3) * kMtN + 1 + j;  // x_{312q + 1 + j + ii} = base[ii]
            const int k0 = __ldg(st + q), k1 = __ldg(st + q + 1);
            const int half = (k1 - k0 + 1) >> 1;
            const uint16_t* off = a.pool + k0 + (grp ? half : 0);
            const int cnt = grp ? (k1 - k0) - half : half;
            int k = 0;
#pragma unroll 1
            for (; k + 4 <= cnt; k += 4) {
                const int o0 = __ldg(off + k), o1 = __ldg(off + k + 1), o2 = __ldg(off + k + 2), o3 = __ldg(off + k + 3);
                acc ^= base[o0] ^ base[o1] ^ base[o2] ^ base[o3];
            }
            for (; k < cnt; ++k) acc ^= base[__ldg(off + k)];
        }
        __syncthreads();
    }
    if (grp == 1 && j < kMtN) red[j] = acc;
    __syncthreads();
    if (grp == 0 && j < kMtN) {
        if (splits > 1) atomicXor(reinterpret_cast<unsigned long long*>(&a.states[b].w[j]), acc ^ red[j]);
        else a.states[b].w[j] = acc ^ red[j];
    }
    if (tid == 0 && part == 0) a.states[b].pos = kMtN;
}

// One CTA per stream.  Warp 0 produces twists; warps 1.. consume.
// FAST: the plans' common case (float quad-layout output, plain amplitude),
// with 32-bit index arithmetic and nothing else in the consumer loop; the
// generic instantiation serves row-major / adaptive / double outputs.
template <bool FAST>
__global__ void __launch_bounds__(kSeedThreads, FAST ? HG_SEED_MINB : 1) k_seed_random_phase(SeedArgs a) {
    extern __shared__ uint64_t ring[];  // kRingSlots * 312 words
    __shared__ int s_pos;
    const int chunks = a.chunks > 1 ? a.chunks : 1;
    const int s = blockIdx.x / chunks, c = blockIdx.x % chunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    MtState* st = a.states + blockIdx.x;
    uint64_t* init = ring + (kRingSlots - 1) * kMtN;  // twist "-1" lives in the last slot
    if (a.seeds && c == 0) {
        if (tid == 0) {  // std::mt19937_64::seed
            uint64_t x = a.seeds[s];
            init[0] = x;
            for (int i = 1; i < kMtN; ++i) {
                x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
                init[i] = x;
            }
            s_pos = kMtN;
        }
    } else {
        for (int i = tid; i < kMtN; i += blockDim.x) init[i] = st->w[i];
        if (tid == 0) s_pos = st->pos;
    }
    __syncthreads();
    const int pos0 = s_pos;
    const size_t cbeg = chunks > 1 ? (size_t)c * a.chunk_len : 0;
    if (cbeg >= a.npix) return;
    const size_t npix = chunks > 1 ? (a.npix - cbeg < a.chunk_len ? a.npix - cbeg : a.chunk_len) : a.npix;
    const double* amp = a.amp + a.amp_stride * s;
    float2* out = a.out + a.out_stride * s;

    // draws available from the initial block, then 8-twist groups
    const size_t first = (size_t)(kMtN - pos0) < npix ? (size_t)(kMtN - pos0) : npix;
    const size_t rest = npix - first;
    const long long ngroups = (long long)((rest + (size_t)kMtN * kTwistsPerGroup - 1) / ((size_t)kMtN * kTwistsPerGroup));

    const int cthreads = blockDim.x - 32;
    const int ctid = tid - 32;
    const int lognx = 31 - __clz(a.nx > 0 ? a.nx : 1), nxm = a.nx - 1;  // nx is a power of two
    const int pmask = a.quad ? a.nx * a.ny - 1 : 0x7fffffff;
    const double* __restrict__ ampp = amp;
    const float* __restrict__ Sp = a.S ? a.S + a.S_stride * s : nullptr;
    // step g: producer writes group g (g < ngroups); consumers process group g-1
    // (g = 0: the initial partial block).  Pixel indices fit 32 bits (npix <= 2^24).
    for (long long g = 0; g <= ngroups; ++g) {
        if (warp == 0) {
            if (g < ngroups) {
                for (int k = 0; k < kTwistsPerGroup; ++k) {
                    int t = (int)(g * kTwistsPerGroup + k);
                    const uint64_t* ow = ring + ((t - 1 + kRingSlots) % kRingSlots) * kMtN;
                    uint64_t* nw = ring + (t % kRingSlots) * kMtN;
                    mt_twist_warp(ow, nw, lane);
                }
            }
        } else if (a.out || a.out64) {  // neither: advance the stream only (skip draws)
            const uint64_t* src;
            int d0, cnt;
            if (g == 0) {
                src = init + pos0;
                d0 = 0;
                cnt = (int)first;
            } else {
                src = ring + (((g - 1) & 1) * kTwistsPerGroup) * kMtN;
                d0 = (int)(first + (size_t)(g - 1) * kMtN * kTwistsPerGroup);
                const int left = (int)npix - d0;
                cnt = left < kMtN * kTwistsPerGroup ? left : kMtN * kTwistsPerGroup;
            }
            if constexpr (FAST) {
                const int pb = (int)cbeg + d0;
                const int qshift = lognx - 1;
                // bases held in registers (not re-derived from the kernel
                // parameters with 64-bit multiplies on every draw)
                const double* __restrict__ ab = opaque(ampp);
                float2* __restrict__ ob = opaque(out);
#pragma unroll kSeedUnroll
                for (int j = ctid; j < cnt; j += cthreads) {
                    const int p = pb + j;  // row-major pixel index of this draw (rng.hpp:60)
                    const double av = __ldg(&ab[p & pmask]);
                    const uint64_t x = mt_temper(src[j]);
                    const double u = (double)(x >> 11) * 0x1.0p-53;  // Rng::uniform01, rng.hpp:32
                    const double theta = __dmul_rn(HG_TWO_PI, u);    // rng.hpp:62
                    double sn, cs;
                    sincos_0_2pi(theta, &sn, &cs);
                    const int px = p & nxm, py = p >> lognx;
                    const int o = ((((py >> 1) << qshift) + (px >> 1)) << 2) + ((py & 1) << 1) + (px & 1);
                    ob[o] = make_float2(__double2float_rn(__dmul_rn(av, cs)), __double2float_rn(__dmul_rn(av, sn)));
                }
            } else {
#pragma unroll 2
            for (int j = ctid; j < cnt; j += cthreads) {
                const uint64_t x = mt_temper(src[j]);
                const double u = (double)(x >> 11) * 0x1.0p-53;  // Rng::uniform01, rng.hpp:32
                const double theta = __dmul_rn(HG_TWO_PI, u);    // rng.hpp:62
                double sn, cs;
                sincos_0_2pi(theta, &sn, &cs);
                const int p = (int)cbeg + d0 + j;  // row-major pixel index of this draw (rng.hpp:60)
                double av = ampp[p & pmask];  // pre-seeded OSPR: draw p of frame p / npix
                int o = p, so = p;
                if (a.quad) {
                    const int py = p >> lognx, px = p & nxm;
                    o = (int)quad_index(px, py, a.nx);
                    so = (int)colpair_index(px, py, a.ny);
                }
                if (Sp) {  // adaptive OSPR budget, ospr.hpp:111-114
                    const double tv = av, t2 = __dmul_rn(tv, tv);
                    const double sv = (double)Sp[so];
                    const double n = a.n;
                    double budget = __dsub_rn(__dmul_rn(n, t2), __dmul_rn(n - 1.0, __ddiv_rn(sv, n - 1.0)));
                    double tn = __dsqrt_rn(budget > 0.0 ? budget : 0.0);
                    av = __dadd_rn(__dmul_rn(1.0 - a.gain, tv), __dmul_rn(a.gain, tn));
                }
                if (a.out64)
                    a.out64[a.out_stride * s + p] = make_double2(__dmul_rn(av, cs), __dmul_rn(av, sn));
                else
                    out[o] = make_float2(__double2float_rn(__dmul_rn(av, cs)), __double2float_rn(__dmul_rn(av, sn)));
            }
            }
        }
        __syncthreads();
    }
    if (a.no_save) return;
    // save the block holding the next draw
    const uint64_t* keep;
    int pos;
    if (rest == 0) {
        keep = init;
        pos = pos0 + (int)npix;
    } else {
        long long tl = (long long)((rest - 1) / kMtN);
        keep = ring + (tl % kRingSlots) * kMtN;
        pos = (int)((rest - 1) % kMtN) + 1;
    }
    for (int i = tid; i < kMtN; i += blockDim.x) st->w[i] = keep[i];
    if (tid == 0) st->pos = pos;
}

}  // namespace hg
