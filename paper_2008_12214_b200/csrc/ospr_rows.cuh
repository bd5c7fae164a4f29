// ospr_rows.cuh — the rows-first OSPR subframe (ospr.hpp:105-147).
//
// The column-first subframe is four HBM round trips: seed, column IFFT, row
// pass (row IFFT, quantise, row FFT), column FFT + accumulation (61 B/px).
// Regrouping the 2-D transforms' halves rows-first gives three, with the seed
// folded into the first:
//   A  k_ospr_seed_rows   seed a tile of RPC rows into shared memory (the
//                         bit-exact mt19937_64 draws + double sincos of
//                         mt64.cuh), IFFT the rows, store           [W field]
//   B  k_col<COL_OSPR_MID> IFFT columns, *norm, quantise (+levels),
//                         FFT columns                             [R+W field]
//   C  k_ospr_row_acc     FFT rows, *norm, S += |R|^2, frame and cumulative
//                         MSE partials                     [R field, R+W S]
// (41 B/px per subframe with levels).  A tile's draws start at an arbitrary
// point of its job's stream, so k_mt_walk (one warp per job, launched per
// frame beside the previous frame's passes) walks the stream and stores the
// mt19937_64 window holding the first draw of every tile; the seed pass then
// regenerates only its own tile's draws.
//
// Measured at BASELINE config 3 (148 jobs x 1024^2 x 24 frames, one B200):
// walk 0.97 ms, A 1.38 ms, B 1.04 ms, C 0.69 ms per frame batch; 39.9k
// subframes/s against 52.5k for the column-first loop (seed 1.35 ms beside
// col_inv 0.44 + row 0.78 + col_acc 0.72 ms).  A tile's 26 stream blocks are a
// serial twist chain, so pass A runs at the old seed's per-SM draw rate; with
// the walk storing every raw word instead (HG_OSPR_ROWS=3) A drops to 0.93 ms
// but the walk itself (1.64 ms) then competes with the passes: 36.5k.  Opt-in
// only (HG_OSPR_ROWS, ospr_plan.cu); parity-tested (tests/test_gpu_ospr_rows.py).
#pragma once
#include "mt64.cuh"
#include "ospr_rows_args.h"
#include "passes.cuh"

namespace hg {

// ---------------------------------------------------------------- walker
constexpr int kWalkWarps = 4;

static __global__ void __launch_bounds__(32 * kWalkWarps) k_mt_walk(WalkArgs a) {
    __shared__ uint64_t win[kWalkWarps][2][kMtN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int s = blockIdx.x * kWalkWarps + w;
    if (s >= a.streams) return;
    uint64_t* cur = win[w][0];
    uint64_t* nxt = win[w][1];
    int pos;
    if (a.seeds) {
        if (lane == 0) {  // std::mt19937_64::seed
            uint64_t x = a.seeds[s];
            cur[0] = x;
            for (int i = 1; i < kMtN; ++i) {
                x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
                cur[i] = x;
            }
        }
        pos = kMtN;
    } else {
        for (int i = lane; i < kMtN; i += 32) cur[i] = a.states[s].w[i];
        pos = a.states[s].pos;
    }
    __syncwarp();
    if (a.raw) {  // store the frame's raw words in draw order
        uint64_t* out = a.raw + (size_t)s * a.chunks * a.len;
        const int total = a.chunks * a.len;
        for (int d = 0; d < total;) {
            if (pos == kMtN) {
                mt_twist_warp(cur, nxt, lane);
                uint64_t* t = cur;
                cur = nxt;
                nxt = t;
                pos = 0;
            }
            const int take = min(kMtN - pos, total - d);
            for (int i = lane; i < take; i += 32) out[d + i] = cur[pos + i];
            pos += take;
            d += take;
        }
        for (int i = lane; i < kMtN; i += 32) a.states[s].w[i] = cur[i];
        if (lane == 0) a.states[s].pos = pos;
        return;
    }
    MtState* ck = a.ck + (size_t)s * a.chunks;
    for (int c = 0; c < a.chunks; ++c) {
        for (int i = lane; i < kMtN; i += 32) ck[c].w[i] = cur[i];
        if (lane == 0) ck[c].pos = pos;
        int left = a.len;  // skip this tile's draws
        while (left > 0) {
            if (pos == kMtN) {
                mt_twist_warp(cur, nxt, lane);
                uint64_t* t = cur;
                cur = nxt;
                nxt = t;
                pos = 0;
            }
            const int take = min(kMtN - pos, left);
            pos += take;
            left -= take;
        }
    }
    for (int i = lane; i < kMtN; i += 32) a.states[s].w[i] = cur[i];
    if (lane == 0) a.states[s].pos = pos;
}

// ------------------------------------------------------- A: seed + row IFFT
template <int NX>
struct SeedRowCfg {
    using Cfg = RowCfg<NX, LAY_QUAD>;
    static constexpr int RPC = Cfg::RPC, T = Cfg::T, E = Cfg::E;
    static constexpr int LEN = RPC * NX;                       // draws per tile
    static constexpr int LOGNX = ilog2(NX);
    static constexpr int XB = Cfg::SMEM;                       // exchange / tile buffer bytes
    static constexpr int SMEM = XB + (int)kSeedSmem;           // + the twist ring
    static constexpr bool ok = Cfg::THREADS == kSeedThreads && NX > E && T >= 2 && XB % 128 == 0;
};

// One CTA per (tile of RPC rows, job): warp 0 twists the tile's stream blocks
// into the ring while warps 1.. temper and convert (k_seed_random_phase<true>'s
// loop, rng.hpp:54-67) into the tile's quad-layout landing slots; then the
// whole CTA transforms the rows (the row half of P^-1) and bulk-stores them.
template <int NX>
__global__ void __launch_bounds__(kSeedThreads, 2) k_ospr_seed_rows(SeedRowArgs a) {
    using SC = SeedRowCfg<NX>;
    constexpr int T = SC::T, E = SC::E, LEN = SC::LEN;
    extern __shared__ __align__(128) float2 smem[];
    uint64_t* ring = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + SC::XB);
    __shared__ int s_pos;
    const int c = blockIdx.x, s = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.raw) {  // the walk stored the raw words: every thread tempers and converts
        const uint64_t* __restrict__ rw = a.raw + a.npix * s + (size_t)c * LEN;
        const double* __restrict__ ab = a.amp + a.amp_stride * s + (size_t)c * LEN;
#pragma unroll 2
        for (int d = tid; d < LEN; d += kSeedThreads) {
            const double av = __ldg(&ab[d]);
            const uint64_t x = mt_temper(__ldg(&rw[d]));
            const double u = (double)(x >> 11) * 0x1.0p-53;  // Rng::uniform01, rng.hpp:32
            const double theta = __dmul_rn(HG_TWO_PI, u);    // rng.hpp:62
            double sn, cs;
            sincos_0_2pi(theta, &sn, &cs);
            const int px = d & (NX - 1), ly = d >> SC::LOGNX;
            const int o = (ly >> 1) * (2 * NX) + (px >> 1) * 4 + (ly & 1) * 2 + (px & 1);
            smem[o] = make_float2(__double2float_rn(__dmul_rn(av, cs)), __double2float_rn(__dmul_rn(av, sn)));
        }
        __syncthreads();
    } else {
        const MtState* st = a.ck + (size_t)s * a.chunks + c;
        uint64_t* init = ring + (kRingSlots - 1) * kMtN;  // twist "-1" lives in the last slot
        for (int i = tid; i < kMtN; i += blockDim.x) init[i] = st->w[i];
        if (tid == 0) s_pos = st->pos;
        __syncthreads();
        const int pos0 = s_pos;
        const int first = min(kMtN - pos0, LEN);
        const int rest = LEN - first;
        constexpr int kGroup = kMtN * kTwistsPerGroup;
        const int ngroups = (rest + kGroup - 1) / kGroup;
        const double* __restrict__ amp = a.amp + a.amp_stride * s;
        const int p0 = c * LEN;  // row-major pixel index of the tile's first draw (rng.hpp:60)
        constexpr int lognx = SC::LOGNX;
        for (int g = 0; g <= ngroups; ++g) {
            if (warp == 0) {
                if (g < ngroups)
                    for (int k = 0; k < kTwistsPerGroup; ++k) {
                        const int t = g * kTwistsPerGroup + k;
                        mt_twist_warp(ring + ((t - 1 + kRingSlots) % kRingSlots) * kMtN, ring + (t % kRingSlots) * kMtN,
                                      lane);
                    }
            } else {
                const uint64_t* src;
                int d0, cnt;
                if (g == 0) {
                    src = init + pos0;
                    d0 = 0;
                    cnt = first;
                } else {
                    src = ring + (((g - 1) & 1) * kTwistsPerGroup) * kMtN;
                    d0 = first + (g - 1) * kGroup;
                    cnt = min(LEN - d0, kGroup);
                }
                const double* __restrict__ ab = opaque(amp);
                for (int j = tid - 32; j < cnt; j += kSeedThreads - 32) {
                    const int d = d0 + j;  // draw within the tile
                    const double av = __ldg(&ab[p0 + d]);
                    const uint64_t x = mt_temper(src[j]);
                    const double u = (double)(x >> 11) * 0x1.0p-53;  // Rng::uniform01, rng.hpp:32
                    const double theta = __dmul_rn(HG_TWO_PI, u);    // rng.hpp:62
                    double sn, cs;
                    sincos_0_2pi(theta, &sn, &cs);
                    const int px = d & (NX - 1), ly = d >> lognx;
                    const int o = (ly >> 1) * (2 * NX) + (px >> 1) * 4 + (ly & 1) * 2 + (px & 1);
                    smem[o] = make_float2(__double2float_rn(__dmul_rn(av, cs)), __double2float_rn(__dmul_rn(av, sn)));
                }
            }
            __syncthreads();
        }
    }
    // the row half of the inverse transform (k_row's thread mapping)
    const int pr = tid / (2 * T), q = tid % (2 * T);
    const int r = (q >> 1) & 1, t = ((q >> 2) << 1) | (q & 1);
    const int lr = 2 * pr + r;
    const RowSmemIdx idx{lr * RowStride<NX>::value};
    const int lb = (lr >> 1) * (2 * NX) + (t >> 1) * 4 + (lr & 1) * 2 + (t & 1);
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = smem[lb + e * 2 * T];
    __syncthreads();  // the tile becomes the exchange buffer
    fft_line<NX, +1, SC::Cfg::EM>(v, t, smem, idx, a.tw);
    const int lbo = opaque(lb);
#pragma unroll
    for (int e = 0; e < E; ++e) smem[lbo + e * 2 * T] = v[e];
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        bulk_s2g(a.field + a.npix * s + (size_t)c * LEN, smem, LEN * (int)sizeof(float2));
        bulk_commit();
        bulk_wait_read0();
    }
}

// ------------------------------------------- C: row FFT + accumulation
template <int NX>
struct RowAccCfg {
    using Cfg = RowCfg<NX, LAY_QUAD>;
    static constexpr int RPC = Cfg::RPC, LEN = RPC * NX;
    static constexpr int XB = Cfg::SMEM;
    static constexpr int SMEM = XB + LEN * (int)sizeof(float);
    static constexpr bool ok = Cfg::THREADS == 512 && NX > Cfg::E && Cfg::T >= 2 && XB % 128 == 0;
};

// One CTA per (tile of RPC rows, job): the tile and its S slice land by bulk
// copies; FFT rows (completes P), *norm, S += |R|^2, and the seven partial
// sums of COL_OSPR (ospr.hpp:134-145: frame MSE of R, cumulative MSE of
// sqrt(S/n), over the mask); S goes back by one bulk store.  R itself is not
// stored (nothing reads it).
template <int NX>
__global__ void __launch_bounds__(512, 2) k_ospr_row_acc(RowAccArgs a) {
    using AC = RowAccCfg<NX>;
    using Cfg = typename AC::Cfg;
    constexpr int RPC = AC::RPC, T = Cfg::T, E = Cfg::E, LEN = AC::LEN;
    extern __shared__ __align__(128) float2 smem[];
    float* Ssm = reinterpret_cast<float*>(reinterpret_cast<char*>(smem) + AC::XB);
    __shared__ uint64_t bar;
    const int c = blockIdx.x, s = blockIdx.y;
    const int tid = threadIdx.x;
    float* Sg = a.S + a.npix * s + (size_t)c * LEN;
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, LEN * (int)(sizeof(float2) + sizeof(float)));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem)),
                     "l"(a.field + a.npix * s + (size_t)c * LEN), "r"(LEN * (int)sizeof(float2)), "r"(smem_u32(&bar))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(Ssm)),
                     "l"(Sg), "r"(LEN * (int)sizeof(float)), "r"(smem_u32(&bar))
                     : "memory");
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    const int pr = tid / (2 * T), q = tid % (2 * T);
    const int r = (q >> 1) & 1, t = ((q >> 2) << 1) | (q & 1);
    const int lr = 2 * pr + r;
    const RowSmemIdx idx{lr * RowStride<NX>::value};
    const int lb = (lr >> 1) * (2 * NX) + (t >> 1) * 4 + (lr & 1) * 2 + (t & 1);
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = smem[lb + e * 2 * T];
    __syncthreads();
    fft_line<NX, -1, Cfg::EM>(v, t, smem, idx, a.tw);  // completes P
    const int y = c * RPC + lr;
    const float* __restrict__ tg = a.target + a.t_bstride * s + (size_t)y * NX;
    const uint8_t* __restrict__ roi = a.roi ? a.roi + (size_t)y * NX : nullptr;
    const float inv_n = a.inv_n, norm = a.norm;
    float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int x = t + e * T;
        const float2 R = cscale(v[e], norm);
        const float I = R.x * R.x + R.y * R.y;
        const float sv = Ssm[lr * NX + x] + I;
        Ssm[lr * NX + x] = sv;
        const float m = (!roi || roi[x]) ? 1.f : 0.f;
        const float amp = __ldg(&tg[x]) * m;
        const float rr = sqrtf(I) * m;
        const float d = amp - rr;
        acc[0] = fmaf(d, d, acc[0]);
        acc[1] = fmaf(amp, rr, acc[1]);
        acc[2] = fmaf(I, m, acc[2]);
        acc[3] = fmaf(amp, amp, acc[3]);
        const float rc = sqrtf(sv * inv_n) * m;
        const float dc = amp - rc;
        acc[4] = fmaf(dc, dc, acc[4]);
        acc[5] = fmaf(amp, rc, acc[5]);
        acc[6] = fmaf(rc, rc, acc[6]);
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        bulk_s2g(Sg, Ssm, LEN * (int)sizeof(float));
        bulk_commit();
    }
    block_sum_float_store<7>(acc, a.partials + ((size_t)s * gridDim.x + c) * 8);
    if (tid == 0) bulk_wait_read0();
}

}  // namespace hg
