// passes.cuh — the two fused HBM round trips of an IFTA iteration and the
// OSPR subframe passes.
//
// Layout in HBM: every field is complex64 row-major [target][ny][nx]
// (ComplexField<float>, field.hpp:27-46).  The 2-D inverse transform is done
// columns-first, the forward one rows-first, so one iteration of
// run_ifta (ifta.hpp:166-226) is exactly two passes:
//
//   ROW pass (aperture plane):  IFFT rows (completes P^-1)  -> *norm
//        -> *conj(Q) (Fresnel)  -> quantise (+levels)  -> *Q (Fresnel)
//        -> FFT rows (starts P)                                    [R+W field]
//   COL pass (replay plane):    FFT cols (completes P) -> *norm -> MSE partials
//        -> constraint (+WGS weights) -> IFFT cols (starts next P^-1) [R+W field,
//                                                            R target]
//   The last iteration's column pass stores the replay instead.
//
// OSPR (ospr.hpp:105-147) uses: seed kernel -> COL inverse -> ROW fused
// (levels out) -> COL forward with intensity accumulation + both MSE traces.
#pragma once
#include "fft.cuh"
#include "quant.cuh"

#ifndef HG_NULL_COMPUTE
#define HG_NULL_COMPUTE 0
#endif
#ifndef HG_ROWQ_MINB  // resident CTAs / SM asked of the quad-layout row pass (register cap)
#define HG_ROWQ_MINB 2
#endif
#ifndef HG_COLQ_MINB
#define HG_COLQ_MINB 2
#endif


namespace hg {

// --------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV doubles; thread 0 writes them to out[0..NV).  Fixed order.
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* out) {
    __shared__ double red[32][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) red[warp][i] = v[i];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = lane < nw ? red[lane][i] : 0.0;
            x = warp_sum(x);
            if (lane == 0) out[i] = x;
        }
    }
}

// ---------------------------------------------------------------- row pass
enum RowMode { ROW_FUSED = 0, ROW_PLAIN = 1 };

struct RowArgs {
    const float2* tw;  // twiddle table (fft.cuh)
    float2* field;
    size_t bstride;   // elements per target
    int ny;
    int layout;       // Layout (dispatch)
    float norm;       // (float)(1/sqrt(nx*ny)) applied after the row IFFT (fused) / the row FFT (plain, if apply_norm)
    int sign;         // ROW_PLAIN: -1 forward, +1 inverse
    int apply_norm;   // ROW_PLAIN
    const float2* fresnel_q;  // [ny][nx] row-major or nullptr
    QuantParams q;
    uint8_t* levels8;         // [target][ny][nx] row-major or nullptr
    uint16_t* levels16;
    size_t lv_bstride;
    int rpc;                  // quad layout: rows per CTA this launch (even, <= RowCfg::RPC; 0 = RowCfg::RPC)
};

template <int N>
struct RowStride {  // padded smem row; == 8 (mod 16) so a row pair sits 16 banks apart
    static constexpr int p = PaddedLen<N>::value;
    static constexpr int value = p + ((8 - p % 16) + 16) % 16;
};

// Elements per thread of the quad-layout passes for lines of at most
// HG_SMALL_NMAX points: 8 (radix-8 passes), twice the threads of the
// 16-element form.  A single small field leaves most SMs with 2-4 warps, so
// its passes are latency chains, not throughput (config 1, 512^2: 11.7 ->
// 10.2 us per iteration; at 1024 it lost: 23.2 -> 23.9 us, OSPR 53.0k ->
// 47.9k subframes/s).  Chosen by line length only, so batched and single
// runs of one size stay bit-identical.
#ifndef HG_SMALL_EM
#define HG_SMALL_EM 8
#endif
#ifndef HG_SMALL_NMAX
#define HG_SMALL_NMAX 512
#endif
template <int N, int LAY>
__host__ __device__ constexpr int quad_em() {
    return (LAY == LAY_QUAD && N <= HG_SMALL_NMAX) ? HG_SMALL_EM : 16;
}

template <int NX, int LAY>
struct RowCfg {
    static constexpr int EM = quad_em<NX, LAY>();
    static constexpr int E = LineCfg<NX, EM>::E, T = LineCfg<NX, EM>::T;
    static constexpr int RPC = LAY == LAY_QUAD ? (512 / T < 2 ? 2 : 512 / T) : (T >= 256 ? 1 : 256 / T);
    static constexpr int THREADS = T * RPC;
    static constexpr int SMEM = (NX > E) ? RPC * RowStride<NX>::value * (int)sizeof(float2) : 0;
    static constexpr int MIN_BLOCKS = LAY == LAY_QUAD ? (THREADS >= 512 ? HG_ROWQ_MINB : 1) : (THREADS >= 256 ? 3 : 1);
};

// The aperture-plane work of one row (thread t's elements x = t + e*T of row y
// of target b, in registers): IFFT (completes P^-1), *norm, *conj(Q),
// quantise (+levels), *Q, FFT (starts P).
template <int NX, int QK, int FQ, int LV, class Sync = CtaSync, int EM = 16>
__device__ __forceinline__ void row_fused_body(float2 (&v)[LineCfg<NX, EM>::E], int t, int y, int b, bool valid,
                                               float2* smem, const RowSmemIdx& idx, const RowArgs& a,
                                               const float2* sstates, const Sync& sync = Sync{}) {
    constexpr int E = LineCfg<NX, EM>::E, T = LineCfg<NX, EM>::T;
    fft_line<NX, +1, EM>(v, t, smem, idx, a.tw, sync);  // completes the 2-D inverse (propagation.hpp:89-95)
    const int rowbase = y * NX;
    const float norm = a.norm;
    const float2* __restrict__ fq = FQ == 0 ? nullptr : a.fresnel_q;
    const bool hasq = FQ == 1 || (FQ == 2 && fq != nullptr);
    uint8_t* __restrict__ lv8 = (LV != 0 && a.levels8) ? a.levels8 + a.lv_bstride * b : nullptr;
    uint16_t* __restrict__ lv16 = (LV != 0 && a.levels16) ? a.levels16 + a.lv_bstride * b : nullptr;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = rowbase + t + e * T;  // row-major pixel index (levels, Q, illumination)
        float2 f = cscale(v[e], norm);                        // fftw_backend.cpp:121-123
        if (hasq) f = cmul_conj_rn(f, __ldg(&fq[i]));         // propagation.hpp:93
#ifndef HG_ROW_VARIANT  // diagnostic builds: 1 = no quantiser, 2 = no forward row transform
#define HG_ROW_VARIANT 0
#endif
#if HG_ROW_VARIANT == 1
        const int k = (__float_as_int(f.x) >> 20) & 255;
#else
        const int k = quant_decide_kind<QK>(a.q, f.x, f.y, i);  // quantise.hpp:211-215
#endif
        if constexpr (QK == QK_BINARY) f = k ? a.q.s1 : a.q.s0;
        else if constexpr (QK == QK_FULL) f = HG_STATES_SMEM ? sstates[k] : __ldg(&a.q.states[k]);  // phase mode, no illumination
        else f = quant_state(a.q, k, i);
        if constexpr (LV != 0) {
            if (lv8 && valid) lv8[i] = (uint8_t)k;
            if (lv16 && valid) lv16[i] = (uint16_t)k;
        }
        if (hasq) f = cmul_rn(f, __ldg(&fq[i]));              // propagation.hpp:85
        v[e] = f;
    }
#if HG_ROW_VARIANT != 2
    fft_line<NX, -1, EM>(v, t, smem, idx, a.tw, sync);  // starts the forward transform
#endif
}

#ifndef HG_ROW_BULK
#define HG_ROW_BULK 1
#endif
// FQ: Fresnel Q in the fused pass — 0 absent, 1 present (compile time, the
// specialised quantisers), 2 decided at run time from a.fresnel_q.
// LV: level indices out — 0 never (compile time: the K-1 non-final iterations
// carry no store code or index registers), 1 when a.levels8/16 is set, 2
// decided at run time.
// The row pass of one CTA: row block bx (RPC rows) of target by.
template <int NX, int MODE, int QK, int LAY, int FQ, int LV>
__device__ __forceinline__ void row_cta(const RowArgs& a, const int bx, const int by) {
    using Cfg = RowCfg<NX, LAY>;
    constexpr int E = Cfg::E, T = Cfg::T;
    extern __shared__ __align__(128) float2 smem[];
    int lr, t;
    if constexpr (LAY == LAY_QUAD) {
        // the 2T threads of a row pair interleave so a warp covers 2 rows x 16
        // consecutive x = 8 whole quads (256 contiguous bytes)
        const int pr = threadIdx.x / (2 * T), q = threadIdx.x % (2 * T);
        int r;
        if constexpr (T >= 2) {
            r = (q >> 1) & 1;
            t = ((q >> 2) << 1) | (q & 1);
        } else {
            r = q & 1;
            t = 0;
        }
        lr = 2 * pr + r;
    } else {
        lr = threadIdx.x / T;
        t = threadIdx.x % T;
    }
    // rows per CTA: the compile-time tile, or fewer when a launch would leave SMs idle
    const int RPCr = (LAY == LAY_QUAD && Cfg::RPC > 2 && a.rpc > 0) ? a.rpc : Cfg::RPC;
    const int y = bx * RPCr + lr;
    const int b = by;
    RowSmemIdx idx{lr * RowStride<NX>::value};
    const bool valid = y < a.ny;  // (ny is a multiple of RPC except for tiny fields)
    const int yy = valid ? y : 0;
    float2* fb = a.field + a.bstride * b;
    // element e of this thread sits at x = t + e*T
    auto addr = [&](int e) -> size_t {
        if constexpr (LAY == LAY_QUAD) {
            if constexpr (T >= 2)
                return quad_index(t, yy, NX) + (size_t)e * (2 * T);  // x>>1 advances by T/2 quads
            else
                return quad_index(t + e * T, yy, NX);
        } else {
            return (size_t)yy * NX + t + e * T;
        }
    };
    float2 v[E];
    // Bulk path (quad layout): the CTA's RPC rows are RPC/2 whole quad rows,
    // contiguous in HBM, so one cp.async.bulk brings them into smem and one
    // writes them back; thread element e sits at landing slot lb + e*2T.
    constexpr bool kBulk = HG_ROW_BULK && LAY == LAY_QUAD && NX > E && T >= 2;
    __shared__ uint64_t rbar;
    // QK_FULL state table (<= 256 levels, quant_kind) in shared memory: the
    // per-pixel gather k -> state hits ~1 bank-conflict group instead of ~14 L1 lines
    constexpr bool kSmemStates = HG_STATES_SMEM && MODE == ROW_FUSED && QK == QK_FULL;
    __shared__ float2 sstates[kSmemStates ? 256 : 1];
    if constexpr (kSmemStates) {
        for (int i = threadIdx.x; i < a.q.levels; i += blockDim.x) sstates[i] = __ldg(&a.q.states[i]);
        if constexpr (!kBulk) __syncthreads();
    }
    // (recomputed where used, so nothing extra stays live across the transforms)
    auto tile_bytes = [&] {
        return (uint32_t)(min(RPCr, a.ny - (int)bx * RPCr) * NX * (int)sizeof(float2));
    };
    auto tile = [&] { return a.field + a.bstride * by + quad_index(0, bx * RPCr, NX); };
    auto lbase = [&] { return (lr >> 1) * (2 * NX) + (t >> 1) * 4 + (lr & 1) * 2 + (t & 1); };
    if constexpr (kBulk) {
        if (threadIdx.x == 0) {
            mbar_init(&rbar, 1);
            bulk_g2s(smem, tile(), tile_bytes(), &rbar);
        }
        __syncthreads();
        mbar_wait(&rbar, 0);
        const int lb = lbase();
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = smem[lb + e * 2 * T];
        __syncthreads();  // landing area becomes the exchange buffer
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = ld_stream(&fb[addr(e)]);
    }

    if constexpr (MODE == ROW_PLAIN) {
        // Propagator<float>::forward / inverse halves (propagation.hpp:81-95):
        // forward rows start from f*Q; inverse rows finish with *norm *conj(Q).
        const size_t rowbase = (size_t)yy * NX;
        if (a.sign < 0) {
            if (a.fresnel_q)
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmul_rn(v[e], __ldg(&a.fresnel_q[rowbase + t + e * T]));
            fft_line<NX, -1, Cfg::EM>(v, t, smem, idx, a.tw);
        } else {
            fft_line<NX, +1, Cfg::EM>(v, t, smem, idx, a.tw);
        }
        if (a.apply_norm)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], a.norm);
        if (a.sign > 0 && a.fresnel_q)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cmul_conj_rn(v[e], __ldg(&a.fresnel_q[rowbase + t + e * T]));
    } else {
#if !HG_NULL_COMPUTE  // diagnostic build: the passes' memory traffic alone
#if HG_ROW_VARIANT == 3  // diagnostic: the aperture-plane work twice per tile (compute without tile traffic)
#pragma unroll 1
        for (int rep = 0; rep < 2; ++rep)
#endif
        row_fused_body<NX, QK, FQ, LV, CtaSync, Cfg::EM>(v, t, yy, b, valid, smem, idx, a, sstates);  // (padding rows: row 0's side arrays)
#endif
    }
#ifndef HG_ROW_DIRECT_STORE  // bulk-loaded tiles stored by per-thread coalesced stores (no EXIT wait on the bulk read)
#define HG_ROW_DIRECT_STORE 0
#endif
    if constexpr (kBulk && !HG_ROW_DIRECT_STORE) {
        const int lb = opaque(lbase());
#pragma unroll
        for (int e = 0; e < E; ++e) smem[lb + e * 2 * T] = v[e];
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_s2g(tile(), smem, tile_bytes());
            bulk_commit();
            bulk_wait_read0();
        }
    } else if (valid) {
        float2* ob = opaque(fb);
#pragma unroll
        for (int e = 0; e < E; ++e) ob[addr(e)] = v[e];
    }
}

template <int NX, int MODE, int QK, int LAY, int FQ, int LV = 2>
__global__ void __launch_bounds__(RowCfg<NX, LAY>::THREADS, RowCfg<NX, LAY>::MIN_BLOCKS) k_row(RowArgs a) {
    row_cta<NX, MODE, QK, LAY, FQ, LV>(a, blockIdx.x, blockIdx.y);
}

// ------------------------------------------------ persistent row pass
// The fused row pass as a software pipeline (one 1024-thread CTA per SM):
// two groups of 512 threads each own an exchange buffer and take the CTA's
// tiles in turn (group k & 1 takes the CTA's k-th tile); one shared landing
// buffer receives the next tile by TMA while both groups compute.  A group
// copies its landed tile into registers, releases the landing buffer (the
// next tile's bulk load is issued at once), transforms, and bulk-stores the
// result from its exchange buffer without waiting for the write.  So tile
// traffic overlaps the transforms instead of alternating with them: the
// non-persistent pass costs its memory time plus its compute time (two
// resident CTAs per SM start, land, compute and store in phase).
// Per-group full barriers (full[g], one phase per tile of that group) keep
// the landing order unambiguous.  Smem: 2 x RowCfg::SMEM + one tile.
template <int NX>
struct RowPersistCfg {
    using Cfg = RowCfg<NX, LAY_QUAD>;
    static constexpr bool ok = Cfg::THREADS == 512 && NX > Cfg::E && Cfg::T >= 2;
    static constexpr int TILE = Cfg::RPC * NX * (int)sizeof(float2);
    static constexpr int SMEM = 2 * Cfg::SMEM + TILE;
    static_assert(Cfg::SMEM % 128 == 0, "bulk copies need 128-B aligned smem buffers");
};

template <int NX, int QK, int FQ, int LV>
__global__ void __launch_bounds__(1024, 1) k_row_persist(RowArgs a, int rowblocks, int ntiles) {
    using Cfg = RowCfg<NX, LAY_QUAD>;
    constexpr int E = Cfg::E, T = Cfg::T, RPC = Cfg::RPC;
    constexpr int TILE = RowPersistCfg<NX>::TILE;
    extern __shared__ __align__(128) float2 smem[];
    __shared__ uint64_t full[2];
    const int g = threadIdx.x >> 9, tg = threadIdx.x & 511;
    float2* xg = smem + g * (Cfg::SMEM / (int)sizeof(float2));  // this group's exchange buffer
    float2* land = smem + 2 * (Cfg::SMEM / (int)sizeof(float2));
    const GroupSync gsync{1 + g, 512};
    // thread mapping of k_row (a warp covers 2 rows x 16 consecutive x)
    const int pr = tg / (2 * T), q = tg % (2 * T);
    const int r = (q >> 1) & 1, t = ((q >> 2) << 1) | (q & 1);
    const int lr = 2 * pr + r;
    const RowSmemIdx idx{lr * RowStride<NX>::value};
    const int lb = (lr >> 1) * (2 * NX) + (t >> 1) * 4 + (lr & 1) * 2 + (t & 1);
    auto tile_ptr = [&](int s) {
        const int bx = s % rowblocks, by = s / rowblocks;
        return a.field + a.bstride * by + quad_index(0, bx * RPC, NX);
    };
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        if ((int)blockIdx.x < ntiles) bulk_g2s(land, tile_ptr(blockIdx.x), TILE, &full[0]);
    }
    __syncthreads();
    const bool leader = tg == 0;
#ifndef HG_ROWP_NOMEM  // diagnostic: the first tile only, no tile loads or stores after it (compute alone)
#define HG_ROWP_NOMEM 0
#endif
#if HG_ROWP_NOMEM
    mbar_wait(&full[0], 0);
#endif
#pragma unroll 1
    for (int k = g, s = blockIdx.x + g * G; s < ntiles; k += 2, s += 2 * G) {
        float2 v[E];
#if !HG_ROWP_NOMEM
        mbar_wait(&full[g], (k >> 1) & 1);
#endif
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = land[lb + e * 2 * T];
        if (leader) bulk_wait_read0();  // this group's previous store has left its exchange buffer
        gsync();                        // every thread of the group has its tile: release the landing buffer
        if (!HG_ROWP_NOMEM && leader && s + G < ntiles) bulk_g2s(land, tile_ptr(s + G), TILE, &full[g ^ 1]);
        const int bx = s % rowblocks, by = s / rowblocks;
        row_fused_body<NX, QK, FQ, LV, GroupSync, Cfg::EM>(v, t, bx * RPC + lr, by, true, xg, idx, a, nullptr, gsync);
        const int lbo = opaque(lb);
#pragma unroll
        for (int e = 0; e < E; ++e) xg[lbo + e * 2 * T] = v[e];
        fence_proxy_async();
        gsync();
        if (!HG_ROWP_NOMEM && leader) {
            bulk_s2g(tile_ptr(s), xg, TILE);
            bulk_commit();
        }
    }
    if (tg == 0) bulk_wait_read0();
}

// ------------------------------------------------------------- column pass
// COL_GS_FAST / COL_WGS_FAST: no ROI, no LT schedule, phase freedom (the
// benchmark configurations); COL_GS_GENERIC: every TargetSpec / variant.
// COL_OSPR_MID (+ quantiser kind << 4): the rows-first OSPR subframe's middle
// pass (ospr_rows.cuh): IFFT columns, *norm, quantise (+levels), FFT columns.
enum ColMode { COL_PLAIN = 0, COL_GS_GENERIC = 1, COL_OSPR = 2, COL_GS_FAST = 3, COL_WGS_FAST = 4, COL_OSPR_MID = 5 };
// The last iteration's GS column pass also reduces the diffraction-efficiency
// sums (a separate instantiation, so the K-1 others carry no extra registers).
constexpr int COL_EFF = 8;  // flag added to COL_GS_GENERIC / COL_GS_FAST / COL_WGS_FAST
__host__ __device__ constexpr int col_base_mode(int m) { return m & 7; }

struct ColArgs {
    const float2* tw;
    float2* field;
    size_t bstride;
    int nx;
    int layout;      // Layout (dispatch)
    float norm;
    int sign;        // COL_PLAIN
    int apply_norm;  // COL_PLAIN
    // replay-plane constraint (ifta.hpp:185-224)
    const float* target;  // fp32 amplitude [target][ny][nx]
    size_t t_bstride;
    const uint8_t* roi;   // [ny][nx] (shared) or nullptr
    float* weights;       // WGS [target][ny][nx] or nullptr
    const float2* tphase_cs;  // phase-freedom-off: (cos, sin) of target phase [target][ny][nx]
    int phase_freedom, amp_outside_roi, scale_free;
    float clamp_lo, clamp_hi;
    int lt, lt_x0, lt_x1, lt_y0, lt_y1;
    int last;             // last iteration: store R, skip constraint + IFFT
    int ckpt;             // with last: apply the constraint (+WGS weights) first and store the
                          // constrained R (the state iteration K+1 resumes from)
    float2* replay_out;   // where the last iteration's R goes (may alias field)
    double* partials;     // per block: 8 doubles
    // OSPR accumulation
    float* S;             // [job][ny][nx] running sum of |R|^2
    size_t S_bstride;
    float inv_n;          // 1/n for the cumulative replay sqrt(S/n)
    // quad-layout field as a 2-D TMA tensor map (inner: a quad row of 4*nx
    // floats, outer: quad rows); this launch's target b starts at quad row
    // tma_row0 + b * tma_brows.  nullptr: per-thread loads/stores.
    const void* tmap;
    int tma_row0, tma_brows;
    int cw;  // columns per CTA this launch (an instantiated width <= ColCfg::C; 0 = the default)
    // COL_OSPR_MID: the SLM quantiser and the frame's level indices (row-major)
    QuantParams q;
    uint8_t* levels8;
    size_t lv_bstride;
};

template <int NY, int LAY>
struct ColCfg {
#ifndef HG_COL_E8
#define HG_COL_E8 0
#endif
#ifndef HG_COL_TMA
#define HG_COL_TMA 1
#endif
    // EM = 8: 8 elements per thread, 1024-thread CTAs at <= 32 registers, 2 CTAs
    // (64 warps) per SM for the large quad-layout columns; else 16 per thread.
    static constexpr int EM = (HG_COL_E8 && LAY == LAY_QUAD && NY >= 2048) ? 8 : quad_em<NY, LAY>();
    static constexpr int E = LineCfg<NY, EM>::E, T = LineCfg<NY, EM>::T;
    // LAY_ROW: up to 128 KiB of complex64 per CTA (1 CTA / SM at 4096);
    // LAY_QUAD: 64 KiB column-pair tiles (2 CTAs / SM)
#ifndef HG_COLQ_BUDGET
#define HG_COLQ_BUDGET 8192
#endif
    static constexpr int BUDGET = LAY == LAY_QUAD ? HG_COLQ_BUDGET : 16384;
    static constexpr int CMAX0 = (BUDGET / NY) < 16 ? (BUDGET / NY) : 16;
    static constexpr int CMIN = LAY == LAY_QUAD ? 2 : 1;
    static constexpr int C = CMAX0 < CMIN ? CMIN : CMAX0;
    static constexpr int THREADS = T * C;
    static constexpr int MIN_BLOCKS =
        (HG_COL_E8 && LAY == LAY_QUAD && NY >= 2048) ? 2 : ((LAY == LAY_QUAD && THREADS >= 512 && THREADS < 1024) ? HG_COLQ_MINB : 1);
};

#ifndef HG_COL_TGT_BULK
#define HG_COL_TGT_BULK 1
#endif
// The target slice of a TMA column tile is contiguous in the column-pair
// layout (C*NY floats): one cp.async.bulk brings it into smem beside the
// tile at kernel start, read after the forward transform.
template <int NY, int C, int LAY, int MODE>
struct ColTgtBulk;

// Column tiles loaded / stored by 2-D TMA (k_col): quad-layout tiles of C
// columns (C/2 quads = 16*C bytes per quad row) and at least 256 quad rows,
// in boxes of 256 quad rows.  Their launches must carry ColArgs::tmap, whose
// box is {4*C floats, 256 quad rows}.
template <int NY, int C, int LAY>
struct ColTma {
    static constexpr bool on =
        HG_COL_TMA && LAY == LAY_QUAD && C >= 2 && NY >= 512 && NY > LineCfg<NY, ColCfg<NY, LAY>::EM>::E;
    static constexpr int kBoxRows = 256;
    // landing slot of element (column c, row y) of the tile: [quad row][quad][2x2]
    static __device__ __forceinline__ int slot(int c, int y) {
        if constexpr (C == 2) return 2 * y + c;  // = the unpadded [y][c] column layout
        else return (y >> 1) * (2 * C) + (c >> 1) * 4 + (y & 1) * 2 + (c & 1);
    }
};
template <int NY, int C, int LAY, int MODE>
struct ColTgtBulk {
    // GS / WGS: the fp32 target slice.  OSPR: the job's running intensity sum
    // S instead (read and written, always in HBM; the shared OSPR target stays
    // L2-resident and is read directly).
    static constexpr int M = col_base_mode(MODE);
    static constexpr bool on = HG_COL_TGT_BULK && ColTma<NY, C, LAY>::on && M != COL_PLAIN && M != COL_OSPR_MID;
    static constexpr bool target = on && M != COL_OSPR;
    static constexpr bool S = on && M == COL_OSPR;
    static constexpr int BYTES = on ? C * NY * (int)sizeof(float) : 0;
};
template <int NY, int C, int MODE, int LAY>
constexpr int col_smem_bytes() {
    return (NY > LineCfg<NY, ColCfg<NY, LAY>::EM>::E ? PaddedLen<NY>::value * C * (int)sizeof(float2) : 0) +
           ColTgtBulk<NY, C, LAY, MODE>::BYTES;
}


// Per-thread float partials -> warp sums in float (32 terms) -> per-warp
// doubles -> fixed-order double block sum; thread 0 stores NV doubles.
template <int NV, int DUP = -1>  // DUP >= 0: also store sum DUP into slot NV
__device__ __forceinline__ void block_sum_float_store(float (&v)[NV], double* out) {
    __shared__ double red[32][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) red[warp][i] = (double)v[i];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = lane < nw ? red[lane][i] : 0.0;
            x = warp_sum(x);
            if (lane == 0) {
                out[i] = x;
                if (DUP == i) out[NV] = x;
            }
        }
    }
}

// The column pass of one CTA: column block bx (C columns) of target by, of
// gx column blocks per target (the partial-sum slot).
template <int NY, int C, int MODE, int LAY>
__device__ __forceinline__ void col_cta(const ColArgs& a, const int bx, const int by, const int gx) {
    constexpr int M = col_base_mode(MODE);
    constexpr bool kEff = (MODE & COL_EFF) != 0;
    constexpr int EM = ColCfg<NY, LAY>::EM;
    constexpr int E = LineCfg<NY, EM>::E, T = LineCfg<NY, EM>::T;
    extern __shared__ __align__(128) float2 smem[];
    const int c = threadIdx.x % C, t = threadIdx.x / C;
    const int x = bx * C + c;
    const int b = by;
    const int nx = a.nx;
    ColSmemIdx<C> idx{c};
    // element e of this thread is row y = t + e*T.  Field offsets: per-thread
    // base + e*st (both layouts advance by T*nx elements per e when T is even);
    // side arrays (target, weights, S, roi): base sb + e*ss.
    size_t f0;
    int st;
    size_t sb;
    int ss;
    if constexpr (LAY == LAY_QUAD) {
        f0 = quad_index(x, t, nx);
        st = (T >= 2) ? T * nx : 0;
        sb = colpair_index(x, t, NY);
        ss = 2 * T;
    } else {
        f0 = (size_t)t * nx + x;
        st = T * nx;
        sb = f0;
        ss = st;
    }
    auto fofs = [&](int e) -> size_t {
        if constexpr (LAY == LAY_QUAD && T < 2) return quad_index(x, t + e * T, nx);
        else return f0 + (size_t)e * st;
    };
    float2* base = a.field + a.bstride * b;
    float2 v[E];
    // TMA path (quad tiles): the whole C-column tile lands in smem in its
    // global quad order, replacing 16 scattered global accesses of 8 B per
    // thread (8 L1 wavefronts per warp instruction at C = 2); the same buffer
    // then serves the FFT exchanges.
    using Tma = ColTma<NY, C, LAY>;
    constexpr bool kTma = Tma::on;
    constexpr int kBoxRows = Tma::kBoxRows, kBoxes = NY / 2 / kBoxRows;
    __shared__ uint64_t tbar;
    const int tq = bx * (C / 2) * 8;  // inner coordinate (floats) of this column pair
    const int tr = a.tma_row0 + b * a.tma_brows;
    constexpr bool kTgt = ColTgtBulk<NY, C, LAY, MODE>::target;
    constexpr bool kSB = ColTgtBulk<NY, C, LAY, MODE>::S;
    __shared__ uint64_t gbar;
    float* tsm = reinterpret_cast<float*>(smem + PaddedLen<NY>::value * C);
    if constexpr (kTma) {
        if (threadIdx.x == 0) {
            mbar_init(&tbar, 1);
#ifndef HG_COL_NOMEM  // diagnostic: no tile / target / S traffic (transforms on whatever is in smem)
#define HG_COL_NOMEM 0
#endif
#if HG_COL_NOMEM
            mbar_arrive_plain(&tbar);
#else
            mbar_expect_tx(&tbar, NY * C * (int)sizeof(float2));
#pragma unroll 1
            for (int k = 0; k < kBoxes; ++k)
                tma_load_2d(smem + k * kBoxRows * 2 * C, a.tmap, tq, tr + k * kBoxRows, &tbar);
#endif
            if constexpr (kTgt || kSB) {
                mbar_init(&gbar, 1);
#if HG_COL_NOMEM
                mbar_arrive_plain(&gbar);
#else
                const float* src = kTgt ? a.target + a.t_bstride * b : a.S + a.S_bstride * b;
                bulk_g2s(tsm, src + colpair_index(bx * C, 0, NY), (uint32_t)ColTgtBulk<NY, C, LAY, MODE>::BYTES,
                         &gbar);
#endif
            }
        }
        __syncthreads();  // barrier initialised before anyone waits
        mbar_wait(&tbar, 0);
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = smem[Tma::slot(c, t + e * T)];
        __syncthreads();  // landing area becomes the exchange buffer
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = ld_stream(&base[fofs(e)]);
    }
    // stores recompute their addresses from an opaque base (keeps 16 64-bit
    // pointers from living across the transforms)
    auto store_col = [&](float2* dst) {
        if constexpr (kTma) {  // dst is the tensor map's field (host-checked)
#pragma unroll
            for (int e = 0; e < E; ++e) smem[Tma::slot(c, t + e * T)] = v[e];
            fence_proxy_async();
            __syncthreads();
            if (threadIdx.x == 0 && !HG_COL_NOMEM) {
#pragma unroll 1
                for (int k = 0; k < kBoxes; ++k)
                    tma_store_2d(a.tmap, tq, tr + k * kBoxRows, smem + k * kBoxRows * 2 * C);
                bulk_commit();
                bulk_wait_read0();
            }
        } else {
            float2* p1 = opaque(dst);
#pragma unroll
            for (int e = 0; e < E; ++e) p1[fofs(e)] = v[e];
        }
    };

    if constexpr (M == COL_OSPR_MID) {
        // rows-first OSPR subframe (ospr.hpp:118-131 with the 2-D transforms'
        // halves regrouped): the row IFFT was done by the seed pass
        fft_line<NY, +1, EM>(v, t, smem, idx, a.tw);  // completes P^-1 (unnormalised)
        constexpr int QK = (MODE >> 4) & 3;
        uint8_t* __restrict__ lv = a.levels8 + a.lv_bstride * b;  // (set by the plan)
        const int i0 = t * nx + x, di = T * nx;  // row-major pixel index (levels, illumination): npix <= 2^24
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = i0 + e * di;
            const float2 f = cscale(v[e], a.norm);  // fftw_backend.cpp:121-123
            const int k = quant_decide_kind<QK>(a.q, f.x, f.y, i);  // quantise.hpp:211-215
            lv[i] = (uint8_t)k;
            if constexpr (QK == QK_BINARY) v[e] = k ? a.q.s1 : a.q.s0;
            else if constexpr (QK == QK_FULL) v[e] = __ldg(&a.q.states[k]);
            else v[e] = quant_state(a.q, k, i);
        }
        fft_line<NY, -1, EM>(v, t, smem, idx, a.tw);  // starts P (rows finish it)
        store_col(base);
        return;
    } else if constexpr (M == COL_PLAIN) {
        if (a.sign < 0) fft_line<NY, -1, EM>(v, t, smem, idx, a.tw);
        else fft_line<NY, +1, EM>(v, t, smem, idx, a.tw);
        if (a.apply_norm)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], a.norm);
        store_col(base);
        return;
    } else {
#if !HG_NULL_COMPUTE
        fft_line<NY, -1, EM>(v, t, smem, idx, a.tw);  // completes the forward transform
#endif
        const float norm = a.norm;
        const float* tg = a.target + a.t_bstride * b + sb;
        // target element e: from the bulk-loaded slice (same column-pair offsets) or global
        const int tso = (int)(sb - colpair_index(bx * C, 0, NY));
        if constexpr (kTgt) mbar_wait(&gbar, 0);
        auto tload = [&](int e) -> float {
            if constexpr (kTgt) return tsm[tso + e * ss];
            else return __ldg(&tg[e * ss]);
        };
        // partial sums per CTA.  GS modes: [0..2] the MSE sums (metrics.hpp:70-97:
        // (T-|R|)^2, T|R|, |R|^2 over the mask; sum T^2 is the same every
        // iteration and comes from the plan, hgc_ifta_plan::stt); the last
        // iteration (kEff) also [3] the replay power on the target's support
        // (T > 0, in the mask) and [4] the total replay power (fast modes: stored
        // as a copy of [2], no mask): the diffraction efficiency (k_finalize;
        // DESIGN.md §3, an extension).
        constexpr int NV = M == COL_OSPR ? 7 : (kEff ? (M == COL_GS_GENERIC ? 5 : 4) : 3);
        float acc[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[i] = 0.f;
        if constexpr (M == COL_GS_FAST || M == COL_WGS_FAST) {
            // GS/WGS, no ROI, phase freedom: mse partials (metrics.hpp:70-97) and
            // R <- amp * R/|R| (ifta.hpp:198-214), branch-free
            const bool last = a.last && !a.ckpt;  // skip the constraint
            float* w = M == COL_WGS_FAST ? a.weights + a.t_bstride * b + sb : nullptr;
            const float lo = a.clamp_lo, hi = a.clamp_hi;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const float2 R = cscale(v[e], norm);
                const float r2 = R.x * R.x + R.y * R.y;
                const float amp0 = tload(e);
                const float ri = rsqrtf(r2);                 // +inf at r2 == 0
                const float r = r2 > 0.f ? r2 * ri : 0.f;    // |R|
                const float d = amp0 - r;
                acc[0] = fmaf(d, d, acc[0]);
                acc[1] = fmaf(amp0, r, acc[1]);
                acc[2] += r2;
                if constexpr (kEff) acc[3] += amp0 > 0.f ? r2 : 0.f;
                float amp = amp0;
                if constexpr (M == COL_WGS_FAST) {
                    if (!last && amp0 > 0.f) {  // ifta.hpp:198-204
                        const float cand = w[e * ss] * amp0 * (r > 1e-12f ? ri : 1e12f);
                        const float wn = fminf(fmaxf(cand, lo), hi);
                        w[e * ss] = wn;
                        amp = amp0 * wn;
                    }
                }
                const float sc = amp * ri;
                v[e] = r2 > 0.f ? make_float2(R.x * sc, R.y * sc) : make_float2(amp, 0.f);
                if (last) v[e] = R;
            }
        } else if constexpr (M == COL_GS_GENERIC) {
            float* w = a.weights ? a.weights + a.t_bstride * b + sb : nullptr;
            const float2* tcs = a.tphase_cs ? a.tphase_cs + a.t_bstride * b + sb : nullptr;
            const uint8_t* roi = a.roi ? a.roi + sb : nullptr;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int y = t + e * T;
                const size_t so = (size_t)e * ss;
                float2 R = cscale(v[e], norm);
                const bool in_roi = !roi || roi[so];
                float amp = tload(e);
                float r = sqrtf(R.x * R.x + R.y * R.y);
                if (in_roi) {  // mse partials (metrics.hpp:70-97)
                    float d = amp - r;
                    acc[0] += d * d;
                    acc[1] += amp * r;
                    acc[2] += r * r;
                    if constexpr (kEff)
                        if (amp > 0.f) acc[3] += r * r;
                }
                if constexpr (kEff) acc[4] += r * r;
                if (!a.last || a.ckpt) {  // replay-plane constraint, ifta.hpp:190-223
                    if (in_roi) {
                        const bool active = !a.lt || (x >= a.lt_x0 && x < a.lt_x1 && y >= a.lt_y0 && y < a.lt_y1);
                        if (active) {
                            if (w && amp > 0.f) {
                                float cand = w[so] * amp / fmaxf(r, 1e-12f);
                                float wn = fminf(fmaxf(cand, a.clamp_lo), a.clamp_hi);
                                w[so] = wn;
                                amp *= wn;
                            }
                            if (a.phase_freedom) {
                                if (r > 0.f) {
                                    float sc = amp / r;
                                    R = make_float2(R.x * sc, R.y * sc);
                                } else {
                                    R = make_float2(amp, 0.f);
                                }
                            } else {
                                float2 cs = tcs[so];
                                R = make_float2(amp * cs.x, amp * cs.y);
                            }
                        }
                    } else if (!a.amp_outside_roi) {
                        R = make_float2(0.f, 0.f);
                    }
                }
                v[e] = R;
            }
        } else {  // COL_OSPR: ospr.hpp:134-145
            if constexpr (kSB) mbar_wait(&gbar, 0);
            float* S = kSB ? tsm + tso : a.S + a.S_bstride * b + sb;  // bulk-landed slice or global
            const float inv_n = a.inv_n;
            const uint8_t* roi = a.roi ? a.roi + sb : nullptr;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const float2 R = cscale(v[e], norm);
                const float I = R.x * R.x + R.y * R.y;
                const float sv = S[e * ss] + I;
                S[e * ss] = sv;
                const float m = (!roi || roi[e * ss]) ? 1.f : 0.f;
                const float amp = tload(e) * m;
                const float r = sqrtf(I) * m;
                const float d = amp - r;
                acc[0] = fmaf(d, d, acc[0]);
                acc[1] = fmaf(amp, r, acc[1]);
                acc[2] = fmaf(I, m, acc[2]);
                acc[3] = fmaf(amp, amp, acc[3]);
                const float rc = sqrtf(sv * inv_n) * m;
                const float dc = amp - rc;
                acc[4] = fmaf(dc, dc, acc[4]);
                acc[5] = fmaf(amp, rc, acc[5]);
                acc[6] = fmaf(rc, rc, acc[6]);
            }
        }
        if constexpr (M != COL_OSPR) {
            if (a.last) {
                store_col(a.replay_out + a.bstride * b);
            } else {
#if !HG_NULL_COMPUTE
                fft_line<NY, +1, EM>(v, t, smem, idx, a.tw);  // starts the next inverse transform
#endif
                store_col(base);
            }
        }
        const size_t blk = (size_t)by * gx + bx;
        if constexpr (kSB) {  // the updated S slice back to HBM in one bulk store
            fence_proxy_async();
            __syncthreads();
            if (threadIdx.x == 0) {
                bulk_s2g(a.S + a.S_bstride * b + colpair_index(bx * C, 0, NY), tsm,
                         (uint32_t)ColTgtBulk<NY, C, LAY, MODE>::BYTES);
                bulk_commit();
                bulk_wait_read0();
            }
        }
        block_sum_float_store<NV, (kEff && (M == COL_GS_FAST || M == COL_WGS_FAST)) ? 2 : -1>(acc,
                                                                                              a.partials + blk * 8);
    }
}

template <int NY, int C, int MODE, int LAY>
__global__ void __launch_bounds__(LineCfg<NY, ColCfg<NY, LAY>::EM>::T * C, ColCfg<NY, LAY>::MIN_BLOCKS)
    k_col(ColArgs a) {
    col_cta<NY, C, MODE, LAY>(a, blockIdx.x, blockIdx.y, gridDim.x);
}

}  // namespace hg
