// launch_impl.cuh — size/layout dispatch shared by the k_*.cu translation units.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "errors.h"
#include "launch.h"

namespace hg {

inline int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <class K>
inline void set_smem(K kernel, int bytes) {
    // (static shared memory counts against the 48 KB default too: opt in for any dynamic size)
    if (bytes > 0) CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// ------------------------------------------------------------------- rows
template <int NX, int MODE, int QK, int LAY, int FQ, int LV = 2>
inline void row_launch(const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    using Cfg = RowCfg<NX, LAY>;
    auto kern = k_row<NX, MODE, QK, LAY, FQ, LV>;
    if (prepare) {
        set_smem(kern, Cfg::SMEM);
        return;
    }
    int rpc = Cfg::RPC;
    if (LAY == LAY_QUAD && Cfg::RPC > 2) {  // small launches: fewer rows per CTA until every SM has one
        const int min_rpc = std::max(2, 64 / Cfg::T);
        while (rpc > min_rpc && (long long)((a.ny + rpc - 1) / rpc) * batch < sm_count()) rpc /= 2;
    }
    RowArgs ar = a;
    ar.rpc = rpc;
    dim3 grid((a.ny + rpc - 1) / rpc, batch);
    kern<<<grid, Cfg::T * rpc, Cfg::SMEM, st>>>(ar);
    CK(cudaGetLastError());
}

// Persistent pipelined row pass (k_row_persist): one 1024-thread CTA per SM
// over all (row block, target) tiles.  Used for the large fused launches
// (>= 2 tiles per SM); returns false when it does not apply.
inline bool row_persist_on() {
    static const bool on = [] {
        const char* e = getenv("HG_ROW_PERSIST");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}
template <int NX, int QK, int FQ, int LV>
inline bool row_persist_launch(const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    if constexpr (!RowPersistCfg<NX>::ok) {
        return false;
    } else {
        using Cfg = RowCfg<NX, LAY_QUAD>;
        auto kern = k_row_persist<NX, QK, FQ, LV>;
        if (prepare) {
            set_smem(kern, RowPersistCfg<NX>::SMEM);
            return true;
        }
        if (!row_persist_on() || a.ny % Cfg::RPC != 0) return false;
        const int rowblocks = a.ny / Cfg::RPC;
        const long long ntiles = (long long)rowblocks * batch;
        const int sms = sm_count();
        if (ntiles < 2LL * sms || ntiles > (1LL << 30)) return false;
        kern<<<sms, 1024, RowPersistCfg<NX>::SMEM, st>>>(a, rowblocks, (int)ntiles);
        CK(cudaGetLastError());
        return true;
    }
}
template <int QK, int FQ, int LV>
inline bool row_persist_dispatch(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    switch (nx) {
        case 1024: return row_persist_launch<1024, QK, FQ, LV>(a, batch, st, prepare);
        case 2048: return row_persist_launch<2048, QK, FQ, LV>(a, batch, st, prepare);
        case 4096: return row_persist_launch<4096, QK, FQ, LV>(a, batch, st, prepare);
        default: return false;
    }
}

// Which specialised quantiser a fused row pass can use (quant.cuh).
inline int quant_kind(const QuantParams& q) {
    const bool illum = q.illum_arg || q.illum || q.illum_unit;
    if (q.mode == 1 && !illum && !q.full_circle && q.levels == 2 && q.min_arg == 0.0 &&
        q.range == 3.1415926535897932384626433832795)
        return QK_BINARY;
    if (q.mode == 1 && !illum && q.full_circle && (q.levels & (q.levels - 1)) == 0 &&
        (!HG_STATES_SMEM || q.levels <= 256))
        return QK_FULL;  // (the fast path's mod L is a mask)
    return QK_GENERIC;
}

template <int MODE, int QK, int LAY, int FQ, int LV = 2>
inline void row_dispatch_q(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    switch (nx) {
#define HG_ROW(N) \
    case N: row_launch<N, MODE, QK, LAY, FQ, LV>(a, batch, st, prepare); break;
        HG_ROW(2) HG_ROW(4) HG_ROW(8) HG_ROW(16) HG_ROW(32) HG_ROW(64) HG_ROW(128) HG_ROW(256)
        HG_ROW(512) HG_ROW(1024) HG_ROW(2048) HG_ROW(4096)
#undef HG_ROW
        default: fail(HGC_EUNSUPPORTED, "row length unsupported");
    }
}

// ---------------------------------------------------------------- columns
template <int NY, int LAY>
inline int col_width(int nx) {
    int c = ColCfg<NY, LAY>::C;
    return c < nx ? c : nx;
}

template <int NY, int C, int MODE, int LAY>
inline void col_launch_c(const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    auto kern = k_col<NY, C, MODE, LAY>;
    constexpr int EM = ColCfg<NY, LAY>::EM;
    constexpr int smem = col_smem_bytes<NY, C, MODE, LAY>();
    if (prepare) {
        set_smem(kern, smem);
        return;
    }
    if (ColTma<NY, C, LAY>::on && !a.tmap) fail(HGC_ECUDA, "column pass: TMA tile launched without a tensor map");
    dim3 grid(a.nx / C, batch);
    kern<<<grid, LineCfg<NY, EM>::T * C, smem, st>>>(a);
    CK(cudaGetLastError());
}

template <int NY, int MODE, int LAY>
inline void col_launch(const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    constexpr int CM = ColCfg<NY, LAY>::C;
    if (prepare) {  // every width a launch may narrow to (col_width_rt): kernel attributes are per device
        if constexpr (CM >= 1 && LAY == LAY_ROW) col_launch_c<NY, 1, MODE, LAY>(a, batch, st, true);
        if constexpr (CM >= 2) col_launch_c<NY, 2, MODE, LAY>(a, batch, st, true);
        if constexpr (CM >= 4) col_launch_c<NY, 4, MODE, LAY>(a, batch, st, true);
        if constexpr (CM >= 8) col_launch_c<NY, 8, MODE, LAY>(a, batch, st, true);
        if constexpr (CM >= 16) col_launch_c<NY, 16, MODE, LAY>(a, batch, st, true);
        return;
    }
    switch (a.cw > 0 ? a.cw : col_width<NY, LAY>(a.nx)) {
        case 1: if constexpr (CM >= 1 && LAY == LAY_ROW) col_launch_c<NY, 1, MODE, LAY>(a, batch, st, prepare); break;
        case 2: if constexpr (CM >= 2) col_launch_c<NY, 2, MODE, LAY>(a, batch, st, prepare); break;
        case 4: if constexpr (CM >= 4) col_launch_c<NY, 4, MODE, LAY>(a, batch, st, prepare); break;
        case 8: if constexpr (CM >= 8) col_launch_c<NY, 8, MODE, LAY>(a, batch, st, prepare); break;
        case 16: if constexpr (CM >= 16) col_launch_c<NY, 16, MODE, LAY>(a, batch, st, prepare); break;
        default: fail(HGC_EUNSUPPORTED, "column tile unsupported");
    }
}

template <int MODE, int LAY>
inline void col_dispatch(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    switch (ny) {
#define HG_COL(N) \
    case N: col_launch<N, MODE, LAY>(a, batch, st, prepare); break;
        HG_COL(2) HG_COL(4) HG_COL(8) HG_COL(16) HG_COL(32) HG_COL(64) HG_COL(128) HG_COL(256)
        HG_COL(512) HG_COL(1024) HG_COL(2048) HG_COL(4096)
#undef HG_COL
        default: fail(HGC_EUNSUPPORTED, "column length unsupported");
    }
}

template <int LAY>
inline int col_tiles_lay(int nx, int ny) {
    int c = 1;
    switch (ny) {
#define HG_CT(N) \
    case N: c = col_width<N, LAY>(nx); break;
        HG_CT(2) HG_CT(4) HG_CT(8) HG_CT(16) HG_CT(32) HG_CT(64) HG_CT(128) HG_CT(256)
        HG_CT(512) HG_CT(1024) HG_CT(2048) HG_CT(4096)
#undef HG_CT
    }
    return nx / c;
}

inline void require_layout(int got, int want, const char* what) {
    if (got != want) fail(HGC_EUNSUPPORTED, std::string(what) + ": layout not instantiated");
}

}  // namespace hg
