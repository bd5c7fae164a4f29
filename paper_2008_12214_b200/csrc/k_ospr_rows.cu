// k_ospr_rows.cu — launches of the rows-first OSPR subframe (ospr_rows.cuh).
#include "launch_impl.cuh"
#include "ospr_rows.cuh"

namespace hg {

bool ospr_rows_supported(int nx, int ny) { return nx == 1024 && ny == 1024; }

int ospr_rows_tiles(int nx, int ny) { return ny / SeedRowCfg<1024>::RPC; }
int ospr_rows_len(int nx) { return SeedRowCfg<1024>::LEN; }

static __global__ void k_d2f(const double* in, float* out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];  // TargetSpec amplitude as the fp32 replay target (as to_colpair)
}
void ospr_rows_target(const double* amp, float* out, size_t n, cudaStream_t st) {
    k_d2f<<<(int)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(amp, out, n);
    CK(cudaGetLastError());
}

void ospr_rows_walk(const WalkArgs& a, cudaStream_t st) {
    k_mt_walk<<<(a.streams + kWalkWarps - 1) / kWalkWarps, 32 * kWalkWarps, 0, st>>>(a);
    CK(cudaGetLastError());
}

void ospr_rows_seed(int nx, const SeedRowArgs& a, int jobs, cudaStream_t st, bool prepare) {
    using SC = SeedRowCfg<1024>;
    static_assert(SC::ok, "seed-row tile");
    if (nx != 1024) fail(HGC_EUNSUPPORTED, "rows-first OSPR: row length not instantiated");
    if (prepare) {
        set_smem(k_ospr_seed_rows<1024>, SC::SMEM);
        return;
    }
    k_ospr_seed_rows<1024><<<dim3(a.chunks, jobs), kSeedThreads, SC::SMEM, st>>>(a);
    CK(cudaGetLastError());
}

void ospr_rows_acc(int nx, const RowAccArgs& a, int chunks, int jobs, cudaStream_t st, bool prepare) {
    using AC = RowAccCfg<1024>;
    static_assert(AC::ok, "row-acc tile");
    if (nx != 1024) fail(HGC_EUNSUPPORTED, "rows-first OSPR: row length not instantiated");
    if (prepare) {
        set_smem(k_ospr_row_acc<1024>, AC::SMEM);
        return;
    }
    k_ospr_row_acc<1024><<<dim3(chunks, jobs), 512, AC::SMEM, st>>>(a);
    CK(cudaGetLastError());
}

template <int QK>
static void col_mid_q(const ColArgs& a, int jobs, cudaStream_t st, bool prepare) {
    constexpr int MODE = COL_OSPR_MID | (QK << 4);
    if (prepare) {
        col_launch_c<1024, 2, MODE, LAY_QUAD>(a, jobs, st, true);
        col_launch_c<1024, 4, MODE, LAY_QUAD>(a, jobs, st, true);
        col_launch_c<1024, 8, MODE, LAY_QUAD>(a, jobs, st, true);
        return;
    }
    switch (a.cw) {
        case 2: col_launch_c<1024, 2, MODE, LAY_QUAD>(a, jobs, st, false); break;
        case 4: col_launch_c<1024, 4, MODE, LAY_QUAD>(a, jobs, st, false); break;
        case 8: col_launch_c<1024, 8, MODE, LAY_QUAD>(a, jobs, st, false); break;
        default: fail(HGC_EUNSUPPORTED, "rows-first OSPR: column tile not instantiated");
    }
}
void ospr_rows_mid(int ny, const ColArgs& a, int qk, int jobs, cudaStream_t st, bool prepare) {
    if (ny != 1024) fail(HGC_EUNSUPPORTED, "rows-first OSPR: column length not instantiated");
    switch (qk) {
        case QK_BINARY: col_mid_q<QK_BINARY>(a, jobs, st, prepare); break;
        case QK_FULL: col_mid_q<QK_FULL>(a, jobs, st, prepare); break;
        default: col_mid_q<QK_GENERIC>(a, jobs, st, prepare); break;
    }
}

}  // namespace hg
