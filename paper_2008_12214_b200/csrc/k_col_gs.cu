// k_col_gs.cu — fused replay-plane pass of the IFTA loop (fast GS / WGS
// specialisations; the generic constraint lives in k_col_gsg.cu).
// The column passes run the transforms on scalar FP32 (measured faster there
// than packed: 5.38 vs 5.58 ms per 64 x 4096^2 GS column pass; the row pass,
// which also carries the quantiser, gains from packing: 6.17 vs 6.81 ms).
#ifndef HG_COL_FFT_SCALAR
#define HG_COL_FFT_SCALAR 1
#endif
#ifndef HG_FFT_SCALAR
#define HG_FFT_SCALAR HG_COL_FFT_SCALAR
#endif
#include "launch_impl.cuh"

namespace hg {
void col_gs_fast(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    if (prepare) {
        col_dispatch<COL_GS_FAST, LAY_QUAD>(ny, a, batch, st, true);
        col_dispatch<COL_WGS_FAST, LAY_QUAD>(ny, a, batch, st, true);
        return;
    }
    if (a.weights) col_dispatch<COL_WGS_FAST, LAY_QUAD>(ny, a, batch, st, false);
    else col_dispatch<COL_GS_FAST, LAY_QUAD>(ny, a, batch, st, false);
}
}  // namespace hg
