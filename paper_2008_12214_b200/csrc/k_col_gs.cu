// k_col_gs.cu — fused replay-plane pass of the IFTA loop (fast GS / WGS
// specialisations; the generic constraint lives in k_col_gsg.cu).
#include "launch_impl.cuh"

namespace hg {
void col_gs_fast(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    if (prepare) {
        col_dispatch<COL_GS_FAST, LAY_QUAD>(ny, a, batch, st, true);
        col_dispatch<COL_WGS_FAST, LAY_QUAD>(ny, a, batch, st, true);
        col_dispatch<COL_GS_FAST | COL_EFF, LAY_QUAD>(ny, a, batch, st, true);
        col_dispatch<COL_WGS_FAST | COL_EFF, LAY_QUAD>(ny, a, batch, st, true);
        return;
    }
    // the last iteration's pass also reduces the efficiency sums
    if (a.weights) {
        if (a.last) col_dispatch<COL_WGS_FAST | COL_EFF, LAY_QUAD>(ny, a, batch, st, false);
        else col_dispatch<COL_WGS_FAST, LAY_QUAD>(ny, a, batch, st, false);
    } else {
        if (a.last) col_dispatch<COL_GS_FAST | COL_EFF, LAY_QUAD>(ny, a, batch, st, false);
        else col_dispatch<COL_GS_FAST, LAY_QUAD>(ny, a, batch, st, false);
    }
}
}  // namespace hg
