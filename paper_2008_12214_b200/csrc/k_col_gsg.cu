// k_col_gsg.cu — generic replay-plane pass (ROI, LT schedule, fixed target
// phase, any variant) and the dispatch between fast and generic passes.
#include "launch_impl.cuh"

namespace hg {
void col_gs_fast(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare);

void col_gs(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    require_layout(a.layout, LAY_QUAD, "col_gs");
    if (prepare) {
        col_dispatch<COL_GS_GENERIC, LAY_QUAD>(ny, a, batch, st, true);
        col_dispatch<COL_GS_GENERIC | COL_EFF, LAY_QUAD>(ny, a, batch, st, true);
        col_gs_fast(ny, a, batch, st, true);
        return;
    }
    const bool fast = !a.roi && !a.lt && a.phase_freedom;
    if (fast) col_gs_fast(ny, a, batch, st, false);
    else if (a.last) col_dispatch<COL_GS_GENERIC | COL_EFF, LAY_QUAD>(ny, a, batch, st, false);
    else col_dispatch<COL_GS_GENERIC, LAY_QUAD>(ny, a, batch, st, false);
}
}  // namespace hg
