// k_col_ospr.cu — OSPR replay pass: forward columns + intensity accumulation
// + per-frame and cumulative MSE partials.
#include "launch_impl.cuh"

namespace hg {
void col_ospr(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    require_layout(a.layout, LAY_QUAD, "col_ospr");
    col_dispatch<COL_OSPR, LAY_QUAD>(ny, a, batch, st, prepare);
}
}  // namespace hg
