// k_col_gs.cu — fused replay-plane pass of the IFTA loop.
#include "launch_impl.cuh"

namespace hg {
void col_gs(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    col_dispatch<COL_GS>(ny, a, batch, st, prepare);
}
}  // namespace hg
