// k_col_plain.cu — plain column transforms (first half of P^-1 in the plans'
// quad layout; the primitive FFT in row-major) and the column tiling rule.
#include "launch_impl.cuh"

namespace hg {
void col_plain(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    if (prepare) {
        col_dispatch<COL_PLAIN, LAY_ROW>(ny, a, batch, st, true);
        col_dispatch<COL_PLAIN, LAY_QUAD>(ny, a, batch, st, true);
        return;
    }
    if (a.layout == LAY_QUAD) col_dispatch<COL_PLAIN, LAY_QUAD>(ny, a, batch, st, false);
    else col_dispatch<COL_PLAIN, LAY_ROW>(ny, a, batch, st, false);
}
int col_tiles(int nx, int ny, int layout) {
    return layout == LAY_QUAD ? col_tiles_lay<LAY_QUAD>(nx, ny) : col_tiles_lay<LAY_ROW>(nx, ny);
}
int col_width_rt(int nx, int ny, int batch) {
    int cw = nx / col_tiles(nx, ny, LAY_QUAD);
    const int em = ny <= HG_SMALL_NMAX ? HG_SMALL_EM : 16;
    const int T = ny / (ny < em ? ny : em);  // threads per column (LineCfg<ny, ColCfg::EM>::T)
    while (cw > 2 && (long long)(nx / cw) * batch < sm_count() && T * (cw / 2) >= 64) cw /= 2;
    return cw;
}
}  // namespace hg
