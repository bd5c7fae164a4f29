// k_col_plain.cu — plain column transforms (first half of P^-1 in the plans'
// quad layout; the primitive FFT in row-major) and the column tiling rule.
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
    const int T = ny / (ny < 16 ? ny : 16);  // threads per column (LineCfg<ny>::T)
    while (cw > 2 && (long long)(nx / cw) * batch < sm_count() && T * (cw / 2) >= 64) cw /= 2;
    return cw;
}
}  // namespace hg
