// k_col_ospr.cu — OSPR replay pass: forward columns + intensity accumulation
// + per-frame and cumulative MSE partials.
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
void col_ospr(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    require_layout(a.layout, LAY_QUAD, "col_ospr");
    col_dispatch<COL_OSPR, LAY_QUAD>(ny, a, batch, st, prepare);
}
}  // namespace hg
