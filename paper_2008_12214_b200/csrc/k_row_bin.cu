// k_row_bin.cu — fused aperture-plane row pass with the QK_BINARY quantiser
// (quant.cuh), instantiated without (FQ = 0) and with (FQ = 1) Fresnel Q,
// and without (LV = 0, the non-final iterations) and with level output.
#include "launch_impl.cuh"

namespace hg {
void row_fused_binary(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    const bool lv = a.levels8 || a.levels16;
    if (prepare) {
        row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 0, 0>(nx, a, batch, st, true);
        row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 1, 0>(nx, a, batch, st, true);
        row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 0, 1>(nx, a, batch, st, true);
        row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 1, 1>(nx, a, batch, st, true);
        return;
    }
    if (a.fresnel_q) {
        if (lv) row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 1, 1>(nx, a, batch, st, false);
        else row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 1, 0>(nx, a, batch, st, false);
    } else {
        if (lv) row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 0, 1>(nx, a, batch, st, false);
        else row_dispatch_q<ROW_FUSED, QK_BINARY, LAY_QUAD, 0, 0>(nx, a, batch, st, false);
    }
}
}  // namespace hg
