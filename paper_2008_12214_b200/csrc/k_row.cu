// k_row.cu — instantiations of the row pass: the fused aperture-plane pass
// with the generic quantiser (quad layout; Fresnel Q and illumination decided
// at run time) and the plain row transform of the FftBackend / Propagator
// primitives (row-major).  The binary and full-circle quantisers live in
// k_row_bin.cu / k_row_full.cu, specialised on the presence of Fresnel Q.
#include "launch_impl.cuh"

namespace hg {
void row_fused(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    require_layout(a.layout, LAY_QUAD, "row_fused");
    if (prepare) {
        row_dispatch_q<ROW_FUSED, QK_GENERIC, LAY_QUAD, 2>(nx, a, batch, st, true);
        row_fused_binary(nx, a, batch, st, true);
        row_fused_full(nx, a, batch, st, true);
        return;
    }
    switch (quant_kind(a.q)) {
        case QK_BINARY: row_fused_binary(nx, a, batch, st, false); break;
        case QK_FULL: row_fused_full(nx, a, batch, st, false); break;
        default: row_dispatch_q<ROW_FUSED, QK_GENERIC, LAY_QUAD, 2>(nx, a, batch, st, false); break;
    }
}
void row_plain(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    require_layout(a.layout, LAY_ROW, "row_plain");
    row_dispatch_q<ROW_PLAIN, QK_GENERIC, LAY_ROW, 2>(nx, a, batch, st, prepare);
}
}  // namespace hg
