// k_row.cu — instantiations of the row pass (fused aperture-plane pass and
// the plain row transform of the FftBackend primitive).
#include "launch_impl.cuh"

namespace hg {
void row_fused(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    row_dispatch<ROW_FUSED>(nx, a, batch, st, prepare);
}
void row_plain(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare) {
    row_dispatch<ROW_PLAIN>(nx, a, batch, st, prepare);
}
}  // namespace hg
