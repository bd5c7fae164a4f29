// k_col_plain.cu — plain column transforms (first half of P^-1, primitive FFT)
// and the column-tiling rule shared by every column pass.
#include "launch_impl.cuh"

namespace hg {
void col_plain(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare) {
    col_dispatch<COL_PLAIN>(ny, a, batch, st, prepare);
}
int col_tiles(int nx, int ny) {
    int c = 1;
    switch (ny) {
#define HG_CT(N) \
    case N: c = col_width<N>(nx); break;
        HG_CT(2) HG_CT(4) HG_CT(8) HG_CT(16) HG_CT(32) HG_CT(64) HG_CT(128) HG_CT(256)
        HG_CT(512) HG_CT(1024) HG_CT(2048) HG_CT(4096)
#undef HG_CT
    }
    return nx / c;
}
}  // namespace hg
