// ospr_rows_args.h — launch arguments of the rows-first OSPR subframe
// kernels (ospr_rows.cuh), shared with the plan (ospr_plan.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace hg {
struct MtState;

struct WalkArgs {
    MtState* states;         // [streams]: the window holding the next draw (carried frame to frame)
    const uint64_t* seeds;   // [streams] engine seeds (first frame) or nullptr = continue from states
    MtState* ck;             // [streams][chunks]: window + position of each tile's first draw
    int streams, chunks, len;  // a frame is chunks * len draws
    uint64_t* raw;           // instead of ck: every raw (untempered) word of the frame, [streams][chunks * len]
};
struct SeedRowArgs {
    const MtState* ck;   // [jobs][chunks] (k_mt_walk)
    const uint64_t* raw; // or the frame's raw words [jobs][npix] (k_mt_walk with raw)
    const double* amp;   // amplitude (double), per job stride amp_stride (0: shared)
    size_t amp_stride;
    float2* field;       // quad layout, per job stride npix
    size_t npix;
    const float2* tw;
    int chunks;          // tiles per job = ny / RPC
};

struct RowAccArgs {
    const float2* field;  // quad layout, per job stride npix
    size_t npix;
    const float2* tw;
    float norm, inv_n;    // 1/sqrt(nx*ny); 1/n for the cumulative replay sqrt(S/n)
    float* S;             // [job][ny][nx] row-major running sum of |R|^2
    const float* target;  // fp32 amplitude, row-major, per job stride t_bstride (0: shared)
    size_t t_bstride;
    const uint8_t* roi;   // [ny][nx] row-major or nullptr
    double* partials;     // [job][tiles][8]
};

}  // namespace hg
