// launch.h — host entry points of the per-size kernel instantiations, one
// translation unit per pass family so they compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include "ospr_rows_args.h"
#include "passes.cuh"

namespace hg {

// prepare = true only sets the kernel attributes (dynamic shared memory);
// call it outside stream capture before the first launch of a size.
// The layout comes from args.layout: fused passes exist for LAY_QUAD (plans),
// plain transforms for both layouts.
void row_fused(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare = false);
void row_plain(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare = false);
// specialised fused row passes, one translation unit each (k_row_bin.cu, k_row_full.cu)
void row_fused_binary(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare);
void row_fused_full(int nx, const RowArgs& a, int batch, cudaStream_t st, bool prepare);
// unitary complex128 2-D transform in place (k_fft64.cu)
void fft2d_f64(double2* f, int nx, int ny, int sign, int batch, cudaStream_t st);
// any nx, ny >= 1 (Bluestein for non-powers of two <= 2048), in double (k_fft64.cu)
void fft2d_any_f64(double2* f, int nx, int ny, int sign, int batch, cudaStream_t st);
void col_plain(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare = false);
void col_gs(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare = false);
void col_ospr(int ny, const ColArgs& a, int batch, cudaStream_t st, bool prepare = false);
// Column tiles (CTAs) per target of the column pass for an nx x ny field.
int col_tiles(int nx, int ny, int layout);
// Quad-layout column width for a launch over `batch` targets: the default
// tile, halved while the launch would leave SMs idle (< 1 CTA per SM), at
// least 64 threads per CTA.  The plans use it for the launches, the TMA box
// and the number of partial-sum tiles (nx / width).
int col_width_rt(int nx, int ny, int batch);

// Rows-first OSPR subframe (ospr_rows.cuh, k_ospr_rows.cu): field sizes with
// instantiated kernels, tiles (row blocks) per job, draws per tile.
bool ospr_rows_supported(int nx, int ny);
int ospr_rows_tiles(int nx, int ny);
int ospr_rows_len(int nx);
void ospr_rows_target(const double* amp, float* out, size_t n, cudaStream_t st);
void ospr_rows_walk(const WalkArgs& a, cudaStream_t st);
void ospr_rows_seed(int nx, const SeedRowArgs& a, int jobs, cudaStream_t st, bool prepare = false);
void ospr_rows_mid(int ny, const ColArgs& a, int qk, int jobs, cudaStream_t st, bool prepare = false);
void ospr_rows_acc(int nx, const RowAccArgs& a, int chunks, int jobs, cudaStream_t st, bool prepare = false);

}  // namespace hg
