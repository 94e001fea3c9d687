// fill_launch.h -- dispatch from (integrand id, dims) to a compiled fill kernel.
#pragma once
#include <cuda_runtime.h>

#include "fill.cuh"

namespace vpb {

// Launch the fill kernel for (id, dims).  Uses the compile-time-dims kernel
// when one is instantiated (fill_spec.cu), else the generic runtime-dims one
// (fill_generic.cu).  `grid` CTAs of FILL_NT threads, `smem` dynamic bytes.
// a.records / a.pairs / a.smem_hist select the layout of a specialised
// (id, dims) kernel; global-atomic histograms use the generic kernel.
cudaError_t launch_fill(int id, int dims, int grid, size_t smem, cudaStream_t st,
                        const FillArgs &a);
// CTAs per SM the chosen kernel can keep resident with `smem` bytes.
cudaError_t fill_occupancy(int id, int dims, int layout, size_t smem, int *ctas_per_sm);
// 1 if (id, dims) has a compile-time specialisation.
int fill_is_specialised(int id, int dims);

// The split fill (LAYOUT_SPLIT: 2-CTA clusters, half the axes per CTA) for
// (id, dims) if compiled; its launch (cluster dims 2) and the clusters that
// can be resident at once with `smem` bytes per CTA.
int fill_has_split(int id, int dims);
cudaError_t launch_fill_split(int id, int dims, int grid, size_t smem, cudaStream_t st,
                              const FillArgs &a);
cudaError_t fill_split_clusters(int id, int dims, size_t smem, int *clusters);
int fill_split_nt(int id, int dims);

// generic kernels (fill_generic.cu)
cudaError_t launch_fill_generic(int id, int grid, size_t smem, cudaStream_t st,
                                const FillArgs &a);
cudaError_t fill_occupancy_generic(int id, size_t smem, int *ctas);

}  // namespace vpb
