// fill_spec_common.h -- the per-(integrand, dims, layout) launch and
// occupancy helpers shared by the specialisation translation units
// (fill_spec.cu: the registry and BASELINE configurations; fill_spec_extra.cu:
// more dimensions of the Gaussian, compiled in parallel).
#pragma once
#include <atomic>

#include "fill_launch.h"

namespace vpb {

namespace spec {
template <int ID, int D, int LAYOUT>
cudaError_t launch_one(int grid, size_t smem, cudaStream_t st, const FillArgs &a) {
  // the max-dynamic-shared-memory attribute is per device: one bit per ordinal
  static std::atomic<unsigned long long> attr{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(fill_kernel<ID, D, LAYOUT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr.fetch_or(bit, std::memory_order_acq_rel);
  }
  fill_kernel<ID, D, LAYOUT><<<grid, (fill_nt<ID, D, LAYOUT>()), smem, st>>>(a);
  return cudaGetLastError();
}
template <int ID, int D, int LAYOUT>
cudaError_t occ_one(size_t smem, int *ctas) {
  cudaError_t e = cudaFuncSetAttribute(fill_kernel<ID, D, LAYOUT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, fill_kernel<ID, D, LAYOUT>, fill_nt<ID, D, LAYOUT>(),
                                                       smem);
}
}  // namespace spec

// dispatch of one compiled (ID, D) to its layout (FX first: fixed-point
// histograms, then records, pairs, edge rows)
template <int ID, int D>
cudaError_t launch_spec(int grid, size_t smem, cudaStream_t st, const FillArgs &a, bool *ok) {
  *ok = true;
  if (a.fx && a.pairs) return spec::launch_one<ID, D, LAYOUT_PAIRS_FX>(grid, smem, st, a);
  if (a.fx) return spec::launch_one<ID, D, LAYOUT_EDGES_FX>(grid, smem, st, a);
  if (a.records) return spec::launch_one<ID, D, LAYOUT_RECORDS>(grid, smem, st, a);
  if (a.pairs) return spec::launch_one<ID, D, LAYOUT_PAIRS>(grid, smem, st, a);
  if (a.smem_hist) return spec::launch_one<ID, D, LAYOUT_EDGES>(grid, smem, st, a);
  *ok = false;
  return cudaSuccess;
}
template <int ID, int D>
cudaError_t occ_spec(int layout, size_t smem, int *ctas) {
  if (layout == LAYOUT_RECORDS) return spec::occ_one<ID, D, LAYOUT_RECORDS>(smem, ctas);
  if (layout == LAYOUT_PAIRS) return spec::occ_one<ID, D, LAYOUT_PAIRS>(smem, ctas);
  return spec::occ_one<ID, D, LAYOUT_EDGES>(smem, ctas);
}

// fill_spec_extra.cu
int fill_is_specialised_extra(int id, int dims);
cudaError_t launch_fill_extra(int id, int dims, int grid, size_t smem, cudaStream_t st,
                              const FillArgs &a);
cudaError_t fill_occupancy_extra(int id, int dims, int layout, size_t smem, int *ctas);

}  // namespace vpb
