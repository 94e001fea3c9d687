// fill_generic.cu -- runtime-dims (D = 0) fill kernels, one per integrand.
#include <atomic>

#include "fill_launch.h"

namespace vpb {

namespace {
template <int ID>
cudaError_t launch_g(int grid, size_t smem, cudaStream_t st, const FillArgs &a) {
  // the max-dynamic-shared-memory attribute is per device: one bit per ordinal
  static std::atomic<unsigned long long> attr{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(fill_kernel<ID, 0, LAYOUT_RUNTIME>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr.fetch_or(bit, std::memory_order_acq_rel);
  }
  fill_kernel<ID, 0, LAYOUT_RUNTIME><<<grid, FILL_NT, smem, st>>>(a);
  return cudaGetLastError();
}
template <int ID>
cudaError_t occ_g(size_t smem, int *ctas) {
  cudaError_t e = cudaFuncSetAttribute(fill_kernel<ID, 0, LAYOUT_RUNTIME>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, fill_kernel<ID, 0, LAYOUT_RUNTIME>, FILL_NT, smem);
}
}  // namespace

#define VPB_ALL_IDS(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13)

cudaError_t launch_fill_generic(int id, int grid, size_t smem, cudaStream_t st,
                                const FillArgs &a) {
#define X(I) if (id == I) return launch_g<I>(grid, smem, st, a);
  VPB_ALL_IDS(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t fill_occupancy_generic(int id, size_t smem, int *ctas) {
#define X(I) if (id == I) return occ_g<I>(smem, ctas);
  VPB_ALL_IDS(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace vpb
