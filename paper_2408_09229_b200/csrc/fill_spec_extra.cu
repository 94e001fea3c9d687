// fill_spec_extra.cu -- more compile-time-dims instantiations of the fused
// fill: the Gaussian at the dimensions users pick besides the registry's 4
// and BASELINE's 20 (the runtime-dims kernel is ~4x slower: its per-axis
// arrays live in local memory and it has no streamed sums, pair table or
// fixed-point histograms).  A separate translation unit so the build
// compiles it beside fill_spec.cu.
#include "fill_spec_common.h"

namespace vpb {

#define VPB_SPEC_LIST_EXTRA(X) \
  X(VPB_GAUSSIAN, 1)           \
  X(VPB_GAUSSIAN, 2)           \
  X(VPB_GAUSSIAN, 3)           \
  X(VPB_GAUSSIAN, 5)           \
  X(VPB_GAUSSIAN, 6)           \
  X(VPB_GAUSSIAN, 8)           \
  X(VPB_GAUSSIAN, 10)          \
  X(VPB_GAUSSIAN, 12)          \
  X(VPB_GAUSSIAN, 16)

int fill_is_specialised_extra(int id, int dims) {
#define X(I, D) if (id == I && dims == D) return 1;
  VPB_SPEC_LIST_EXTRA(X)
#undef X
  return 0;
}

cudaError_t launch_fill_extra(int id, int dims, int grid, size_t smem, cudaStream_t st,
                              const FillArgs &a) {
  bool ok = false;
#define X(I, D)                                                   \
  if (id == I && dims == D) {                                     \
    const cudaError_t e = launch_spec<I, D>(grid, smem, st, a, &ok); \
    if (ok) return e;                                             \
  }
  VPB_SPEC_LIST_EXTRA(X)
#undef X
  if (a.pairs) return cudaErrorInvalidValue;
  return launch_fill_generic(id, grid, smem, st, a);   // global-atomic histograms
}

cudaError_t fill_occupancy_extra(int id, int dims, int layout, size_t smem, int *ctas) {
#define X(I, D) if (id == I && dims == D) return occ_spec<I, D>(layout, smem, ctas);
  VPB_SPEC_LIST_EXTRA(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace vpb
