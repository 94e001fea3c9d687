// fill_spec.cu -- compile-time-dims instantiations of the fused fill kernel
// for the registry integrands at their registry dimension and the BASELINE
// configurations (cfg1/3: d=4, cfg2: d=8, cfg4: d=6, cfg5: d=20).
#include <atomic>

#include "fill_spec_common.h"

namespace vpb {


#define VPB_SPEC_LIST(X)          \
  X(VPB_GAUSSIAN, 4)              \
  X(VPB_GAUSSIAN, 20)             \
  X(VPB_RIDGE, 4)                 \
  X(VPB_MULTIPEAK, 8)             \
  X(VPB_GENZ_OSCILLATORY, 6)      \
  X(VPB_GENZ_PRODUCTPEAK, 6)      \
  X(VPB_SINEXP, 2)                \
  X(VPB_LINEAR, 10)               \
  X(VPB_COSINE, 10)               \
  X(VPB_EXPONENTIAL, 10)          \
  X(VPB_ROOS_ARNOLD, 10)          \
  X(VPB_MOROKOFF, 8)              \
  X(VPB_ASIAN_OPTION, 16)         \
  X(VPB_PATH_INTEGRAL, 7)

int fill_is_specialised(int id, int dims) {
#define X(I, D) if (id == I && dims == D) return 1;
  VPB_SPEC_LIST(X)
#undef X
  return fill_is_specialised_extra(id, dims);
}

cudaError_t launch_fill(int id, int dims, int grid, size_t smem, cudaStream_t st,
                        const FillArgs &a) {
  if (a.det) return launch_fill_generic(id, grid, smem, st, a);   // deterministic mode
#define X(I, D)                                                                  \
  if (id == I && dims == D) {                                                    \
    if (a.fx && a.pairs) return spec::launch_one<I, D, LAYOUT_PAIRS_FX>(grid, smem, st, a); \
    if (a.fx) return spec::launch_one<I, D, LAYOUT_EDGES_FX>(grid, smem, st, a);       \
    if (a.records) return spec::launch_one<I, D, LAYOUT_RECORDS>(grid, smem, st, a);   \
    if (a.pairs) return spec::launch_one<I, D, LAYOUT_PAIRS>(grid, smem, st, a);       \
    if (a.smem_hist) return spec::launch_one<I, D, LAYOUT_EDGES>(grid, smem, st, a);   \
  }
  VPB_SPEC_LIST(X)
#undef X
  if (fill_is_specialised_extra(id, dims)) return launch_fill_extra(id, dims, grid, smem, st, a);
  if (a.pairs) return cudaErrorInvalidValue;
  return launch_fill_generic(id, grid, smem, st, a);   // incl. global-atomic histograms
}

// ---- split (2-CTA cluster) kernels
#define VPB_SPLIT_LIST(X) X(VPB_GAUSSIAN, 20)

namespace {
template <int ID, int D>
cudaLaunchConfig_t split_config(int grid, size_t smem, cudaStream_t st,
                                cudaLaunchAttribute *attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)fill_nt<ID, D, LAYOUT_SPLIT>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}
template <int ID, int D, int L = LAYOUT_SPLIT>
cudaError_t split_attr() {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fill_kernel<ID, D, L>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  done.fetch_or(bit, std::memory_order_acq_rel);
  return cudaSuccess;
}
template <int ID, int D, int L>
cudaError_t launch_split_one(int grid, size_t smem, cudaStream_t st, const FillArgs &a) {
  cudaError_t e = split_attr<ID, D, L>();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = split_config<ID, D>(grid, smem, st, attr);
  return cudaLaunchKernelEx(&cfg, fill_kernel<ID, D, L>, a);
}
template <int ID, int D>
cudaError_t split_clusters_one(size_t smem, int *clusters) {
  cudaError_t e = split_attr<ID, D>();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = split_config<ID, D>(2, smem, nullptr, attr);
  return cudaOccupancyMaxActiveClusters(clusters, fill_kernel<ID, D, LAYOUT_SPLIT>, &cfg);
}
}  // namespace

int fill_has_split(int id, int dims) {
#define X(I, D) if (id == I && dims == D) return 1;
  VPB_SPLIT_LIST(X)
#undef X
  return 0;
}
int fill_split_nt(int id, int dims) {
#define X(I, D) if (id == I && dims == D) return fill_nt<I, D, LAYOUT_SPLIT>();
  VPB_SPLIT_LIST(X)
#undef X
  return 0;
}
cudaError_t launch_fill_split(int id, int dims, int grid, size_t smem, cudaStream_t st,
                              const FillArgs &a) {
#define X(I, D) \
  if (id == I && dims == D) return launch_split_one<I, D, LAYOUT_SPLIT>(grid, smem, st, a);
  VPB_SPLIT_LIST(X)
#undef X
  return cudaErrorInvalidValue;
}
cudaError_t fill_split_clusters(int id, int dims, size_t smem, int *clusters) {
#define X(I, D) if (id == I && dims == D) return split_clusters_one<I, D>(smem, clusters);
  VPB_SPLIT_LIST(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t fill_occupancy(int id, int dims, int layout, size_t smem, int *ctas) {
#define X(I, D)                                                                  \
  if (id == I && dims == D && layout != LAYOUT_RUNTIME) {                        \
    if (layout == LAYOUT_RECORDS) return spec::occ_one<I, D, LAYOUT_RECORDS>(smem, ctas); \
    if (layout == LAYOUT_PAIRS) return spec::occ_one<I, D, LAYOUT_PAIRS>(smem, ctas);  \
    return spec::occ_one<I, D, LAYOUT_EDGES>(smem, ctas);                              \
  }
  VPB_SPEC_LIST(X)
#undef X
  if (fill_is_specialised_extra(id, dims) && layout != LAYOUT_RUNTIME)
    return fill_occupancy_extra(id, dims, layout, smem, ctas);
  if (layout == LAYOUT_PAIRS) return cudaErrorInvalidValue;
  return fill_occupancy_generic(id, smem, ctas);
}

}  // namespace vpb
