// hist.cuh -- interval histograms from fill records (large d * n_intervals).
//
// kernels.accumulate's map part (vp/kernels.py:100-105):
//     map_w[j, iv_j] += w2,  map_counts[j, iv_j] += 1   for every run and axis j
// When the d*ng histograms do not fit in one SM's shared memory next to the
// map edges (cfg5: d = 20, ng = 1024 -> 246 KB of histograms + 164 KB of
// edges), the fill kernel writes per-run records instead -- the 16-bit
// intervals in groups of 8 axes and w2 -- for one chunk of runs at a time, and
// hist_records_kernel accumulates each axis group in shared memory.  Same
// layout and bank argument as the fill kernel's shared histograms: rows of
// 8 axes per interval, lanes update the axes in lane-rotated order.
//
// Each (group, CTA) owns a private slice in global memory that persists over
// the chunks of an iteration; rec_reduce_kernel sums the slices in CTA order
// (deterministic), exactly like hist_reduce_kernel does for the fill's slices.
#pragma once
#include <cstdint>

namespace vpb {

#ifndef VPB_HR_NT
#define VPB_HR_NT 512
#endif
constexpr int HR_NT = VPB_HR_NT;   // threads per CTA (two CTAs per SM)

__host__ __device__ inline size_t hist_records_smem(int ng) {
  return (size_t)ng * 8 * (sizeof(double) + sizeof(unsigned));
}

// grid (B, G): blockIdx.y = group g0 + y, covering record axes [8g, 8g + JN);
// JN = axes per group (compile time: the full groups of a chunk run in one
// launch, two CTAs per SM; a partial last group gets its own launch).  Group
// g's B slices start at hw_rec / hc_rec + g * B * ng * 8.
template <int JN>
__global__ void __launch_bounds__(HR_NT, 2)
    hist_records_kernel(const unsigned short *rec_iv, const double *rec_w2, long long rec_ch,
                        long long tile_lo, const Sched *sched, int ng, int g0,
                        double *hw_rec, unsigned *hc_rec, int first, const int *status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *s_hw = reinterpret_cast<double *>(smem_raw);
  unsigned *s_hc = reinterpret_cast<unsigned *>(smem_raw + (size_t)ng * 8 * sizeof(double));
  if (*status & 1) return;
  const Sched S = *sched;
  const long long run0 = tile_lo * FILL_TILE;              // chunk start relative to lo
  const long long n = max(0ll, min(rec_ch, S.hi - S.lo - run0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = g0 + (int)blockIdx.y;
  const size_t slice = ((size_t)g * gridDim.x + blockIdx.x) * ng * 8;
  double *gw = hw_rec + slice;
  unsigned *gc = hc_rec + slice;
  if (n == 0) {                                             // block-uniform
    if (first)
      for (int i = tid; i < ng * 8; i += HR_NT) { gw[i] = 0.0; gc[i] = 0u; }
    return;
  }
  for (int i = tid; i < ng * 8; i += HR_NT) {
    s_hw[i] = first ? 0.0 : gw[i];
    s_hc[i] = first ? 0u : gc[i];
  }
  __syncthreads();
  // Record slots are lane-interleaved per fill tile (slot = tile*TILE +
  // step*32 + lane holds run tile*TILE + lane*RPT + step, so a warp's record
  // stores are coalesced); the last tile of the shard may have empty slots.
  const long long nslots = (n + FILL_TILE - 1) / FILL_TILE * FILL_TILE;
  // warp w of CTA b takes span w*B + b of NW*B equal spans: the warps sharing
  // this CTA's histograms sit n/NW records apart (different strata)
  constexpr int NW = HR_NT / 32;
  const long long spans = (long long)NW * gridDim.x;
  const long long per = ((nslots + spans - 1) / spans + 31) / 32 * 32;
  const long long beg = ((long long)warp * gridDim.x + blockIdx.x) * per;
  const long long end = min(beg + per, nslots);
  const unsigned short *iv_g = rec_iv + (size_t)g * rec_ch * 8;
  const int rot = lane % JN;
  auto valid = [&](long long s) {
    const long long t = s / FILL_TILE, q = s - t * FILL_TILE;
    return t * FILL_TILE + (q & 31) * FILL_RPT + (q >> 5) < n;
  };
  // one record ahead in flight (the loop body is a chain of shared atomics)
  long long i = beg + lane;
  uint4 vn = make_uint4(0, 0, 0, 0);
  double wn = 0.0;
  if (i < end) { vn = *reinterpret_cast<const uint4 *>(iv_g + (size_t)i * 8); wn = rec_w2[i]; }
  for (; i < end; i += 32) {
    const uint4 v = vn;
    const double w2 = wn;
    if (i + 32 < end) {
      vn = *reinterpret_cast<const uint4 *>(iv_g + (size_t)(i + 32) * 8);
      wn = rec_w2[i + 32];
    }
    if (!valid(i)) continue;
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
    int idx[JN];
#pragma unroll
    for (int j = 0; j < JN; j++)
      idx[j] = (int)((wv[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) * 8 + j;
#pragma unroll
    for (int b = 1; b < JN; b <<= 1) {   // barrel rotation by rot
      const bool on = (rot & b) != 0;
      int t[JN];
#pragma unroll
      for (int j = 0; j < JN; j++) t[j] = on ? idx[(j + b) % JN] : idx[j];
#pragma unroll
      for (int j = 0; j < JN; j++) idx[j] = t[j];
    }
#pragma unroll
    for (int j = 0; j < JN; j++) {
      atomicAdd(&s_hw[idx[j]], w2);
      atomicAdd(&s_hc[idx[j]], 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < ng * 8; i += HR_NT) {
    gw[i] = s_hw[i];
    gc[i] = s_hc[i];
  }
}

// map_w[j][iv] = sum over CTAs b (in order) of the group-(j/8) slices;
// block (32 intervals x 8 partitions) as hist_reduce_kernel.
__global__ void rec_reduce_kernel(const double *hw_rec, const unsigned *hc_rec, int nparts,
                                  int dims, int ng, double *map_w, long long *map_counts,
                                  const int *status) {
  // dims = axes in the records (the map rows after the fill's own k0 axes;
  // map_w / map_counts point at row k0)
  __shared__ double sw[8][33];
  __shared__ long long sc[8][33];
  if (*status & 1) return;
  const long long i = (long long)blockIdx.x * 32 + threadIdx.x;   // flat [j][iv]
  const long long m = (long long)dims * ng;
  const int p = threadIdx.y;
  const int per = (nparts + 7) / 8;
  const int b0 = p * per, b1 = min(nparts, b0 + per);
  double w = 0.0;
  long long c = 0;
  if (i < m) {
    const int j = (int)(i / ng), iv = (int)(i - (long long)j * ng);
    const size_t gbase = (size_t)(j >> 3) * nparts * ng * 8;
    const size_t off = (size_t)iv * 8 + (j & 7);
    for (int b = b0; b < b1; b++) {
      w = __dadd_rn(w, hw_rec[gbase + (size_t)b * ng * 8 + off]);
      c += hc_rec[gbase + (size_t)b * ng * 8 + off];
    }
  }
  sw[p][threadIdx.x] = w;
  sc[p][threadIdx.x] = c;
  __syncthreads();
  if (p == 0 && i < m) {
    double t = sw[0][threadIdx.x];
    long long k = sc[0][threadIdx.x];
    for (int q = 1; q < 8; q++) { t = __dadd_rn(t, sw[q][threadIdx.x]); k += sc[q][threadIdx.x]; }
    map_w[i] = t;
    map_counts[i] = k;
  }
}

}  // namespace vpb
