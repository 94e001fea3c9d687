// update.cuh -- plan, results, allocation and refinement kernels.
//
//   strat.build_run_plan          vp/strat.py:131-137   alloc/scan/offsets kernels
//   strat.compute_results         vp/strat.py:183-208   results_leaf + pw_tree kernels
//   strat.update_evals_per_cube   vp/strat.py:88-113    results_leaf (pow) + alloc kernel
//   maps.smooth_and_damp          vp/maps.py:160-199    refine_kernel
//   maps.update_grid              vp/maps.py:202-234    refine_kernel
//
// All of them are deterministic and atomic-free, so every rank computes the
// same replicated update from the all-reduced accumulators.  numpy's pairwise
// summation tree is reproduced exactly: the host builds the
// tree for a given length once (PwPlan in capi.cu); leaves run in parallel,
// inner nodes combine level by level in one CTA.
#pragma once
#include <cstdint>

#include "devmath.cuh"
#include "fill.cuh"

namespace vpb {

struct PwPlanDev {
  const long long *leaf_off;   // [L]
  const int *leaf_len;         // [L]
  const int *node_l, *node_r;  // [I] children ids (leaves 0..L-1, inner L..)
  const int *level_start;      // [H+1] inner nodes grouped by height
  int L, I, H;
};

// numpy's `array ** scalar` fast paths, else pow.
__device__ __forceinline__ double np_scalar_pow(double x, double e) {
  if (e == 1.0) return x;
  if (e == 2.0) return __dmul_rn(x, x);
  if (e == 0.5) return __dsqrt_rn(x);
  if (e == 0.0) return 1.0;
  return pow(x, e);
}

// ---------------------------------------------------------------- results --
// Per cube (vp/strat.py:199-207): c = n_h (every planned run was evaluated
// once), m = s1/c, rv = max(s2/c - m*m, 0), d_h = sqrt(rv)*V, and for the
// allocation dp = d_h**beta.  Leaf partial sums of m, rv/c and dp follow
// numpy's 8-accumulator leaf exactly: 8 lanes per leaf, lane j owns
// accumulator r[j] (elements j, j+8, ...), the lanes combine as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) (IEEE addition is commutative, so the
// butterfly gives numpy's bits), and lane 0 adds the tail sequentially.
__device__ __forceinline__ void cube_terms(const double *s1, const double *s2,
                                           const long long *offsets, long long h, double V,
                                           double beta, bool want_dp, double *d_h, double *dp,
                                           double &m, double &t, double &p) {
  const double c = (double)(offsets[h + 1] - offsets[h]);
  m = __ddiv_rn(s1[h], c);
  double rv = __dadd_rn(__ddiv_rn(s2[h], c), -__dmul_rn(m, m));
  rv = (rv < 0.0) ? 0.0 : rv;   // np.maximum(rv, 0) keeps NaN
  t = __ddiv_rn(rv, c);
  const double dh = __dmul_rn(__dsqrt_rn(rv), V);
  d_h[h] = dh;
  p = 0.0;
  if (want_dp) {
    p = np_scalar_pow(dh, beta);
    dp[h] = p;
  }
}

// numpy's pairwise leaf over precomputed per-cube terms (terms[0|n|2n]): 8
// lanes per leaf, lane j owns accumulator r[j] -- the cooperative update's
// second phase (update_coop_kernel)
__device__ void results_leaf_body(long long gt, const double *terms, long long n, PwPlanDev pw,
                                  double *vals) {
  const int leaf = (int)(gt >> 3), j = (int)(gt & 7);
  const bool live = leaf < pw.L;
  const long long o = live ? pw.leaf_off[leaf] : 0;
  const int len = live ? pw.leaf_len[leaf] : 0;
  const double *tm = terms, *tt = terms + n, *tp = terms + 2 * n;
  double rm = 0.0, rt = 0.0, rp = 0.0;
  const int full = len < 8 ? 0 : len - (len % 8);
  if (live && len >= 8) {
    rm = tm[o + j]; rt = tt[o + j]; rp = tp[o + j];
    for (int i = 8 + j; i < full; i += 8) {
      rm = __dadd_rn(rm, tm[o + i]); rt = __dadd_rn(rt, tt[o + i]); rp = __dadd_rn(rp, tp[o + i]);
    }
  }
#pragma unroll
  for (int x = 1; x < 8; x <<= 1) {   // pairs, then quads, then halves
    const double om = __shfl_xor_sync(0xffffffffu, rm, x);
    const double ot = __shfl_xor_sync(0xffffffffu, rt, x);
    const double op = __shfl_xor_sync(0xffffffffu, rp, x);
    rm = __dadd_rn(rm, om); rt = __dadd_rn(rt, ot); rp = __dadd_rn(rp, op);
  }
  if (!live || j != 0) return;
  if (len < 8) { rm = 0.0; rt = 0.0; rp = 0.0; }
  for (int i = full; i < len; i++) {   // numpy's sequential tail (or n < 8)
    rm = __dadd_rn(rm, tm[o + i]); rt = __dadd_rn(rt, tt[o + i]); rp = __dadd_rn(rp, tp[o + i]);
  }
  vals[3 * leaf + 0] = rm;
  vals[3 * leaf + 1] = rt;
  vals[3 * leaf + 2] = rp;
}


// cube_terms_kernel + results_leaf_kernel in one launch without serialising
// the per-cube divisions/sqrt/pow: 128 threads per leaf (leaves have <= 128
// cubes) compute one cube's terms each into shared memory, then 8 lanes sum
// the leaf exactly as results_leaf_body (numpy's 8 accumulators, the fixed
// combine, the sequential tail).  8 leaves per 1024-thread block.
constexpr int TL_LEAVES = 8;
__global__ void __launch_bounds__(1024) results_terms_leaf_kernel(
    const double *s1, const double *s2, const long long *offsets, long long n, double V,
    double beta, double *d_h, double *dp, PwPlanDev pw, double *vals, const int *status) {
  __shared__ double tm[TL_LEAVES][128], tt[TL_LEAVES][128], tp[TL_LEAVES][128];
  if (*status & 1) return;
  const int slot = threadIdx.x >> 7, e = threadIdx.x & 127;
  const int leaf = blockIdx.x * TL_LEAVES + slot;
  const bool live = leaf < pw.L;
  const long long o = live ? pw.leaf_off[leaf] : 0;
  const int len = live ? pw.leaf_len[leaf] : 0;
  if (e < len) {
    double m, t, q;
    cube_terms(s1, s2, offsets, o + e, V, beta, beta != 0.0, d_h, dp, m, t, q);
    tm[slot][e] = m;
    tt[slot][e] = t;
    tp[slot][e] = q;
  }
  __syncthreads();
  if (e >= 8) return;   // lanes 0..7 of the leaf's first warp: numpy's accumulators
  const int j = e;
  double rm = 0.0, rt = 0.0, rp = 0.0;
  const int full = len < 8 ? 0 : len - (len % 8);
  if (len >= 8) {
    rm = tm[slot][j]; rt = tt[slot][j]; rp = tp[slot][j];
    for (int i = 8 + j; i < full; i += 8) {
      rm = __dadd_rn(rm, tm[slot][i]); rt = __dadd_rn(rt, tt[slot][i]);
      rp = __dadd_rn(rp, tp[slot][i]);
    }
  }
#pragma unroll
  for (int x = 1; x < 8; x <<= 1) {   // pairs, then quads, then halves (lanes 0-7 only)
    const double om = __shfl_xor_sync(0xffu, rm, x);
    const double ot = __shfl_xor_sync(0xffu, rt, x);
    const double op = __shfl_xor_sync(0xffu, rp, x);
    rm = __dadd_rn(rm, om); rt = __dadd_rn(rt, ot); rp = __dadd_rn(rp, op);
  }
  if (!live || j != 0) return;
  if (len < 8) { rm = 0.0; rt = 0.0; rp = 0.0; }
  for (int i = full; i < len; i++) {
    rm = __dadd_rn(rm, tm[slot][i]); rt = __dadd_rn(rt, tt[slot][i]);
    rp = __dadd_rn(rp, tp[slot][i]);
  }
  vals[3 * leaf + 0] = rm;
  vals[3 * leaf + 1] = rt;
  vals[3 * leaf + 2] = rp;
}

// Generic leaf kernel for a plain array (parity entry point vpb_pairwise_sum).
__global__ void array_leaf_kernel(const double *a, PwPlanDev pw, double *vals) {
  const int leaf = blockIdx.x * blockDim.x + threadIdx.x;
  if (leaf >= pw.L) return;
  vals[3 * leaf] = pw_leaf(a + pw.leaf_off[leaf], pw.leaf_len[leaf]);
  vals[3 * leaf + 1] = 0.0;
  vals[3 * leaf + 2] = 0.0;
}

// Inner nodes of the pairwise tree, by height, one CTA; three sums at once.
// Shared-memory staging (`flags`, from pw_tree_flags): bit 0 -- the leaf
// values are copied into `sm` and every level combines there; bit 1 -- the
// node tables (children, level starts) are copied too, so the H dependent
// levels read no global memory (after an L2 flush each level's index loads
// were a DRAM round trip).  Without staging the levels combine in `vals`.
__device__ void pw_tree_combine(PwPlanDev pw, double *vals, unsigned char *sm = nullptr,
                                int flags = 0) {
  double *v = vals;
  const int *nl = pw.node_l, *nr = pw.node_r, *ls = pw.level_start;
  unsigned char *p = sm;
  if (flags & 1) {
    double *sv = reinterpret_cast<double *>(p);
    for (int i = threadIdx.x; i < 3 * pw.L; i += blockDim.x) sv[i] = vals[i];
    v = sv;
    p += sizeof(double) * 3 * (size_t)(pw.L + pw.I);
  }
  if (flags & 2) {
    int *si = reinterpret_cast<int *>(p);
    for (int i = threadIdx.x; i < pw.I; i += blockDim.x) {
      si[i] = pw.node_l[i];
      si[pw.I + i] = pw.node_r[i];
    }
    for (int i = threadIdx.x; i <= pw.H; i += blockDim.x) si[2 * pw.I + i] = pw.level_start[i];
    nl = si;
    nr = si + pw.I;
    ls = si + 2 * pw.I;
  }
  if (flags) __syncthreads();
  for (int h = 0; h < pw.H; h++) {
    for (int i = ls[h] + threadIdx.x; i < ls[h + 1]; i += blockDim.x) {
      const int l = nl[i], r = nr[i], me = pw.L + i;
#pragma unroll
      for (int c = 0; c < 3; c++) v[3 * me + c] = __dadd_rn(v[3 * l + c], v[3 * r + c]);
    }
    __syncthreads();
  }
  if ((flags & 1) && threadIdx.x < 3) {   // the root, for the caller
    const int root = pw.I > 0 ? pw.L + pw.I - 1 : 0;
    vals[3 * root + threadIdx.x] = v[3 * root + threadIdx.x];
  }
  __syncthreads();
}

constexpr size_t PW_TREE_SMEM_MAX = 220 * 1024;
inline size_t pw_tree_vals_bytes(const PwPlanDev &pw) {
  return sizeof(double) * 3 * (size_t)(pw.L + pw.I);
}
inline size_t pw_tree_idx_bytes(const PwPlanDev &pw) {
  return sizeof(int) * (2 * (size_t)pw.I + pw.H + 1);
}
// staging flags for pw_tree_combine: values and tables if both fit, else the
// tables alone
inline int pw_tree_flags(const PwPlanDev &pw) {
  const size_t vb = pw_tree_vals_bytes(pw), ib = pw_tree_idx_bytes(pw);
  if (vb + ib <= PW_TREE_SMEM_MAX) return 3;
  return ib <= PW_TREE_SMEM_MAX ? 2 : 0;
}
inline size_t pw_tree_smem(const PwPlanDev &pw) {
  const int f = pw_tree_flags(pw);
  return ((f & 1) ? pw_tree_vals_bytes(pw) : 0) + ((f & 2) ? pw_tree_idx_bytes(pw) : 0);
}

struct Scalars {
  double estimate, variance, total_dp;
  int valid;
};

// Finishes compute_results (vp/strat.py:205-207) and records the history.
__device__ void results_tree_body(unsigned char *tree_sm, PwPlanDev pw, double *vals, long long n,
                                  double V, Scalars *sc, double *hist_est, double *hist_var,
                                  Sched *sched, int record, int flags) {
  pw_tree_combine(pw, vals, tree_sm, flags);
  if (threadIdx.x == 0) {
    const int root = pw.I > 0 ? pw.L + pw.I - 1 : 0;
    const double sm = vals[3 * root], st = vals[3 * root + 1], sp = vals[3 * root + 2];
    sc->estimate = __ddiv_rn(sm, (double)n);
    sc->variance = __dmul_rn(__dmul_rn(st, V), V);
    sc->total_dp = sp;
    sc->valid = 1;
    if (record) {
      hist_est[sched->it] = sc->estimate;
      hist_var[sched->it] = sc->variance;
    }
  }
}

__global__ void results_tree_kernel(PwPlanDev pw, double *vals, long long n, double V,
                                    Scalars *sc, double *hist_est, double *hist_var,
                                    Sched *sched, const int *status, int record, int flags) {
  extern __shared__ __align__(16) unsigned char tree_sm[];
  if (*status & 1) return;
  results_tree_body(tree_sm, pw, vals, n, V, sc, hist_est, hist_var, sched, record, flags);
}

__global__ void array_tree_kernel(PwPlanDev pw, double *vals, double *out) {
  pw_tree_combine(pw, vals);
  if (threadIdx.x == 0) *out = vals[3 * (pw.I > 0 ? pw.L + pw.I - 1 : 0)];
}

// -------------------------------------------------------------- allocation --
// n_h = max(ceil(n_eval * (dp/total)), 2), or the uniform share when beta == 0
// or total <= 0 (vp/strat.py:101-113).  Also the per-block sums for the plan.
constexpr int PLAN_NT = 1024;

// One PLAN_NT-cube block vb of the allocation (a PLAN_NT-thread block).
__device__ void alloc_block(long long vb, const double *dp, long long n, double beta, double ne,
                            long long uniform_nh, const Scalars *sc, int use_uniform,
                            long long *n_h, long long *bsum) {
  __shared__ long long red[PLAN_NT / 32];
  const long long h = vb * PLAN_NT + threadIdx.x;
  long long v = 0;
  if (h < n) {
    const double tot = sc->total_dp;
    if (use_uniform || beta == 0.0 || !(tot > 0.0)) {
      v = uniform_nh;
    } else {
      v = (long long)ceil(__dmul_rn(ne, __ddiv_rn(dp[h], tot)));
      v = v < 2 ? 2 : v;
    }
    n_h[h] = v;
  }
  long long s = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) bsum[vb] = s;
  }
  __syncthreads();   // red[] is reused by the caller's next block
}

__global__ void alloc_kernel(const double *dp, long long n, double beta, double ne,
                             long long uniform_nh, const Scalars *sc, int use_uniform,
                             long long *n_h, long long *bsum, const int *status) {
  if (*status & 1) return;
  alloc_block(blockIdx.x, dp, n, beta, ne, uniform_nh, sc, use_uniform, n_h, bsum);
}

// Block sums of a host-provided n_h (vpb_set_allocation).
__global__ void nh_blocksum_kernel(const long long *n_h, long long n, long long *bsum) {
  __shared__ long long red[PLAN_NT / 32];
  const long long h = (long long)blockIdx.x * PLAN_NT + threadIdx.x;
  long long s = h < n ? n_h[h] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) bsum[blockIdx.x] = s;
  }
}

// Inclusive int64 scan of one value per thread over a PLAN_NT-thread block:
// shuffles within warps, one shared step across the 32 warp totals (exact
// integer sums, so the order is free).  `wsum`: PLAN_NT/32 shared slots; the
// block must call it uniformly.
__device__ __forceinline__ long long block_incl_scan(long long v, long long *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < PLAN_NT / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < PLAN_NT / 32) wsum[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += wsum[warp - 1];
  return v;
}

// Smallest cube start offsets[h] >= t (t in (0, total)): the rank shards are
// snapped to hypercube boundaries, so every cube has exactly one owner.
// Block-wide: bpre = exclusive block prefixes (PLAN_NT cubes per block),
// n_h the allocation.  Cube starts are strictly increasing (n_h >= 1).
__device__ long long snap_to_cube(long long t, const long long *bpre, long long nb,
                                  const long long *n_h, long long n, long long total,
                                  long long *wsum, long long *s_out) {
  if (t <= 0) return 0;
  if (t >= total) return total;
  if (threadIdx.x == 0) {   // last block whose first cube starts at or before t
    long long lo = 0, hi = nb - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (bpre[mid] <= t) lo = mid; else hi = mid - 1;
    }
    s_out[0] = lo;
    s_out[1] = lo + 1 < nb ? bpre[lo + 1] : total;   // the next block's start
  }
  __syncthreads();
  const long long b = s_out[0];
  const long long h = b * PLAN_NT + threadIdx.x;
  const long long v = h < n ? n_h[h] : 0;
  const long long start = bpre[b] + block_incl_scan(v, wsum) - v;
  const long long prev_start = (h < n && threadIdx.x > 0) ? start - n_h[h - 1] : start;
  __syncthreads();
  // the first cube of the block starting at or after t
  if (h < n && start >= t && (threadIdx.x == 0 || prev_start < t)) s_out[1] = start;
  __syncthreads();
  const long long r = s_out[1];
  __syncthreads();
  return r;
}

// Exclusive scan of the block sums; total; this rank's shard of the run
// range and run_base bookkeeping (vp/core.py:208) and the evals history.
// Shards: the reference's partition rule (vp/executor.py:41-57: the first
// total % world ranks get +1) gives the split points, each snapped forward to
// the next hypercube start ("sharded by hypercube range"): every cube's runs
// -- its s1, s2 -- belong to one rank, and the shards stay balanced to
// within one cube.
__global__ void plan_scan_kernel(long long *bsum, long long nb, Sched *sched, int world, int rank,
                                 long long *hist_evals, int record, long long ntiles_cap,
                                 int *status, const long long *explicit_run_base,
                                 const long long *n_h, long long n_cubes) {
  __shared__ long long wsum[PLAN_NT / 32];
  __shared__ long long s_snap[2];
  if (*status) return;   // a failed iteration freezes the plan (error reporting)
  long long carry = 0;
  for (long long b0 = 0; b0 < nb; b0 += PLAN_NT) {
    const long long i = b0 + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    const long long inc = block_incl_scan(v, wsum);
    if (i < nb) bsum[i] = carry + inc - v;   // exclusive
    carry += wsum[PLAN_NT / 32 - 1];         // this chunk's total (uniform)
    __syncthreads();                         // wsum reused by the next chunk
  }
  const long long total = carry;
  const long long q = total / world, rem = total % world;
  const long long t0 = rank * q + (rank < rem ? rank : rem);
  const long long t1 = t0 + q + (rank < rem ? 1 : 0);
  long long lo = t0, hi = t1;
  if (world > 1) {
    lo = snap_to_cube(t0, bsum, nb, n_h, n_cubes, total, wsum, s_snap);
    hi = snap_to_cube(t1, bsum, nb, n_h, n_cubes, total, wsum, s_snap);
  }
  if (threadIdx.x == 0) {
    Sched s = *sched;
    if (explicit_run_base) {
      s.run_base = *explicit_run_base;
    } else {
      s.run_base = s.run_base_next;
      s.run_base_next = s.run_base + total;
    }
    s.total = total;
    s.lo = lo;
    s.hi = hi;
    const long long tr = 32ll * sched_rpt(s);
    s.ntiles = (s.hi - s.lo + tr - 1) / tr;
    if (s.ntiles > ntiles_cap) { atomicOr(status, 2); s.ntiles = 0; }
    *sched = s;
    if (record) hist_evals[s.it] = total;
  }
}

// offsets[h] = exclusive prefix of n_h; tile -> first cube table for the fill.
__global__ void plan_offsets_kernel(const long long *n_h, long long n, const long long *bpre,
                                    long long *offsets, const Sched *sched, int *tile_cube,
                                    const int *status) {
  __shared__ long long wsum[PLAN_NT / 32];
  if (status && *status) return;
  const long long h = (long long)blockIdx.x * PLAN_NT + threadIdx.x;
  const long long v = h < n ? n_h[h] : 0;
  const long long inc = block_incl_scan(v, wsum);
  const bool valid = h < n;
  long long t0 = 0, t1 = 0;
  if (valid) {
    const long long beg = bpre[blockIdx.x] + inc - v;
    const long long end = beg + v;
    offsets[h] = beg;
    if (h == n - 1) offsets[n] = end;
    const long long lo = sched->lo, hi = sched->hi;
    const long long a = beg > lo ? beg : lo, b = end < hi ? end : hi;
    if (a < b) {
      // tiles whose first run lies in [a, b)
      const long long tr = 32ll * sched_rpt(*sched);
      t0 = (a - lo + tr - 1) / tr;
      t1 = (b - lo + tr - 1) / tr;
      if (b == hi) tile_cube[sched->ntiles] = (int)h;   // sentinel: cube of the last run
    }
  }
  // short ranges by their own thread; the big cubes of an adapted plan
  // (thousands of tiles) by the whole warp, coalesced
  constexpr long long SHORT = 32;
  const bool longr = t1 - t0 > SHORT;
  if (!longr)
    for (long long t = t0; t < t1; t++) tile_cube[t] = (int)h;
  unsigned todo = __ballot_sync(0xffffffffu, longr);
  const int lane = threadIdx.x & 31;
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const long long u0 = __shfl_sync(0xffffffffu, t0, src), u1 = __shfl_sync(0xffffffffu, t1, src);
    const int hh = (int)__shfl_sync(0xffffffffu, h, src);
    for (long long t = u0 + lane; t < u1; t += 32) tile_cube[t] = hh;
  }
}

__global__ void set_iteration_kernel(Sched *sched, int it) { sched->it = it; }

// ----------------------------------------------------------------- fill ----
// Cube chains spanning tiles, in tile order (deterministic).
// A chain = a root tile whose tail cube starts inside it, the following
// "through" tiles lying entirely inside that cube, and the tile whose head
// closes it.  Chains with up to 8 through tiles are closed by the root's own
// thread (tile order); longer ones continue (cubes of many thousand runs: the peaks of an adapted
// allocation) by the whole warp, 256 tiles per step (8 per lane, loads in
// flight together): a ballot finds where the chain ends and the through
// values are summed per lane in tile order, then by a fixed xor butterfly,
// so the result is deterministic (the order differs from a left fold,
// within the cube-sum tolerance).
// One warp's 32 consecutive tiles t (lane = t & 31); all 32 lanes call it.
__device__ void fixup_tiles(const FillArgs &a, long long t) {
  const long long nt = a.sched->ntiles;
  const int lane = threadIdx.x & 31;
  const bool in = t < nt;
  if (in && t == 0 && a.ck_head[0] >= 0) {   // cube begun before this shard
    a.s1[a.ck_head[0]] = a.cv_head[0];
    a.s2[a.ck_head[0]] = a.cv_head[1];
  }
  const long long key = in ? a.ck_tail[t] : -1;
  const bool root = key >= 0 && (!a.ct_through[t] || t == 0);
  double v1 = 0.0, v2 = 0.0;
  bool longc = false;
  long long next = t + 1;   // first tile not yet summed
  if (root) {
    constexpr int SHORT = 8;   // through tiles a lane walks on its own
    v1 = a.cv_tail[2 * t];
    v2 = a.cv_tail[2 * t + 1];
    bool done = false;
    for (int k = 0; k <= SHORT && !done; k++, next++) {
      if (next < nt && a.ck_tail[next] == key && a.ct_through[next]) {
        if (k == SHORT) { longc = true; break; }
        v1 = __dadd_rn(v1, a.cv_tail[2 * next]);
        v2 = __dadd_rn(v2, a.cv_tail[2 * next + 1]);
        continue;
      }
      if (next < nt && a.ck_head[next] == key) {
        v1 = __dadd_rn(v1, a.cv_head[2 * next]);
        v2 = __dadd_rn(v2, a.cv_head[2 * next + 1]);
      }
      done = true;
    }
    if (done) {
      a.s1[key] = v1;
      a.s2[key] = v2;
    }
  }
  unsigned todo = __ballot_sync(0xffffffffu, longc);
  while (todo) {
    const int leader = __ffs(todo) - 1;
    todo &= todo - 1;
    const long long K = __shfl_sync(0xffffffffu, key, leader);
    const long long T = __shfl_sync(0xffffffffu, next, leader);
    double acc1 = __shfl_sync(0xffffffffu, v1, leader);
    double acc2 = __shfl_sync(0xffffffffu, v2, leader);
    constexpr int PER = 8;   // tiles per lane per step: 256 tiles per warp step
    for (long long base = T;; base += 32 * PER) {
      const long long u0 = base + (long long)lane * PER;
      bool cont[PER];
      double q1[PER], q2[PER];
#pragma unroll
      for (int k = 0; k < PER; k++) {   // independent loads, issued together
        const long long u = u0 + k;
        cont[k] = u < nt && a.ck_tail[u] == K && a.ct_through[u];
        q1[k] = cont[k] ? a.cv_tail[2 * u] : 0.0;
        q2[k] = cont[k] ? a.cv_tail[2 * u + 1] : 0.0;
      }
      int brk = PER;   // this lane's first non-through tile
#pragma unroll
      for (int k = PER - 1; k >= 0; k--) if (!cont[k]) brk = k;
      double p1 = 0.0, p2 = 0.0;
#pragma unroll
      for (int k = 0; k < PER; k++)
        if (k < brk) { p1 = __dadd_rn(p1, q1[k]); p2 = __dadd_rn(p2, q2[k]); }
      const unsigned bm = __ballot_sync(0xffffffffu, brk < PER);
      const int first = bm ? __ffs(bm) - 1 : 32;   // lane holding the chain's end
      if (lane > first) { p1 = 0.0; p2 = 0.0; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p1 = __dadd_rn(p1, __shfl_xor_sync(0xffffffffu, p1, o));
        p2 = __dadd_rn(p2, __shfl_xor_sync(0xffffffffu, p2, o));
      }
      acc1 = __dadd_rn(acc1, p1);
      acc2 = __dadd_rn(acc2, p2);
      if (first < 32) {
        const long long c = base + (long long)first * PER + __shfl_sync(0xffffffffu, brk, first);
        if (c < nt && a.ck_head[c] == K) {   // the closing tile
          acc1 = __dadd_rn(acc1, a.cv_head[2 * c]);
          acc2 = __dadd_rn(acc2, a.cv_head[2 * c + 1]);
        }
        break;
      }
    }
    if (lane == leader) {
      a.s1[K] = acc1;
      a.s2[K] = acc2;
    }
  }
}

__global__ void fill_fixup_kernel(FillArgs a) {
  if (*a.status) return;   // failed (now or earlier): the iteration is discarded
  fixup_tiles(a, (long long)blockIdx.x * blockDim.x + threadIdx.x);
}

// Sum the per-CTA histogram slices in CTA order (deterministic): block
// (32 elements x 8 partitions); partition p sums its contiguous range of CTA
// slices in order, then thread p = 0 adds the 8 partials in order.
// One 32-interval group (vb) by 256 threads (tx = interval, ty = slice
// partition); sw/sc: [8][33] shared partials of the calling block.
__device__ void hist_reduce_group(long long vb, int tx, int ty, double (*sw)[33],
                                  long long (*sc)[33], const double *hw_part,
                                  const unsigned *hc_part, int nparts, long long m,
                                  double *map_w, long long *map_counts) {
  const long long i = vb * 32 + tx;
  const int p = ty;
  const int per = (nparts + 7) / 8;
  const int b0 = p * per, b1 = min(nparts, b0 + per);
  double w = 0.0;
  long long c = 0;
  if (i < m) {
    // loads issued ahead in groups of 8; the adds stay in slice order
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      double wv[8];
      unsigned cv[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        wv[k] = hw_part[(size_t)(b + k) * m + i];
        cv[k] = hc_part[(size_t)(b + k) * m + i];
      }
#pragma unroll
      for (int k = 0; k < 8; k++) { w = __dadd_rn(w, wv[k]); c += cv[k]; }
    }
    for (; b < b1; b++) {
      w = __dadd_rn(w, hw_part[(size_t)b * m + i]);
      c += hc_part[(size_t)b * m + i];
    }
  }
  sw[p][tx] = w;
  sc[p][tx] = c;
  __syncthreads();
  if (p == 0 && i < m) {
    double t = sw[0][tx];
    long long k = sc[0][tx];
    for (int q = 1; q < 8; q++) { t = __dadd_rn(t, sw[q][tx]); k += sc[q][tx]; }
    map_w[i] = t;
    map_counts[i] = k;
  }
}

__global__ void hist_reduce_kernel(const double *hw_part, const unsigned *hc_part, int nparts,
                                   long long m, double *map_w, long long *map_counts,
                                   const int *status, const int *gate = nullptr) {
  __shared__ double sw[8][33];
  __shared__ long long sc[8][33];
  if (*status) return;   // failed (now or earlier): the iteration is discarded
  if (gate != nullptr && *gate == 0) return;   // the fixed-point sums stand (fx_reduce_kernel)
  hist_reduce_group(blockIdx.x, threadIdx.x, threadIdx.y, sw, sc, hw_part, hc_part, nparts, m,
                    map_w, map_counts);
}

// ---- deterministic mode (vpb_desc flags: VPB_FLAG_DETERMINISTIC) --------
// Pass 1 finds, per (axis, interval), the largest w2 (u64 max of the bit
// patterns, exact) and the count n; k = 61 - ilogb(max) - ceil(log2 n) keeps
// the pass-2 fixed-point sum below 2^62.  Pass 2 adds round(w2 * 2^k) with
// 64-bit integer atomics -- exact, hence independent of the update order and
// of the sharding (the int64 sums are all-reduced exactly) -- and map_w =
// sum * 2^-k rounds once.  Every input of k is exact, so the scales, and with
// them the sums, repeat bitwise.  Rounding: <= n/2 units of 2^-62 n max, i.e.
// ~1e-16 relative for any interval whose values are within 1e3 of each other
// (the reference's own sequential f64 sums carry the same order of error).
__global__ void hist_reduce_max_kernel(const unsigned long long *hw_part, const unsigned *hc_part,
                                       int nparts, long long m, double *map_w,
                                       long long *map_counts, const int *status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || *status) return;
  unsigned long long mx = 0;
  long long c = 0;
  for (int b = 0; b < nparts; b++) {
    mx = max(mx, hw_part[(size_t)b * m + i]);
    c += hc_part[(size_t)b * m + i];
  }
  map_w[i] = __longlong_as_double((long long)mx);
  map_counts[i] = c;
}
__global__ void det_scale_kernel(const double *map_max, const long long *map_counts, long long m,
                                 int *bin_k, const int *status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || *status) return;
  const double v = map_max[i];
  const long long n = map_counts[i];
  int lg = 0;
  while ((1ll << lg) < n) lg++;   // ceil(log2 n)
  bin_k[i] = (v > 0.0 && isfinite(v)) ? 61 - ilogb(v) - lg : 0;
}
// fixed-point slices (u64 bit patterns in the f64 slice buffers) -> map_q
__global__ void hist_reduce_q_kernel(const unsigned long long *hw_part, int nparts, long long m,
                                     long long *map_q, const int *status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || *status) return;
  unsigned long long t = 0;
  for (int b = 0; b < nparts; b++) t += hw_part[(size_t)b * m + i];
  map_q[i] = (long long)t;
}
__global__ void det_convert_kernel(const long long *map_q, const int *bin_k, long long m,
                                   double *map_w, const int *status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || *status) return;
  map_w[i] = scalbn(__ull2double_rn((unsigned long long)map_q[i]), -bin_k[i]);
}

// ------------------------------------------------ fixed-point histograms --
// State of the FX mode (fill.cuh LAYOUT_FX) of one context, device-resident so
// the captured iteration graph decides by itself which fill runs.
struct FxState {
  int gate_fx;    // this iteration's fixed-point fill runs
  int gate_f64;   // this iteration's f64 fill runs (no prediction, or a redo)
  int refill;     // set by fx_reduce_kernel: the fixed-point sums failed a proof
  int fails;      // redone iterations since reset (FX stops after FX_MAX_FAILS)
  int pred;       // refine_kernel CTAs that wrote a prediction (must be d)
  int enabled;    // host switch
  long long n_fx, n_redo;   // statistics: fixed-point iterations, redone ones
  unsigned long long spills;   // values summed in f64 instead (global, rare)
};
constexpr int FX_MAX_FAILS = 3;

// Start of an iteration's fill phase: the fixed-point fill runs when every
// axis has a prediction from the previous iteration's refinement (not the
// first refinement from the uniform map: its jump is too large to predict)
// and FX has not failed too often; otherwise only the f64 fill.
__global__ void fx_begin_kernel(FxState *fx, const Sched *sched, int dims, const int *status) {
  const bool use = fx->enabled && fx->pred == dims && sched->it >= 2 &&
                   fx->fails < FX_MAX_FAILS && *status == 0;
  fx->gate_fx = use ? 1 : 0;
  fx->gate_f64 = use ? 0 : 1;
  fx->refill = 0;
  fx->pred = 0;
  if (use) fx->n_fx++;
}

// Sum of the CTAs' fixed-point slices per interval (exact, 128-bit), the
// spilled f64 sums added, -> map_w / map_counts; and the proof that decides
// whether the iteration stands:
//   * no wrap-around: every value summed is < 2^L units, so a CTA slice with
//     count c holds < c 2^L; every slice must have c <= 2^(64-L);
//   * precision: each value rounds by <= 1/2 unit, so an interval with n
//     values and total S units (fixed point + spill) is within n/2 units,
//     i.e. 2^-(P+1) relative when S >= 2^P n (e = 255 intervals have no
//     fixed-point rounding worth the name: scale 2^1023).
// A failed proof anywhere sets fx->refill and opens the f64 fill (gated
// second launch in the graph), which recomputes the whole iteration's
// histograms; its hist_reduce_kernel then overwrites map_w / map_counts.
__global__ void fx_reduce_kernel(const unsigned long long *hw_part, const unsigned *hc_part,
                                 int nparts, long long m, int ng, int dims, const int *fx_k,
                                 const int *fx_kmin,
                                 int L, double *map_w, long long *map_counts, double *spill,
                                 FxState *fx, const int *status) {
  __shared__ unsigned long long s_lo[8][33], s_hi[8][33];
  __shared__ long long s_c[8][33];
  __shared__ unsigned s_cm[8][33];
  __shared__ int s_bad[33];
  if (!fx->gate_fx || *status) return;
  const long long i = (long long)blockIdx.x * 32 + threadIdx.x;
  const int p = threadIdx.y;
  const int per = (nparts + 7) / 8;
  const int b0 = p * per, b1 = min(nparts, b0 + per);
  unsigned long long lo = 0, hi = 0;
  long long c = 0;
  unsigned cm = 0;
  int K = FX_K_NONE;
  for (int j = 0; j < dims; j++) K = min(K, fx_kmin[j]);
  const int e0 = 1023 + max(min(K, 1023 - 254), -1022);
  const unsigned ef = i < m ? (unsigned)fx_biased_exp(fx_k[i], e0) : 0u;
  bool exp_ok = true;
  if (i < m) {
    for (int b = b0; b < b1; b++) {
      const unsigned w = hc_part[(size_t)b * m + i];
      // the slice's (hi:lo) minus the 0x43300000 every value added to hi
      const unsigned long long v =
          hw_part[(size_t)b * m + i] -
          ((unsigned long long)((w & 0xFFFFFu) * 0x43300000u) << 32);
      lo += v;
      hi += lo < v ? 1ull : 0ull;
      c += w & 0xFFFFFu;
      cm = max(cm, w & 0xFFFFFu);
      exp_ok = exp_ok && (w >> 20) == ef;   // a count past 2^20 would show here
    }
  }
  s_lo[p][threadIdx.x] = lo;
  s_hi[p][threadIdx.x] = hi;
  s_c[p][threadIdx.x] = c;
  s_cm[p][threadIdx.x] = cm;
  if (p == 0) s_bad[threadIdx.x] = 0;
  __syncthreads();
  if (!exp_ok) s_bad[threadIdx.x] = 1;
  __syncthreads();
  if (p != 0 || i >= m) return;
  for (int q = 1; q < 8; q++) {
    const unsigned long long v = s_lo[q][threadIdx.x];
    lo += v;
    hi += (lo < v ? 1ull : 0ull) + s_hi[q][threadIdx.x];
    c += s_c[q][threadIdx.x];
    cm = max(cm, s_cm[q][threadIdx.x]);
  }
  const int k = (int)ef - 1023;     // the interval's scale 2^k
  const double units = fma(__ull2double_rn(hi), 0x1p64, __ull2double_rn(lo));
  const double sp = spill[i];
  spill[i] = 0.0;
  map_w[i] = __dadd_rn(scalbn(units, -k), sp);
  map_counts[i] = c;
  const bool wrap_free = (double)cm <= ldexp(1.0, 64 - L) && !s_bad[threadIdx.x];
  const bool precise = c == 0 || ef == 2046u ||
                       __dadd_rn(units, scalbn(sp, k)) >= ldexp((double)c, VPB_FX_P);
  if (!(wrap_free && precise)) {
    if (atomicExch(&fx->refill, 1) == 0) {
      fx->gate_f64 = 1;
      fx->fails++;
      fx->n_redo++;
    }
  }
}

// The exchange's control word, all-reduced with MAX next to the accumulators
// so that every rank sees every rank's failure (vp/executor.py:151-165: the
// reference re-raises the lowest failing worker's exception for the whole
// integration): [non-finite flag, assert flag, -(first failing run)].  The
// run index is plan-global, so MAX of its negation is the lowest failing run
// over all ranks; "none" (~0) maps to -INT64_MAX.
__global__ void ctl_pack_kernel(const int *status, const unsigned long long *err_run,
                                long long *ctl) {
  const int st = *status;
  const unsigned long long e = *err_run;
  ctl[0] = st & 1;
  ctl[1] = (st >> 1) & 1;
  ctl[2] = e == ~0ull ? -0x7FFFFFFFFFFFFFFFll : -(long long)e;
}
__global__ void ctl_unpack_kernel(int *status, unsigned long long *err_run, const long long *ctl) {
  *status |= (int)(ctl[0] | (ctl[1] << 1));
  *err_run = ctl[2] == -0x7FFFFFFFFFFFFFFFll ? ~0ull : (unsigned long long)(-ctl[2]);
}

__global__ void hist_glob_convert_kernel(const unsigned long long *hc, long long m,
                                         long long *map_counts) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) map_counts[i] = (long long)hc[i];
}

// --------------------------------------------------------------- refine ----
// numpy pairwise sum of a shared-memory row of length n <= 4096 by a whole
// block: thread 0 flattens numpy's split tree into a postfix program (leaf
// ids and adds), 8 lanes per leaf compute the 8-accumulator leaves, thread 0
// evaluates the program.  Bit-identical to pw_sum_rt / np.sum.
struct BlockPw {
  int n_leaf, n_tok;
  int leaf_off[32], leaf_len[32];
  int tok[64];          // >= 0: leaf id, -1: add the two top values
  double leaf_val[32];
  double out;
};

__device__ double block_pairwise(const double *a, int n, BlockPw &S) {
  if (threadIdx.x == 0) {
    // explicit-stack post-order walk of numpy's recursion
    int st_off[16], st_n[16], st_state[16], sp = 0, nl = 0, nt = 0;
    st_off[0] = 0; st_n[0] = n; st_state[0] = 0;
    while (sp >= 0) {
      const int o = st_off[sp], m = st_n[sp];
      if (m <= 128) {
        S.leaf_off[nl] = o; S.leaf_len[nl] = m; S.tok[nt++] = nl++;
        sp--;
        continue;
      }
      int n2 = m / 2; n2 -= n2 % 8;
      if (st_state[sp] == 0) {
        st_state[sp] = 1; sp++; st_off[sp] = o; st_n[sp] = n2; st_state[sp] = 0;
      } else if (st_state[sp] == 1) {
        st_state[sp] = 2; sp++; st_off[sp] = o + n2; st_n[sp] = m - n2; st_state[sp] = 0;
      } else {
        S.tok[nt++] = -1;
        sp--;
      }
    }
    S.n_leaf = nl; S.n_tok = nt;
  }
  __syncthreads();
  for (int base = 0; base < 8 * S.n_leaf; base += blockDim.x) {
    const int t = base + threadIdx.x, leaf = t >> 3, j = t & 7;
    const bool live = leaf < S.n_leaf;
    const int o = live ? S.leaf_off[leaf] : 0, len = live ? S.leaf_len[leaf] : 0;
    const int full = len < 8 ? 0 : len - (len % 8);
    double r = 0.0;
    if (live && len >= 8) {
      r = a[o + j];
      for (int i = 8 + j; i < full; i += 8) r = __dadd_rn(r, a[o + i]);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, true);
#pragma unroll
    for (int x = 1; x < 8; x <<= 1) r = __dadd_rn(r, __shfl_xor_sync(mask, r, x));
    if (live && j == 0) {
      if (len < 8) r = 0.0;
      for (int i = full; i < len; i++) r = __dadd_rn(r, a[o + i]);
      S.leaf_val[leaf] = r;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double stk[32];
    int sp = 0;
    for (int k = 0; k < S.n_tok; k++) {
      if (S.tok[k] >= 0) stk[sp++] = S.leaf_val[S.tok[k]];
      else { stk[sp - 2] = __dadd_rn(stk[sp - 2], stk[sp - 1]); sp--; }
    }
    S.out = stk[0];
  }
  __syncthreads();
  return S.out;
}

// One CTA per dimension: smooth_and_damp (vp/maps.py:160-199) then
// update_grid (vp/maps.py:202-234) on a shared-memory copy of the row.
// numpy's pairwise sums run block-wide (block_pairwise); the cumsum is
// inherently sequential (numpy's rounding) and runs on one thread.
constexpr int REFINE_NT = 1024;
constexpr int REFINE_SMEM_NG = 2048;   // rows up to this length live in smem

// Sum over a block (any order: heuristics only).
__device__ double block_sum_f64(double v) {
  __shared__ double part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
  return t;
}

__device__ void refine_body(int j, double *rsm, double *edges, const double *map_w,
                            const long long *map_counts, int ng, double alpha, double *scratch,
                            int *status, double *damped_out, int *fx_k, int *fx_kmin,
                            FxState *fx, double *fx_tot) {
  __shared__ BlockPw S;
  __shared__ int s_skip;
  double *d, *sm, *dw, *cum, *ne, *e;
  if (ng <= REFINE_SMEM_NG) {
    d = rsm; sm = d + ng; dw = sm + ng; cum = dw + ng; ne = cum + ng + 1; e = ne + ng + 1;
  } else {
    d = scratch + (size_t)j * (6 * ng + 3);
    sm = d + ng; dw = sm + ng; cum = dw + ng; ne = cum + ng + 1; e = ne + ng + 1;
  }
  const double *w = map_w + (size_t)j * ng;
  const long long *c = map_counts + (size_t)j * ng;
  double *eg = edges + (size_t)j * (ng + 1);
  if (*status) return;
  int nz = 0;
  for (int i = threadIdx.x; i < ng; i += blockDim.x) {
    const double v = c[i] > 0 ? __ddiv_rn(w[i], (double)c[i]) : 0.0;
    d[i] = v;
    nz |= (v != 0.0);
  }
  for (int i = threadIdx.x; i <= ng; i += blockDim.x) e[i] = eg[i];
  nz = __syncthreads_or(nz);
  auto zero_out = [&]() {
    if (damped_out)
      for (int i = threadIdx.x; i < ng; i += blockDim.x) damped_out[(size_t)j * ng + i] = 0.0;
  };
  if (!nz) { zero_out(); return; }
  for (int i = threadIdx.x; i < ng; i += blockDim.x) {
    double v;
    if (i == 0) v = __dadd_rn(__dmul_rn(7.0, d[0]), d[1]);
    else if (i == ng - 1) v = __dadd_rn(d[ng - 2], __dmul_rn(7.0, d[ng - 1]));
    else v = __dadd_rn(__dadd_rn(d[i - 1], __dmul_rn(6.0, d[i])), d[i + 1]);
    sm[i] = __dmul_rn(v, 0.125);   // /8.0 (exact power of two)
  }
  __syncthreads();
  const double tot = ng <= 4096 ? block_pairwise(sm, ng, S) : pw_sum_rt(sm, ng);
  if (!(tot > 0.0)) { zero_out(); return; }
  for (int i = threadIdx.x; i < ng; i += blockDim.x) {
    const double v = __ddiv_rn(sm[i], tot);
    double r;
    if (fabs(__dadd_rn(v, -1.0)) < 1e-15) r = 1.0;
    else if (v >= 1e-30) r = np_scalar_pow(__ddiv_rn(__dadd_rn(v, -1.0), log(v)), alpha);
    else r = 0.0;
    dw[i] = r;
    if (damped_out) damped_out[(size_t)j * ng + i] = r;
  }
  __syncthreads();
  const double tot2 = ng <= 4096 ? block_pairwise(dw, ng, S) : pw_sum_rt(dw, ng);
  if (threadIdx.x == 0) {
    s_skip = !(tot2 > 0.0);
    if (!s_skip) {   // sequential cumsum (np.cumsum)
      double acc = 0.0;
      cum[0] = 0.0;
      int i = 0;
      for (; i + 8 <= ng; i += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = dw[i + k];
#pragma unroll
        for (int k = 0; k < 8; k++) { acc = __dadd_rn(acc, v[k]); cum[i + k + 1] = acc; }
      }
      for (; i < ng; i++) { acc = __dadd_rn(acc, dw[i]); cum[i + 1] = acc; }
    }
  }
  __syncthreads();
  if (s_skip) return;
  const double delta = __ddiv_rn(tot2, (double)ng);
  for (int i = 1 + threadIdx.x; i < ng; i += blockDim.x) {
    const double goal = __dmul_rn((double)i, delta);
    // searchsorted(cum[1:], goal, 'left'): first iv with cum[iv+1] >= goal
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cum[mid + 1] >= goal) hi = mid; else lo = mid + 1;
    }
    const int iv = lo;
    const double frac = __ddiv_rn(__dadd_rn(goal, -cum[iv]), dw[iv]);
    ne[i] = __dadd_rn(e[iv], __dmul_rn(frac, __dadd_rn(e[iv + 1], -e[iv])));
  }
  __syncthreads();
  int bad = 0;
  for (int i = threadIdx.x; i < ng; i += blockDim.x) {
    const double a = i == 0 ? e[0] : ne[i];
    const double b = i == ng - 1 ? e[ng] : ne[i + 1];
    bad |= !(b > a);
  }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (threadIdx.x == 0) atomicOr(status, 2);
    return;
  }
  if (fx_k != nullptr) {
    // FX: the next iteration's fixed-point scale per new interval, from the
    // average w2 of the old interval holding its midpoint, times the change
    // of this axis's Jacobian factor (w2 carries (ng dx)^2):
    //   avg' ~ avg_old (dx_new / dx_old)^2,   k = T - ilogb(avg')
    // so that the interval's values sit near 2^T units (the counts per
    // interval stay ~n/ng: samples are uniform in y).  Trend: the other axes'
    // maps move too, which scales every interval of this axis alike; the row
    // total (sum of w2 over all samples) fell by r over the last iteration,
    // so expect it to fall by about r again (r clamped to [2^-16, 1]: rises
    // only cost spills, falls cost precision).
    double rs = 0.0;
    for (int i = threadIdx.x; i < ng; i += blockDim.x) rs += w[i];
    rs = block_sum_f64(rs);
    const double prev_tot = fx_tot[j];
    double trend = 1.0;
    if (prev_tot > 0.0 && rs > 0.0) trend = fmin(fmax(rs / prev_tot, 0x1p-16), 1.0);
    // a row total that jumped up (the first refinement from the uniform map:
    // x8900 on the three-peak Gaussian) says nothing about the next step --
    // no prediction, the next iteration stays f64 (instead of a redo)
    const bool jumped = prev_tot > 0.0 && rs > 4.0 * prev_tot;
    __syncthreads();
    if (threadIdx.x == 0) fx_tot[j] = rs;
    int kmin = FX_K_NONE;
    for (int i = threadIdx.x; i < ng; i += blockDim.x) {
      const double a0 = i == 0 ? e[0] : ne[i], a1 = i == ng - 1 ? e[ng] : ne[i + 1];
      const double mid = __dadd_rn(a0, __dmul_rn(0.5, __dadd_rn(a1, -a0)));
      int lo = 0, hi = ng - 1;   // last old interval with e[ob] <= mid
      while (lo < hi) {
        const int md = (lo + hi + 1) >> 1;
        if (e[md] <= mid) lo = md; else hi = md - 1;
      }
      const double r = __dadd_rn(a1, -a0) / __dadd_rn(e[lo + 1], -e[lo]);
      const double pa = d[lo] * r * r * trend;
      const int k = (pa > 0.0 && isfinite(pa)) ? VPB_FX_T - ilogb(pa) : FX_K_NONE;
      fx_k[(size_t)j * ng + i] = k;
      kmin = min(kmin, k);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    __shared__ int s_kmin;
    if (threadIdx.x == 0) s_kmin = FX_K_NONE;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMin(&s_kmin, kmin);
    __syncthreads();
    if (threadIdx.x == 0) {
      fx_kmin[j] = s_kmin;
      if (!jumped) atomicAdd(&fx->pred, 1);
    }
  }
  for (int i = 1 + threadIdx.x; i < ng; i += blockDim.x) eg[i] = ne[i];
}

__global__ void __launch_bounds__(REFINE_NT) refine_kernel(double *edges, const double *map_w,
                                                          const long long *map_counts, int ng,
                                                          double alpha, double *scratch,
                                                          int *status, double *damped_out,
                                                          int *fx_k = nullptr,
                                                          int *fx_kmin = nullptr,
                                                          FxState *fx = nullptr,
                                                          double *fx_tot = nullptr) {
  extern __shared__ __align__(16) double rsm[];
  refine_body(blockIdx.x, rsm, edges, map_w, map_counts, ng, alpha, scratch, status, damped_out,
              fx_k, fx_kmin, fx, fx_tot);
}

inline size_t refine_smem_bytes(int ng) {
  return ng <= REFINE_SMEM_NG ? sizeof(double) * (6 * (size_t)ng + 3) : 0;
}

// ------------------------------------------------- cooperative update ----
// The whole post-fill part of an iteration in ONE launch (single GPU, no
// exchange): cube-chain fixup + histogram reduction | barrier | refinement
// on CTAs [0, d) concurrently with the fused per-cube terms + pairwise
// leaves on the others | barrier | pairwise tree (CTA d) | barrier |
// allocation + plan block sums | the last CTA out ends the iteration.
// Replaces nine launches (fixup, hist_reduce, cube_terms, results_leaf,
// results_tree, alloc, refine, end_iteration + the side-stream fork/join)
// whose launch gaps and single-CTA latencies are most of the non-fill time
// of small iterations (cfg1).  Opt-in (VPB_COOP=1): on the B200 its phases
// (globaltimer, cfg1: fixup+reduce 3.7 us, barrier 3.5, terms + leaves 15,
// tree 9.6, allocation 3.7; refinement 22 us beside them) sum to about the
// chain's critical path, and the following fill measured 12 us slower, so
// the chain (with the refinement on a side stream) stays the default.  Launched cooperatively (all CTAs resident),
// so the spin barriers below cannot deadlock; the same device bodies as the
// separate kernels, so the results are bitwise those of the launch chain.
struct UpdArgs {
  FillArgs fa;                       // fixup (tiles, carries, s1/s2)
  const double *hw_part;             // histogram slices
  const unsigned *hc_part;
  int nparts;
  long long m;
  double *map_w;
  long long *map_counts;
  const int *hist_gate;              // FX: f64 slices only when gate_f64
  double *edges;                     // refinement
  int ng, dims;
  double alpha;
  double *refine_scr;
  int *fx_k, *fx_kmin;
  FxState *fxs;
  double *fx_tot;
  const double *s1, *s2;             // results
  const long long *offsets;
  long long n_cubes;
  double V, beta;
  double *d_h, *dp;
  PwPlanDev pw;
  double *pwvals, *pwterms;
  Scalars *sc;
  double *h_est, *h_var;
  Sched *sched;
  int record, tree_flags;
  double ne;                         // allocation
  long long uniform_nh;
  long long *n_h, *bsum;
  long long nb;
  int *status, *fail_it;
  unsigned *bar;                     // [5] barrier counters, zero between launches
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_arrive(unsigned *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c, 1u);
  }
}
__device__ __forceinline__ void grid_wait(unsigned *c, unsigned n) {
  if (threadIdx.x == 0) {
    while (ld_acquire_u32(c) < n) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

#ifndef VPB_COOP_PROF
#define VPB_COOP_PROF 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#if VPB_COOP_PROF
#define COOP_TS(k) do { if (threadIdx.x == 0) ts[k] = gtimer(); } while (0)
#else
#define COOP_TS(k) do {} while (0)
#endif
constexpr int UPD_NT = 1024;   // = PLAN_NT = REFINE_NT
__global__ void __launch_bounds__(UPD_NT, 1) update_coop_kernel(UpdArgs u) {
  extern __shared__ __align__(16) unsigned char usm[];
  __shared__ double sw[4][8][33];
  __shared__ long long scn[4][8][33];
  const unsigned G = gridDim.x;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int st0 = *u.status;   // refinement may add its assert bit below, nothing else
#if VPB_COOP_PROF
  unsigned long long ts[10] = {0};
#endif
  COOP_TS(0);
  // ---- phase 1: cube chains across tiles || interval histogram slices
  if (st0 == 0) {
    const long long nt = u.fa.sched->ntiles;
    for (long long base = (long long)b * UPD_NT; base < nt; base += (long long)G * UPD_NT)
      fixup_tiles(u.fa, base + tid);   // whole warps: base + tid covers 32 consecutive tiles
    if (u.hist_gate == nullptr || *u.hist_gate) {
      const long long groups = (u.m + 31) / 32;
      for (long long r = b; r * 4 < groups; r += G) {   // 4 groups of 32 intervals per round
        const int sub = tid >> 8;
        hist_reduce_group(r * 4 + sub, tid & 31, (tid >> 5) & 7, sw[sub], scn[sub], u.hw_part,
                          u.hc_part, u.nparts, u.m, u.map_w, u.map_counts);
      }
    }
  }
  COOP_TS(1);
  grid_arrive(u.bar + 0);
  grid_wait(u.bar + 0, G);
  COOP_TS(2);
  if (b < u.dims) {
    // ---- refinement CTAs: nothing below depends on them; arrive and refine
    grid_arrive(u.bar + 1);
    grid_arrive(u.bar + 2);
    if (st0 == 0)
      refine_body(b, reinterpret_cast<double *>(usm), u.edges, u.map_w, u.map_counts, u.ng,
                  u.alpha, u.refine_scr, u.status, nullptr, u.fx_k, u.fx_kmin, u.fxs, u.fx_tot);
    COOP_TS(3);
#if VPB_COOP_PROF
    if (b == 0 && threadIdx.x == 0)
      printf("coop refine: p1 %llu b1 %llu refine %llu (ns)\n", ts[1] - ts[0], ts[2] - ts[1],
             ts[3] - ts[2]);
#endif
  } else {
    const unsigned W = G - u.dims;
    const int wb = b - u.dims;
    // ---- per-cube terms (fully parallel: the divisions, sqrt and pow of a
    // cube do not serialise inside a leaf), then the pairwise leaves; the
    // barrier between them is among these CTAs only (the refinement CTAs
    // arrive once, up front)
    if (!(st0 & 1)) {
      const bool want_dp = u.beta != 0.0;
      for (long long h = (long long)wb * UPD_NT + tid; h < u.n_cubes; h += (long long)W * UPD_NT) {
        double m, t, q;
        cube_terms(u.s1, u.s2, u.offsets, h, u.V, u.beta, want_dp, u.d_h, u.dp, m, t, q);
        u.pwterms[h] = m;
        u.pwterms[u.n_cubes + h] = t;
        u.pwterms[2 * u.n_cubes + h] = q;
      }
    }
    grid_arrive(u.bar + 4);
    grid_wait(u.bar + 4, W);
    if (!(st0 & 1)) {
      const long long nv = 8LL * u.pw.L;
      for (long long base = (long long)wb * UPD_NT; base < nv; base += (long long)W * UPD_NT)
        results_leaf_body(base + tid, u.pwterms, u.n_cubes, u.pw, u.pwvals);
    }
    COOP_TS(3);
    grid_arrive(u.bar + 1);
    grid_wait(u.bar + 1, G);
    COOP_TS(4);
    // ---- pairwise tree: the estimate, variance and allocation total
    if (wb == 0 && !(st0 & 1))
      results_tree_body(usm, u.pw, u.pwvals, u.n_cubes, u.V, u.sc, u.h_est, u.h_var, u.sched,
                        u.record, u.tree_flags);
    COOP_TS(5);
    grid_arrive(u.bar + 2);
    grid_wait(u.bar + 2, G);
    COOP_TS(6);
    // ---- allocation for the next iteration + the plan's block sums
    if (!(st0 & 1))
      for (long long vb = wb; vb < u.nb; vb += W)
        alloc_block(vb, u.dp, u.n_cubes, u.beta, u.ne, u.uniform_nh, u.sc, 0, u.n_h, u.bsum);
    COOP_TS(7);
#if VPB_COOP_PROF
    if (wb == 0 && threadIdx.x == 0)
      printf("coop main: p1 %llu b1 %llu leaves %llu b2 %llu tree %llu b3 %llu alloc %llu (ns)\n",
             ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3], ts[5] - ts[4],
             ts[6] - ts[5], ts[7] - ts[6]);
#endif
  }
  // ---- the last CTA out ends the iteration (vpb end_iteration_kernel) and
  // re-arms the barriers for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(u.bar + 3, 1u) == G - 1) {
      __threadfence();
      const int st = *(volatile int *)u.status;
      if (st) {
        if (*u.fail_it < 0) *u.fail_it = u.sched->it;
      } else {
        u.sched->it = u.sched->it + 1;
      }
      u.bar[0] = 0u; u.bar[1] = 0u; u.bar[2] = 0u; u.bar[3] = 0u; u.bar[4] = 0u;
      __threadfence();
    }
  }
}

inline size_t update_coop_smem(int ng, const PwPlanDev &pw) {
  const size_t r = refine_smem_bytes(ng), t = pw_tree_smem(pw);
  return r > t ? r : t;
}

// ---------------------------------------------------------- parity kernels --
__global__ void philox_kernel(const uint64_t *block, const uint64_t *stream, const uint64_t *seed,
                              long long n, uint64_t *out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PhiloxKeys K(seed[i]);
  uint64_t w0, w1;
  philox((uint32_t)block[i], (uint32_t)(block[i] >> 32), (uint32_t)stream[i],
         (uint32_t)(stream[i] >> 32), K, w0, w1);
  out[2 * i] = w0;
  out[2 * i + 1] = w1;
}

__global__ void uniform_kernel(const uint64_t *seed, const uint64_t *stream, const uint64_t *pos,
                               long long n, double *out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PhiloxKeys K(seed[i]);
  uint64_t w0, w1;
  const uint64_t blk = pos[i] >> 1;
  philox((uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)stream[i], (uint32_t)(stream[i] >> 32),
         K, w0, w1);
  out[i] = unit_from_word((pos[i] & 1) ? w1 : w0);
}

// kernels.sample_runs for runs [run_start, run_start+n): one thread per run,
// cube by binary search (strat.run_to_cube, vp/strat.py:140-144).  The same
// per-dimension arithmetic as the fill kernel.
__global__ void sample_runs_kernel(unsigned long long seed, long long batch, long long run_base,
                                   long long run_start, long long n, const long long *offsets,
                                   long long n_cubes, const double *edges, int dims, int ng,
                                   long long n_strat, double *x, double *jac, long long *idx,
                                   long long *cube) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long r = run_start + i;
  long long lo = 0, hi = n_cubes - 1;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const long long c = lo;
  cube[i] = c;
  const PhiloxKeys K(seed);
  const unsigned long long g = (unsigned long long)(run_base + r);
  const unsigned long long sl = g % (unsigned long long)batch, k = g / (unsigned long long)batch;
  const unsigned long long base = k * (unsigned long long)((dims + (dims & 1)) >> 1);
  const double nsf = (double)n_strat, rns = 1.0 / nsf, ngf = (double)ng;
  double nsf2, rns2;
  sample_consts(nsf, rns, nsf2, rns2);
  long long rem = c;
  double jf = 1.0;
  uint64_t w0 = 0, w1 = 0;
  for (int j = 0; j < dims; j++) {
    if ((j & 1) == 0) {
      const unsigned long long blk = base + (unsigned long long)(j >> 1);
      philox((uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)sl, (uint32_t)(sl >> 32), K, w0, w1);
    }
    const long long q = rem / n_strat, dig = rem - q * n_strat;
    rem = q;
    int iv;
    x[i * dims + j] = sample_axis((j & 1) ? w1 : w0, div_exact((double)dig, nsf, rns), nsf2,
                                  rns2, ngf, ng, EdgeRow{edges + (size_t)j * (ng + 1)}, jf, iv);
    idx[i * dims + j] = iv;
  }
  jac[i] = jf;
}

}  // namespace vpb
