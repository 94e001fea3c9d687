// fill.cuh -- the fused VEGAS+ fill kernel (sm_100a).
//
// Replaces executor.parallel_fill -> fill_shard -> kernels.sample_runs +
// f_batch + kernels.accumulate (vp/executor.py:86-166, vp/kernels.py:36-109)
// for one rank's run range [lo, hi) of the current plan.
//
// Work decomposition: the plan's run range is cut into warp tiles of
// TILE = 32*RPT consecutive runs; each lane owns RPT consecutive runs, so a
// lane stays inside one hypercube for long stretches and keeps the cube's
// running sums s1 = sum(jf), s2 = sum(jf^2) in registers.  Cube sums are
// reduced deterministically and without atomics:
//   * a cube entirely inside one lane's runs is stored directly;
//   * a cube spanning lanes is closed by a warp segmented scan (shuffles);
//   * a cube spanning tiles leaves per-tile carries that fill_fixup_kernel
//     adds in tile order.
// The persistent grid's warps are spread over the run range: warp w of CTA b
// walks tiles w*P + b, w*P + b + grid, ... (P = ntiles / warps-per-CTA), so
// the warps sharing a CTA's shared histograms sit in distant hypercubes, i.e.
// in different strata of most axes, and rarely race for the same interval.
// No block barrier is needed inside the tile loop.
// Per-dimension interval histograms (MapWeights.w / .counts) live in shared
// memory (f64 via atom.shared CAS, u32 counts via native ATOMS); each CTA
// writes its private copy to a slice that hist_reduce_kernel sums in CTA
// order.  Cube evaluation counts are not accumulated at all: every run of the
// plan is evaluated exactly once, so counts[h] = n_h (within the shard).
//
// Bitwise contract with vp/kernels.py:36-88: the
// Philox counter layout, u = (w>>11)*2^-53, y = RN(RN(digit/N) + RN(u/N)),
// the y >= 1 clamp, t = RN(y*ng), iv = min(trunc t, ng-1), frac = t - iv,
// x = RN(lo + RN(frac*dx)), jac *= RN(ng*dx), all unfused.
#pragma once
#include <cstdint>

#include "cluster.cuh"
#include "devmath.cuh"
#include "integrands.cuh"

namespace vpb {

#ifndef VPB_FILL_NT
#define VPB_FILL_NT 640
#endif
#ifndef VPB_FILL_RPT
#define VPB_FILL_RPT 16   // the default / small-plan runs per lane; large plans take 32
                          // or 64 per context (Sched.rpt, capi.cu)
#endif
constexpr int FILL_NT = VPB_FILL_NT;
#ifndef VPB_ALL_NT768
#define VPB_ALL_NT768 0
#endif
#ifndef VPB_ROT_STAGES
#define VPB_ROT_STAGES 0   // barrel stages of the histogram lane rotation (0: by d, below)
#endif
#ifndef VPB_STREAM_NT
#define VPB_STREAM_NT 768   // threads of the streamed-sum and many-axis records kernels
#endif    // threads per CTA (one CTA per SM)
constexpr int FILL_RPT = VPB_FILL_RPT;  // consecutive runs per lane per tile
constexpr int FILL_TILE = 32 * FILL_RPT;   // runs per warp tile
constexpr int DQ_TABLE_MAX = 2048;             // digit/N table when N <= this
#ifndef VPB_DQ_REG_MAX
#define VPB_DQ_REG_MAX 12   // dims up to which RN(digit/N) stays in registers
#endif
#ifndef VPB_REC_K0
#define VPB_REC_K0 4
#endif
constexpr int REC_K0 = VPB_REC_K0;   // axes kept in shared memory by a records-layout fill (d >= 12)

// Per-iteration schedule written by the plan kernels (device memory).
struct Sched {
  long long run_base;     // evaluations consumed by earlier iterations
  long long lo, hi;       // this rank's run range of the plan
  long long ntiles;       // ceil((hi-lo)/TILE) warp tiles
  long long total;        // plan.total
  long long run_base_next;
  int it;                 // 0-based iteration index being processed
  int rpt;                // runs per lane per warp tile (0: FILL_RPT); set per context
};
// runs per lane of a schedule: 16, or 32 for large plans (capi.cu choose_rpt)
__host__ __device__ inline int sched_rpt(const Sched &s) { return s.rpt > 0 ? s.rpt : FILL_RPT; }

struct FillArgs {
  const long long *offsets;     // [n_cubes+1]
  long long n_cubes;
  const double *edges;          // [d][ng+1]
  int dims, ng;
  long long n_strat;
  double nsf, rns, ngf;         // N, RN(1/N), ng as doubles
  long long batch;
  unsigned long long seed;
  PhiloxKeys keys;              // round keys (host-computed; constant bank operands)
  MagicDiv nsdiv;               // division by n_strat (cube digits)
  long long dk, ds;             // per-grid-stride advance of (k, slot)
  const Sched *sched;
  const int *tile_cube;         // [ntiles+1]
  double *s1, *s2;              // [n_cubes], zeroed by the caller
  long long *ck_head, *ck_tail; // per tile carry keys (-1 = none)
  double *cv_head, *cv_tail;    // per tile carry values [2*tile + {0,1}]
  int *ct_through;              // per tile: tail chain has no root in the tile
  double *hw_part;              // [grid][d*ng]   (smem histograms)
  unsigned *hc_part;            // [grid][d*ng]
  double *hw_glob;              // [d*ng] (global-atomic histograms)
  unsigned long long *hc_glob;  // [d*ng]
  int smem_hist;                // 1: CTA-private shared histograms
  int hcopies;                  // copies of the shared f64 sums (lanes 0-15 / 16-31)
  int records;                  // 1: write (interval, w^2) records for hist_records_kernel
  int dig_bits;                 // bits per packed cube digit (d > 12 kernels)
  long long tile_lo, tile_hi;   // tiles of this launch (records mode: one chunk)
  unsigned short *rec_iv;       // [n_groups][rec_ch][8] intervals, axes 8g..8g+7
  double *rec_w2;               // [rec_ch]
  long long rec_ch;             // records per chunk (a multiple of FILL_TILE)
  int pairs;                    // 1: (E[i], dx[i]) pair table instead of the edge rows
  int hs;                       // row stride of the shared histograms [interval][axis]
  int det;                      // deterministic mode pass (generic kernel): 0/1 f64, 2 fixed point
  const int *bin_k;             // det pass 2: per (axis, interval) scale exponent [d][ng]
  int *status;                  // bit0 non-finite, bit1 assert
  unsigned long long *err_run;  // min run index with a non-finite value
  IParams P;
  // gate: the launch does nothing unless *gate != 0 (nullptr: always runs).
  // The fixed-point fill and the f64 fill of an iteration are both in the
  // captured graph; fx_begin_kernel / fx_reduce_kernel open one of them.
  const int *gate;
  // FX layouts (fixed-point interval histograms, see below): per (axis,
  // interval) predicted scale exponents and their per-axis minima (written
  // by refine_kernel for the next iteration), the global f64 sums of the
  // values too large for the fixed point, the hi-word limit of
  // RN(w2 2^k) + 2^52 below which a value is summed in fixed point
  const int *fx_k;              // [d][ng]
  const int *fx_kmin;           // [d]
  double *fx_spill;             // [d][ng]
  unsigned fx_lim;               // 0x43300000 + 2^(L-32): hi word of 2^52 + 2^L
  unsigned long long *fx_nspill;   // count of spilled values (statistics)
  int fx;                       // launch the FX layout of the compiled kernel
};

struct SegItem {   // a partial cube segment (key < 0: none)
  int key;
  double v1, v2;
};

// Row stride of the shared interval histograms, which are laid out
// [interval][axis] (stride = next power of two >= d, <= 16) rather than the
// reference's [axis][interval].  Lanes update axes in lane-rotated order, so
// the lanes of one ATOMS instruction hit distinct axes; with the axis as the
// fast index their 8-byte (4-byte) words then fall into distinct bank groups
// except for lanes sharing an axis, which collide with probability
// 1/(banks per row) -- instead of random interval addresses colliding freely.
// The host falls back to the unpadded stride d when the padded rows do not
// fit (e.g. d = 10 at ng = 1024), before giving up on shared histograms.
__host__ __device__ inline int hist_stride(int dims) {
  int s = 1;
  while (s < dims) s <<= 1;
  return s <= 16 ? s : dims;
}

// shared-memory layout helper (bytes)
__host__ __device__ inline size_t fill_smem_bytes(int dims, int ng, long long n_strat,
                                                  int smem_hist, int pairs, int hs,
                                                  int ridge_centres = 0, int hcopies = 1) {
  size_t b = 0;
  if (pairs) b += (size_t)dims * ng * 2 * sizeof(double);              // (E[i], dx[i])
  else b += (size_t)dims * (ng + 1) * sizeof(double);                  // edges
  if (smem_hist) b += (size_t)hs * ng * (hcopies * sizeof(double) + sizeof(unsigned));
  b = (b + 15) & ~(size_t)15;
  b += (n_strat <= DQ_TABLE_MAX ? (size_t)n_strat : 0) * sizeof(double);  // digit/N
  b += (size_t)ridge_centres * sizeof(double);                          // ridge c_i
  b += 16;                                                              // block flags
  return b;
}

// PAIRS: the map is staged as a table of (E[j][i], RN(E[j][i+1] - E[j][i]))
// 16-byte pairs, so each axis of a sample costs one LDS.128 instead of two
// LDS.64 and a DADD (the fill is bound by shared-memory wavefronts; random
// 16-byte accesses cost ~9 wavefronts per warp vs ~12 for two 8-byte ones).
// Kernel layouts (compile time for the (integrand, dims) specialisations;
// LAYOUT_RUNTIME reads the FillArgs flags).
constexpr int LAYOUT_EDGES = 0;     // edge rows + shared histograms
constexpr int LAYOUT_PAIRS = 1;     // pair table + shared histograms
constexpr int LAYOUT_RECORDS = 2;   // edge rows + records (hist.cuh)
constexpr int LAYOUT_RUNTIME = 3;   // generic kernel: a.smem_hist / a.records / global atomics
// SPLIT (many axes, separable integrand: the d = 20 Gaussian of cfg5): a
// cluster of two CTAs (two SMs) processes the same runs; CTA c samples axes
// [c d/2, (c+1) d/2) with their map rows and interval histograms in its own
// shared memory, and the pair swaps one (partial sum of (x_j - mu)^2, partial
// Jacobian) per run through distributed shared memory -- so d * ng
// histograms twice the size of one SM's shared memory stay on chip (no
// records through HBM).  Both CTAs combine the partials with the same
// commutative IEEE ops, i.e. get bit-identical f, jf and w2; CTA 0 keeps the
// cube sums.
constexpr int LAYOUT_SPLIT = 4;
// FX (bit 3 on EDGES or PAIRS): the interval histograms in per-(axis,
// interval) fixed point instead of f64 -- two u32 limbs per interval, the
// interval's scale exponent in the top byte of its u32 count word.  A value
// w2 becomes q = RN(w2 2^k) by one DFMA against 2^52 and is added with a
// value-returning u32 atomic on the low limb and a plain one (high bits +
// carry) on the high limb: three u32 shared atomics that issue back to back
// for all d axes, instead of d serialised LDS -> DADD -> ATOMS.CAST.SPIN
// loops (the f64 CAS loop costs ~2x the shared-memory wavefronts and is the
// L1 bound of the cfg4 fill).  The scales are predicted from the previous
// iteration's interval averages and the new map (refine_kernel); values at
// or above 2^L units go to a global f64 sum instead (fx_spill), and
// fx_reduce_kernel proves every interval's fixed-point sum precise to 2^-P
// of its total and free of wrap-around, or orders the iteration's fill
// redone in f64 (the gated second fill in the graph).
constexpr int LAYOUT_FX = 8;
constexpr int LAYOUT_EDGES_FX = LAYOUT_EDGES | LAYOUT_FX;
constexpr int LAYOUT_PAIRS_FX = LAYOUT_PAIRS | LAYOUT_FX;
constexpr int LAYOUT_SPLIT_FX = LAYOUT_SPLIT | LAYOUT_FX;
#ifndef VPB_FX_T
#define VPB_FX_T 42   // target: predicted interval average at 2^T units
#endif
#ifndef VPB_FX_P
#define VPB_FX_P 38   // precision proof: interval sum >= 2^P units per value
#endif
constexpr int FX_K_NONE = 1 << 20;   // no prediction (zero or non-finite average)
// hi + carry(old + lo): the high limb's addend after the low limb's atomic
// returned `old` (add.cc / addc: one IADD3 with carry out, one IADD.X)
__device__ __forceinline__ unsigned addc_u32(unsigned hi, unsigned old, unsigned lo) {
  unsigned h;
  asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}"
      : "=r"(h)
      : "r"(old), "r"(lo), "r"(hi));
  return h;
}
// Biased exponent (1023 + k) of an interval's scale 2^k: k = K + e with e the
// predicted exponent's offset from the base K = 1023 + e0 clamped to
// [0, 254]; no prediction -> 2^1023 (every normal value goes to the spill).
__host__ __device__ inline int fx_biased_exp(int k_pred, int e0) {
  if (k_pred >= FX_K_NONE) return 2046;
  const int off = k_pred - (e0 - 1023);
  return e0 + (off < 0 ? 0 : (off > 254 ? 254 : off));
}

// shared memory of the split layout (per CTA): map rows and histograms of d/2
// axes, digit table, double-buffered exchange slots and their mbarriers
__host__ __device__ inline size_t fill_split_smem_bytes(int dims, int ng, long long n_strat,
                                                        int nt, int hcopies = 1) {
  const int h = dims / 2;
  size_t b = (size_t)h * (ng + 1) * sizeof(double);
  b += (size_t)h * ng * (hcopies * sizeof(double) + sizeof(unsigned));
  b = (b + 15) & ~(size_t)15;
  b += (n_strat <= DQ_TABLE_MAX ? (size_t)n_strat : 0) * sizeof(double);
  b = (b + 16 + 15) & ~(size_t)15;                   // block flags
  b += (size_t)2 * (nt / 32) * 32 * 16;              // exchange slots [2][warps][32] double2
  b += (size_t)2 * (nt / 32) * 8;                    // their mbarriers
  return b;
}

// Integrands whose value does not depend on the order of the axes (up to the
// rounding of their sums/products): the fill may hand them the coordinates
// in a lane-dependent axis order (XPERM below).
template <int ID>
__host__ __device__ constexpr bool axis_symmetric() {
  return ID == VPB_GAUSSIAN || ID == VPB_MULTIPEAK || ID == VPB_RIDGE || ID == VPB_LINEAR ||
         ID == VPB_COSINE || ID == VPB_EXPONENTIAL || ID == VPB_ROOS_ARNOLD ||
         ID == VPB_MOROKOFF || ID == VPB_ASIAN_OPTION || ID == VPB_CONSTANT;
}

// Threads per CTA: FILL_NT (640: 96 registers), or 768 (80 registers) for
// the kernels whose integrand sums are streamed (Gaussian, 3-peak Gaussian:
// StreamSum keeps few partials live) and the many-axis records kernels --
// they fit 80 registers and gain from the sixth warp per scheduler (cfg2
// -1.3%, cfg1 -7%, cfg4 -5..7%, cfg5 -3%, cfg3 ridge -1% fill time), or
// a per-integrand count in table mode (below); the rest keep 640.
// Table mode: RN(digit/N) read from the shared digit table instead of d
// registers.  Round 1 (f64 CAS histograms) ran every table-mode kernel at
// 64 registers and 1024 threads.  Re-measured with the fixed-point
// histograms (round 2, alternating A/B, tools/ab_pair.sh / ab_registry.sh,
// fill time against 1024 threads): Roos & Arnold -7.4%, linear -7.5%,
// exponential -4.7% at 640 threads (96 registers); Morokoff -2.8%, path
// integral -2.2% at 768 (80); the Ridge (cfg3) stays at 1024 (640: +3.2%);
// and the Genz pair (cfg4a/b) is fastest out of table mode altogether, with
// the digits in registers at 768 threads (-2.9% / -4.0%).  Cosine (its cos
// spills) and the streamed Gaussians (cfg1/cfg2: their table reads compete
// with the pair table) keep the digits in registers.
// VPB_TABLE_NT: -1 per integrand as above, > 0 one count for all, 0 off.
#ifndef VPB_TABLE_NT
#define VPB_TABLE_NT -1
#endif
#ifndef VPB_REC_NT
#define VPB_REC_NT VPB_STREAM_NT
#endif
#ifndef VPB_SPLIT_NT
#define VPB_SPLIT_NT 768   // at most 768: the exchange slots grow with the warps
#endif
#ifndef VPB_TABLE_RIDGE
#define VPB_TABLE_RIDGE 1   // cfg3 -0.4%
#endif
#ifndef VPB_TABLE_MULTIPEAK
#define VPB_TABLE_MULTIPEAK 0
#endif
#ifndef VPB_TABLE_GENZ
#define VPB_TABLE_GENZ 0
#endif
template <int ID, int D>
__host__ __device__ constexpr bool dq_from_table() {
  return (((ID == VPB_GENZ_OSCILLATORY || ID == VPB_GENZ_PRODUCTPEAK) && VPB_TABLE_GENZ) ||
          ID == VPB_ROOS_ARNOLD ||
          (ID == VPB_MULTIPEAK && VPB_TABLE_MULTIPEAK) ||
          ID == VPB_LINEAR || ID == VPB_EXPONENTIAL || ID == VPB_MOROKOFF ||
          ID == VPB_PATH_INTEGRAL || (ID == VPB_RIDGE && VPB_TABLE_RIDGE)) &&
         D >= 3 && D <= 12 && VPB_TABLE_NT != 0;
}
// threads per CTA of a table-mode kernel
template <int ID>
__host__ __device__ constexpr int table_nt() {
  return VPB_TABLE_NT > 0 ? VPB_TABLE_NT
         : (ID == VPB_RIDGE || ID == VPB_GENZ_OSCILLATORY || ID == VPB_GENZ_PRODUCTPEAK) ? 1024
         : (ID == VPB_MOROKOFF || ID == VPB_PATH_INTEGRAL)                               ? 768
                                                                                         : 640;
}

// FX histogram update of one sample's w2 into DX axes' intervals (flat
// indices idx = interval * hs + local axis; the CTA's first axis is ax0).
// Count word = (biased scale exponent << 20) | count, so the count atomic
// returns the interval's scale 2^k as the high word of a double; y = fma(w2,
// 2^k, 2^52) holds q = RN(w2 2^k) in its low 52 bits, and (hi:lo) of y is
// added to the interval's 64-bit (hi:lo) limbs as it is: the low limb's atomic
// returns the old value for the carry, the high limb gains 0x43300000 per
// value on top of q's high bits, which fx_reduce_kernel removes exactly from
// the count.  No selects, no predicates kept across the axes: one max of the
// high words decides the rare spill path, which takes a too-large value back
// out (adds 0x43300000:0 - y) and sums it in f64 in global memory instead.
template <int DX>
__device__ __forceinline__ void fx_update(const int (&idx)[DX], double w2, unsigned *s_fx,
                                          int hs, int ng, int ax0, const FillArgs &a) {
  // slot i = [count word, lo limb, hi limb] at s_fx[3i..3i+2]: one address per
  // axis (IMAD, FMA pipe) for the three atomics, and a 12-byte stride that
  // spreads a warp's random slots over all 32 banks
  unsigned *p[DX];
  unsigned ow[DX], ql[DX], qh[DX];
#pragma unroll
  for (int j = 0; j < DX; j++) p[j] = s_fx + 3 * idx[j];
#pragma unroll
  for (int j = 0; j < DX; j++) ow[j] = atomicAdd(p[j], 1u);
  unsigned mx = 0u;
#pragma unroll
  for (int j = 0; j < DX; j++) {
    const double y = __fma_rn(w2, __hiloint2double((int)(ow[j] & 0xFFF00000u), 0), 0x1p52);
    ql[j] = (unsigned)__double2loint(y);
    qh[j] = (unsigned)__double2hiint(y);
    mx = max(mx, qh[j]);
  }
#pragma unroll
  for (int j = 0; j < DX; j++) ow[j] = atomicAdd(p[j] + 1, ql[j]);
#pragma unroll
  for (int j = 0; j < DX; j++) atomicAdd(p[j] + 2, addc_u32(qh[j], ow[j], ql[j]));
  if (mx >= a.fx_lim) {   // rare: q >= 2^L units (or not finite)
#pragma unroll
    for (int j = 0; j < DX; j++)
      if (qh[j] >= a.fx_lim) {
        const unsigned long long nv =
            (0x43300000ull << 32) - (((unsigned long long)qh[j] << 32) | ql[j]);
        const unsigned nl = (unsigned)nv;
        const unsigned o = atomicAdd(p[j] + 1, nl);
        atomicAdd(p[j] + 2, addc_u32((unsigned)(nv >> 32), o, nl));
        const int b = idx[j] / hs, ax = ax0 + idx[j] - b * hs;
        atomicAdd(a.fx_spill + (size_t)ax * ng + b, w2);
        atomicAdd(a.fx_nspill, 1ull);
      }
  }
}

template <int ID, int D, int LAYOUT_>
__host__ __device__ constexpr int fill_nt() {
  constexpr int LAYOUT = LAYOUT_ & 7;
  return (LAYOUT == LAYOUT_SPLIT)                    ? VPB_SPLIT_NT
         : dq_from_table<ID, D>()                    ? table_nt<ID>()
         : (LAYOUT == LAYOUT_RECORDS && D > 12)      ? VPB_REC_NT
         : ((ID == VPB_GAUSSIAN || ID == VPB_MULTIPEAK || ID == VPB_GENZ_OSCILLATORY ||
             ID == VPB_GENZ_PRODUCTPEAK || ID == VPB_RIDGE || VPB_ALL_NT768) &&
            D > 0 && D <= 12)                        ? VPB_STREAM_NT
                                                     : FILL_NT;
}

template <int ID, int D, int LAYOUT_>
__global__ void __launch_bounds__((fill_nt<ID, D, LAYOUT_>()), 1) fill_kernel(const FillArgs a) {
  constexpr int NT = fill_nt<ID, D, LAYOUT_>();
  constexpr int LAYOUT = LAYOUT_ & 7;
  constexpr bool FX = (LAYOUT_ & LAYOUT_FX) != 0;
  // FX in the split layout (fx_update takes the CTA's axis offset) is not
  // instantiated: measured slower on cfg5
  static_assert(!FX || LAYOUT == LAYOUT_EDGES || LAYOUT == LAYOUT_PAIRS || LAYOUT == LAYOUT_SPLIT,
                "FX: edges, pairs or split");
  if (a.gate != nullptr && *a.gate == 0) return;   // grid-uniform
  constexpr bool PAIRS = LAYOUT == LAYOUT_PAIRS;
  constexpr bool SPLIT = LAYOUT == LAYOUT_SPLIT;
  static_assert(!SPLIT || (ID == VPB_GAUSSIAN && D > 0 && D % 2 == 0),
                "split fill: the Gaussian at even d");
  constexpr int HX = SPLIT ? D / 2 : D;     // axes this CTA samples (SPLIT: half)
  const unsigned crank = SPLIT ? cluster_ctarank() : 0u;
  const unsigned partner = crank ^ 1u;
  const int ax0 = SPLIT ? (int)crank * HX : 0;   // first axis of this CTA
  // records layout with many axes: the first K0 axes are histogrammed in this
  // kernel's spare shared memory (next to the edges), the rest go to records
  constexpr int K0 = (LAYOUT == LAYOUT_RECORDS && D >= 12) ? REC_K0 : 0;
  // cube digits RN(digit/N) per axis in registers for small d; above that the
  // digits are kept packed and RN(digit/N) is read from the shared table
  constexpr bool DQ_REG = D == 0 || (D <= VPB_DQ_REG_MAX && !dq_from_table<ID, D>());
  // XPERM (power-of-two d, pair table, axis-symmetric integrand): at step s
  // lane l samples axis s ^ (l mod d).  The 8 lanes of a quarter-warp then
  // read 8 different axes, and with the pair table laid out [interval][axis]
  // (128-byte rows for d = 8) their 16-byte loads land in 8 different bank
  // quads -- conflict-free instead of ~10 wavefronts per LDS.128 for random
  // intervals of one axis.  Steps 2k, 2k+1 still cover one Philox block
  // (k ^ (l>>1)), so only the word order flips; the histogram updates are
  // already lane-spread (no barrel rotation); x and the Jacobian factors
  // reach the integrand in permuted order (bitwise the same coordinates; sums
  // and products round in a different order, within the parity tolerance).
  constexpr bool XPERM = PAIRS && (D == 2 || D == 4 || D == 8) && axis_symmetric<ID>();
  // STREAM (the Gaussian, and the 3-peak Gaussian of cfg2): the integrand's
  // pairwise sums of (x_j - mu_k)^2 are accumulated while the axes are
  // sampled (StreamSum: bit-identical to numpy's row sum of the terms in the
  // order they are sampled), so neither x[] nor the d squared terms per peak
  // are live across the sampling loop -- up to ~2d(peaks+1) fewer registers.
  // MP_FMA (the three-peak Gaussian, integrands.cuh VPB_MP_FMA): a running
  // fma per peak instead of the pairwise tree, in the lane's step order
  constexpr int NPK = ID == VPB_GAUSSIAN ? 1 : (ID == VPB_MULTIPEAK ? 3 : 0);
  constexpr bool STREAM = NPK > 0 && D >= 1 && D <= 128;
  constexpr bool MP_FMA = VPB_MP_FMA && STREAM && NPK == 3;
  // the Genz functors (cfg4) reduce left to right over the axes in order
  // (never XPERM-permuted): a running dot product / product is the streamed
  // form, bit-identical to integrands.cuh
  constexpr bool GSTREAM = (ID == VPB_GENZ_OSCILLATORY || ID == VPB_GENZ_PRODUCTPEAK) && D > 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // records chunks past this rank's shard: nothing to do (grid-uniform)
  if (a.tile_lo > 0 && a.tile_lo >= a.sched->ntiles) return;
  constexpr int MAXD = D > 0 ? D : VPB_MAX_DIMS;
  const int d = D > 0 ? D : a.dims;
  const int ng = a.ng;
  const int tid = threadIdx.x;
  const int hs = a.hs;   // histogram row stride (hist_stride(d), or d when that does not fit)

  // ---- shared memory carve-up
  double *s_edges = reinterpret_cast<double *>(smem_raw);
  double2 *s_pair = reinterpret_cast<double2 *>(smem_raw);
  size_t off = PAIRS ? (size_t)d * ng * sizeof(double2)
                     : (size_t)(SPLIT ? HX : d) * (ng + 1) * sizeof(double);
  double *s_hw = nullptr;
  unsigned *s_hc = nullptr;
  const int hcopies = (LAYOUT == LAYOUT_RECORDS) ? 1 : a.hcopies;
  if (a.smem_hist) {
    s_hw = reinterpret_cast<double *>(smem_raw + off);
    off += (size_t)hcopies * hs * ng * sizeof(double);
    s_hc = reinterpret_cast<unsigned *>(smem_raw + off);
    off += (size_t)hs * ng * sizeof(unsigned);
  }
  off = (off + 15) & ~(size_t)15;
  const bool dq_tab = a.n_strat <= DQ_TABLE_MAX;
  double *s_dq = reinterpret_cast<double *>(smem_raw + off);
  off += (dq_tab ? (size_t)a.n_strat : 0) * sizeof(double);
  // ridge: centres c_i = RN(i/(n-1)) (integrands.cuh ridge_window)
  constexpr bool RTAB = ID == VPB_RIDGE && D > 0;
  double *s_ctab = reinterpret_cast<double *>(smem_raw + off);
  const int n_cent = RTAB ? (int)a.P.p[0] : 0;
  off += (size_t)n_cent * sizeof(double);
  const int dbits = a.dig_bits;                 // bits per packed digit (!DQ_REG)
  const uint64_t dmask = (1ull << dbits) - 1;
  int *s_flag = reinterpret_cast<int *>(smem_raw + off);
  off = (off + 16 + 15) & ~(size_t)15;
  double2 *s_x = reinterpret_cast<double2 *>(smem_raw + off);   // SPLIT exchange slots
  off += SPLIT ? (size_t)2 * (NT / 32) * 32 * sizeof(double2) : 0;
  uint64_t *s_bar = reinterpret_cast<uint64_t *>(smem_raw + off);

  if constexpr (PAIRS) {
    for (int i = tid; i < d * ng; i += NT) {
      const int j = i / ng, b = i - j * ng;
      const double lo = a.edges[j * (ng + 1) + b];
      // [axis][interval], or [interval][axis] for XPERM
      s_pair[XPERM ? b * D + j : i] = make_double2(lo, __dadd_rn(a.edges[j * (ng + 1) + b + 1], -lo));
    }
  } else if constexpr (SPLIT) {   // this CTA's map rows
    for (int i = tid; i < HX * (ng + 1); i += NT) s_edges[i] = a.edges[(size_t)ax0 * (ng + 1) + i];
  } else {
    for (int i = tid; i < d * (ng + 1); i += NT) s_edges[i] = a.edges[i];
  }
  // FX: the scale base K (min over the axes' predicted exponents, clamped so
  // that every biased exponent 1023 + K + e, e <= 254, is a normal double's)
  // and each interval's offset e in the top byte of its count word (255: no
  // prediction -- the scale 2^1023, so every normal value goes to the spill)
  int fx_e0 = 0;
  if constexpr (FX) {
    int K = FX_K_NONE;
    for (int j = 0; j < d; j++) K = min(K, __ldg(a.fx_kmin + j));
    K = max(min(K, 1023 - 254), -1022);
    fx_e0 = 1023 + K;
  }
  if (a.smem_hist) {
    if constexpr (FX) {   // [count word, lo, hi] triples over s_hw and s_hc (one copy)
      unsigned *s_fx = reinterpret_cast<unsigned *>(s_hw);
      for (int i = tid; i < hs * ng; i += NT) {
        const int b = i / hs, j = i - b * hs;   // SPLIT: local axis j is ax0 + j
        s_fx[3 * i] = j < (SPLIT ? HX : d)
                          ? (unsigned)fx_biased_exp(__ldg(a.fx_k + (size_t)(ax0 + j) * ng + b), fx_e0)
                                << 20
                          : 0u;
        s_fx[3 * i + 1] = 0u;
        s_fx[3 * i + 2] = 0u;
      }
    } else {
      for (int i = tid; i < hcopies * hs * ng; i += NT) s_hw[i] = 0.0;
      for (int i = tid; i < hs * ng; i += NT) s_hc[i] = 0u;
    }
  }
  if (dq_tab)
    for (int i = tid; i < a.n_strat; i += NT) s_dq[i] = div_exact((double)i, a.nsf, a.rns);
  if constexpr (RTAB) {
    const double spacing = (double)n_cent - 1.0, rsp = 1.0 / spacing;
    for (int i = tid; i < n_cent; i += NT) s_ctab[i] = div_exact((double)i, spacing, rsp);
  }

  if (tid == 0) s_flag[0] = *a.status;   // an earlier iteration failed: nothing to fill
  if constexpr (SPLIT) {
    if (tid < 2 * (NT / 32)) {
      mbar_init(smem_u32(s_bar + tid), 1);
      fence_mbar_init_cluster();
    }
  }
  const Sched S = *a.sched;
  const PhiloxKeys &K = a.keys;
  const long long lo = S.lo, hi = S.hi, ntiles = S.ntiles;
  const unsigned long long batch = (unsigned long long)a.batch;
  const unsigned long long stride_half = (unsigned long long)((d + (d & 1)) >> 1);
  __syncthreads();
  int stop = s_flag[0];
  if constexpr (SPLIT) {   // barriers visible to the partner; the pair takes CTA 0's flag
    cluster_sync_all();
    stop = ld_dsmem_s32(mapa_u32(smem_u32(s_flag), 0));
    cluster_sync_all();
  }
  if (stop) return;   // block-uniform (cluster-uniform for SPLIT)

  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int xr = XPERM ? (lane & (D - 1)) : 0;   // XPERM: step s samples axis s ^ xr
  double nsf2, rns2;   // u/N = (2u)/(2N), exact scaling
  sample_consts(a.nsf, a.rns, nsf2, rns2);
  // this warp's tiles: [L + w*P + b, min(L + (w+1)*P, U)) in steps of the grid,
  // [L, U) = the launch's tile range
  const long long tL = a.tile_lo, tU = min(a.tile_hi, ntiles);
  const long long P = (tU - tL + NW - 1) / NW;
  // SPLIT: the two CTAs of a cluster walk the same tiles
  const long long cid = SPLIT ? (long long)(blockIdx.x >> 1) : (long long)blockIdx.x;
  const long long ncl = SPLIT ? (long long)(gridDim.x >> 1) : (long long)gridDim.x;
  const long long t_beg = tL + (long long)warp * P + cid;
  const long long t_end = min(tL + (long long)(warp + 1) * P, tU);
  // runs per lane / per warp tile of this schedule (records mode: FILL_RPT)
  const int rpt = sched_rpt(S);
  const long long tile_runs = 32ll * rpt;
  const long long rec0 = lo + tL * tile_runs;   // run of record 0 (records mode)
  // (k, slot) of this lane's first run in its first tile; advanced per grid stride
  unsigned long long g0 = (unsigned long long)(S.run_base + lo + t_beg * tile_runs +
                                               (long long)lane * rpt);
  unsigned long long kk = g0 / batch, slot = g0 % batch;
  // SPLIT: one swap of per-run partials with the partner CTA's same lane
  // (slot = step parity; the same number of steps in both CTAs)
  unsigned xstep = 0;
  auto pair_xchg = [&](double u, double v) -> double2 {
    const int slot_ = (int)(xstep & 1u);
    const unsigned par = (xstep >> 1) & 1u;
    xstep++;
    const int bi = slot_ * (NT / 32) + (tid >> 5);
    const uint32_t lbar = smem_u32(s_bar + bi);
    const uint32_t lbuf = smem_u32(s_x + bi * 32 + (tid & 31));
    st_async_f64x2(mapa_u32(lbuf, partner), u, v, mapa_u32(lbar, partner));
    if ((tid & 31) == 0) mbar_arrive_expect_tx(lbar, 32 * 16);
    mbar_wait_parity(lbar, par);
    return s_x[bi * 32 + (tid & 31)];
  };

  for (long long tile = t_beg; tile < t_end; tile += ncl) {
    const long long T0 = lo + tile * tile_runs;
    const long long T1 = min(T0 + tile_runs, hi);
    const long long c_first = a.tile_cube[tile];
    const long long c_last = a.tile_cube[tile + 1];
    const int nwin = (int)(c_last - c_first + 2);
    const long long *win = a.offsets + c_first;   // the tile's cube offsets (L1-resident)

    const long long r0 = T0 + (long long)lane * rpt;
    const long long r1 = min(r0 + (long long)rpt, T1);
    SegItem H{-1, 0.0, 0.0}, T{-1, 0.0, 0.0};
    int t_through = 0;
    // SPLIT: every lane takes part in lane 0's number of swaps
    const int nsteps = (int)min((long long)rpt, T1 - T0);

    if (r0 < r1) {
      // cube of r0: largest i with win[i] <= r0
      int lo_i = 0, hi_i = nwin - 2;
      while (lo_i < hi_i) {
        const int mid = (lo_i + hi_i + 1) >> 1;
        if (__ldg(win + mid) <= r0) lo_i = mid; else hi_i = mid - 1;
      }
      // run positions relative to r0 in 32-bit registers (cube bounds clamped
      // to [-1, RPT+1], which keeps every comparison below exact)
      auto rel = [&](long long v) { return (int)max(min(v - r0, (long long)rpt + 1), -1ll); };
      const int n = (int)(r1 - r0);
      int wi = lo_i;
      int cube = (int)c_first + wi;
      int cb = rel(__ldg(win + wi)), ce = rel(__ldg(win + wi + 1));
      int seg_beg = 0;
      double v1 = 0.0, v2 = 0.0;
      unsigned long long k = kk;
      // the batch slot (Philox counter words 2, 3) as two 32-bit halves: when
      // this lane's n runs neither reach the batch end nor carry into the
      // high word (nearly always), the low word just counts up; otherwise the
      // general 64-bit update with the batch wrap (vp/kernels.py:59-62)
      uint32_t sl_lo = (uint32_t)slot, sl_hi = (uint32_t)(slot >> 32);
      const bool sl_fast = slot + (unsigned long long)n < batch && sl_lo <= 0xFFFFFFFFu - (uint32_t)n;
      double dq[DQ_REG ? MAXD : 1];
      uint64_t dpk = 0;   // packed digits (!DQ_REG)
      auto load_digits = [&](int c) {
        uint32_t rem = (uint32_t)c;   // n_cubes < 2^31
        if constexpr (!DQ_REG) dpk = 0;
#pragma unroll
        for (int j = 0; j < (D > 0 ? D : d); j++) {
          const uint32_t q = a.nsdiv.div(rem);
          const uint32_t dig = rem - q * a.nsdiv.d;
          rem = q;
          if constexpr (DQ_REG) dq[j] = dq_tab ? s_dq[dig] : div_exact((double)dig, a.nsf, a.rns);
          else dpk |= (uint64_t)dig << (j * dbits);
        }
        if constexpr (XPERM && DQ_REG) {   // dq[s] <- dq[s ^ xr]: butterfly over the bits of xr
#pragma unroll
          for (int b = 1; b < D; b <<= 1) {
            const bool on = (xr & b) != 0;
#pragma unroll
            for (int j = 0; j < D; j++)
              if ((j & b) == 0) {
                const double lo_ = dq[j], hi_ = dq[j | b];
                dq[j] = on ? hi_ : lo_;
                dq[j | b] = on ? lo_ : hi_;
              }
          }
        }
      };
      // RN(digit_j / N) of the current cube
      auto dq_of = [&](int j) -> double {
        if constexpr (DQ_REG) {
          return dq[j];
        } else {
          const uint32_t dig = (uint32_t)((dpk >> (j * dbits)) & dmask);
          // n_strat**d < 2^31 keeps n_strat <= 1290 <= DQ_TABLE_MAX for d >= 3:
          // the table always exists there
          if constexpr (D >= 3) return s_dq[dig];
          else return dq_tab ? s_dq[dig] : div_exact((double)dig, a.nsf, a.rns);
        }
      };
      auto close_segment = [&](int seg_end) {
        const bool before = cb < seg_beg;   // cube started before this lane
        const bool after = ce > seg_end;    // cube continues past this lane
        if (!before && !after) {
          if (!SPLIT || crank == 0) {
            a.s1[cube] = v1;
            a.s2[cube] = v2;
          }
        } else if (before && !after) {
          H = {cube, v1, v2};
        } else {
          T = {cube, v1, v2};
          t_through = before ? 1 : 0;
        }
      };
      load_digits(cube);
      // Philox block of this run's first axis pair: k*stride/2 (vp/kernels.py:59-66)
      unsigned long long base = k * stride_half;
      for (int rr = 0; rr < n; rr++) {
        if (rr >= ce) {
          close_segment(rr);
          do { wi++; } while (__ldg(win + wi + 1) <= r0 + rr);
          cube = (int)c_first + wi;
          cb = rel(__ldg(win + wi));
          ce = rel(__ldg(win + wi + 1));
          seg_beg = rr;
          v1 = 0.0; v2 = 0.0;
          load_digits(cube);
        }
        // ---- sample (vp/kernels.py:59-88)
        StreamSum<STREAM ? HX : 1> gacc[NPK > 0 ? NPK : 1];
        double mpr[NPK > 0 ? NPK : 1];   // MP_FMA: |x - mu_k|^2 by a running fma
        double gz = ID == VPB_GENZ_PRODUCTPEAK ? 1.0 : 0.0;   // GSTREAM running value
        auto stream_axis = [&](int step, double xs) {   // x of the axis sampled at `step`
          if constexpr (GSTREAM && ID == VPB_GENZ_OSCILLATORY) {   // s += x_j a_j
            gz = __fma_rn(xs, a.P.p[1 + step], gz);
          } else if constexpr (GSTREAM) {   // den *= a_j^-2 + (x_j - u_j)^2
            const double u = __dadd_rn(xs, -a.P.p[D + step]);
            gz = __dmul_rn(gz, __fma_rn(u, u, a.P.p[step]));
          }
          if constexpr (STREAM) {
#pragma unroll
            for (int k = 0; k < NPK; k++) {   // vp/integrands.py:135-139 (x_j - mu_k)^2
              const double u = __dadd_rn(xs, -a.P.p[NPK == 1 ? 0 : 7 + k]);
              if constexpr (MP_FMA) mpr[k] = step == 0 ? __dmul_rn(u, u) : __fma_rn(u, u, mpr[k]);
              else gacc[k].add(step, __dmul_rn(u, u));
            }
          }
        };
        double x[SPLIT ? HX : MAXD];
        int iv[SPLIT ? HX : MAXD];
        double jac = 1.0;
        uint64_t w0 = 0, w1 = 0;
        if constexpr (SPLIT) {
#pragma unroll
          for (int jl = 0; jl < HX; jl++) {   // axes ax0 + jl (ax0 even: same Philox pairs)
            const int j = ax0 + jl;
            if ((jl & 1) == 0) {
              const unsigned long long blk = base + (unsigned long long)(j >> 1);
              philox((uint32_t)blk, (uint32_t)(blk >> 32), sl_lo, sl_hi, K,
                     w0, w1);
            }
            x[jl] = sample_axis((jl & 1) ? w1 : w0, dq_of(j), nsf2, rns2, a.ngf, ng,
                                EdgeRow{s_edges + jl * (ng + 1)}, jac, iv[jl], jl == 0);
            const double u = __dadd_rn(x[jl], -a.P.p[0]);   // (x_j - mu)^2, this half
            gacc[0].add(jl, __dmul_rn(u, u));
          }
        } else if constexpr (XPERM) {
#pragma unroll
          for (int k2 = 0; k2 < D / 2; k2++) {
            const unsigned long long blk = base + (unsigned long long)(k2 ^ (xr >> 1));
            philox((uint32_t)blk, (uint32_t)(blk >> 32), sl_lo, sl_hi, K,
                   w0, w1);
            const uint64_t wa = (xr & 1) ? w1 : w0, wb = (xr & 1) ? w0 : w1;
            const int s0 = 2 * k2, s1 = s0 + 1;
            const double dq0 = DQ_REG ? dq[DQ_REG ? s0 : 0] : dq_of(s0 ^ xr);
            const double dq1 = DQ_REG ? dq[DQ_REG ? s1 : 0] : dq_of(s1 ^ xr);
            x[s0] = sample_axis(wa, dq0, nsf2, rns2, a.ngf, ng,
                                EdgePairsT<D>{s_pair + (s0 ^ xr)}, jac, iv[s0], k2 == 0);
            x[s1] = sample_axis(wb, dq1, nsf2, rns2, a.ngf, ng,
                                EdgePairsT<D>{s_pair + (s1 ^ xr)}, jac, iv[s1]);
            stream_axis(s0, x[s0]);
            stream_axis(s1, x[s1]);
          }
        } else {
#pragma unroll
        for (int j = 0; j < (D > 0 ? D : d); j++) {
          if ((j & 1) == 0) {
            const unsigned long long blk = base + (unsigned long long)(j >> 1);
            philox((uint32_t)blk, (uint32_t)(blk >> 32), sl_lo, sl_hi, K,
                   w0, w1);
          }
          if constexpr (PAIRS)
            x[j] = sample_axis((j & 1) ? w1 : w0, dq_of(j), nsf2, rns2, a.ngf, ng,
                               EdgePairs{s_pair + j * ng}, jac, iv[j], j == 0);
          else
            x[j] = sample_axis((j & 1) ? w1 : w0, dq_of(j), nsf2, rns2, a.ngf, ng,
                               EdgeRow{s_edges + j * (ng + 1)}, jac, iv[j], j == 0);
          stream_axis(j, x[j]);
          if constexpr (LAYOUT == LAYOUT_RECORDS) {
            // the axis group is complete: store its intervals now, so they
            // are not live across the integrand
            if (j >= K0 && (((j - K0) & 7) == 7 || j == D - 1)) {
              const int g = (j - K0) >> 3;   // records hold axes K0 + 8g ..
              uint32_t wv[4];
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const int j0 = K0 + 8 * g + 2 * q, j1 = j0 + 1;
                const uint32_t lo16 = j0 <= j ? (uint32_t)iv[j0 <= j ? j0 : 0] : 0u;
                const uint32_t hi16 = j1 <= j ? (uint32_t)iv[j1 <= j ? j1 : 0] : 0u;
                wv[q] = lo16 | (hi16 << 16);
              }
              *reinterpret_cast<uint4 *>(
                  a.rec_iv + ((size_t)g * a.rec_ch + (T0 - rec0) + rr * 32 + lane) * 8) =
                  make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
          }
        }
        }   // !XPERM
        // ---- integrand (f_batch), finiteness (vp/executor.py:119-127)
        double gsum = 0.0;
        if constexpr (SPLIT) {
          // swap (partial sum, partial Jacobian) with the partner; a + b and
          // a * b are commutative in IEEE arithmetic, so both CTAs get the same bits
          const double2 o = pair_xchg(gacc[0].result(), jac);
          gsum = __dadd_rn(gacc[0].result(), o.x);
          jac = __dmul_rn(jac, o.y);
        } else if constexpr (STREAM) {
          gsum = gacc[0].result();
        }
        double f;
        if constexpr (STREAM && NPK == 1) {   // integrands.cuh VPB_GAUSSIAN, streamed sum
          f = __dmul_rn(a.P.p[2], fast_exp_nonpos(-div_exact(gsum, a.P.p[3], a.P.p[4])));
        } else if constexpr (MP_FMA) {
          double out = 0.0;
#pragma unroll
          for (int k = 0; k < NPK; k++)
            out = __dadd_rn(out, fast_exp_nonpos(__dmul_rn(mpr[k], -a.P.p[5])));
          f = __dmul_rn(out, __dmul_rn(a.P.p[2], a.P.p[6]));
        } else if constexpr (STREAM) {        // VPB_MULTIPEAK with 3 peaks (host-checked)
          double e[NPK];
#pragma unroll
          for (int k = 0; k < NPK; k++)
            e[k] = __dmul_rn(a.P.p[2],
                             fast_exp_nonpos(-div_exact(gacc[k].result(), a.P.p[3], a.P.p[5])));
          double out = 0.0;
#pragma unroll
          for (int k = 0; k < NPK; k++) out = __dadd_rn(out, e[k]);
          f = div_exact(out, a.P.p[4], a.P.p[6]);
        } else if constexpr (GSTREAM && ID == VPB_GENZ_OSCILLATORY) {
          f = cos(__dadd_rn(a.P.p[0], gz));   // cos(2 pi u_1 + a.x)
        } else if constexpr (GSTREAM) {
          f = __drcp_rn(gz);   // 1 / prod of the denominators (integrands.cuh)
        } else {
          f = integrand<ID, D>(x, d, a.P, RTAB ? s_ctab : nullptr);
        }
        if (!isfinite(f)) {
          atomicMin(a.err_run, (unsigned long long)(r0 + rr));
          atomicOr(a.status, 1);
        } else {
          const double jf = __dmul_rn(jac, f);
          const double w2 = __dmul_rn(jf, jf);
          v1 = __dadd_rn(v1, jf);
          v2 = __dadd_rn(v2, w2);
          // ---- interval histograms (vp/kernels.py:100-105)
          constexpr bool RT = LAYOUT == LAYOUT_RUNTIME;
          if (LAYOUT == LAYOUT_RECORDS) {
            a.rec_w2[(T0 - rec0) + rr * 32 + lane] = w2;   // intervals stored while sampling
            if constexpr (K0 > 0) {
              // axes 0..K0-1 here, lane-rotated as below
              const int rot = lane % K0;
              int idx[K0];
#pragma unroll
              for (int j = 0; j < K0; j++) idx[j] = iv[j] * hs + j;
#pragma unroll
              for (int b = 1; b < K0; b <<= 1) {
                const bool on = (rot & b) != 0;
                int t[K0];
#pragma unroll
                for (int j = 0; j < K0; j++) t[j] = on ? idx[(j + b) % K0] : idx[j];
#pragma unroll
                for (int j = 0; j < K0; j++) idx[j] = t[j];
              }
#pragma unroll
              for (int j = 0; j < K0; j++) {
                atomicAdd(&s_hw[idx[j]], w2);
                atomicAdd(&s_hc[idx[j]], 1u);
              }
            }
          } else if (RT && a.records) {
            // deferred to hist_records_kernel: w^2 and the intervals, 8 axes
            // per 16-byte group (coalesced over a warp's RPT-strided rows)
            const long long ri = (T0 - rec0) + rr * 32 + lane;   // lane-interleaved slot
            a.rec_w2[ri] = w2;
            constexpr int NG = (MAXD + 7) / 8;
#pragma unroll
            for (int g = 0; g < NG; g++) {
              if (D == 0 && 8 * g >= d) break;
              uint32_t wv[4];
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const int j0 = 8 * g + 2 * q, j1 = j0 + 1;
                const uint32_t lo16 = (D > 0 ? j0 < D : j0 < d) ? (uint32_t)iv[j0 < MAXD ? j0 : 0] : 0u;
                const uint32_t hi16 = (D > 0 ? j1 < D : j1 < d) ? (uint32_t)iv[j1 < MAXD ? j1 : 0] : 0u;
                wv[q] = lo16 | (hi16 << 16);
              }
              *reinterpret_cast<uint4 *>(a.rec_iv + ((size_t)g * a.rec_ch + ri) * 8) =
                  make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
          } else if constexpr (SPLIT) {
            // this CTA's axes, lane-rotated (barrel rotation by lane % HX)
            const int rot = lane % HX;
            int idx[HX];
#pragma unroll
            for (int jl = 0; jl < HX; jl++) idx[jl] = iv[jl] * hs + jl;
#pragma unroll
            for (int b = 1; b < HX; b <<= 1) {
              const bool on = (rot & b) != 0;
              int t[HX];
#pragma unroll
              for (int jl = 0; jl < HX; jl++) t[jl] = on ? idx[(jl + b) % HX] : idx[jl];
#pragma unroll
              for (int jl = 0; jl < HX; jl++) idx[jl] = t[jl];
            }
            if constexpr (FX) {
              fx_update<HX>(idx, w2, reinterpret_cast<unsigned *>(s_hw), hs, ng, ax0, a);
            } else {
              double *s_hwl = s_hw + (hcopies > 1 ? (size_t)(lane >> 4) * hs * ng : 0);
#pragma unroll
              for (int jl = 0; jl < HX; jl++) {
                atomicAdd(&s_hwl[idx[jl]], w2);
                atomicAdd(&s_hc[idx[jl]], 1u);
              }
            }
          } else if (RT && a.det == 1) {
            // deterministic mode, pass 1: per (axis, interval) the largest w2
            // (u64 max of the non-negative doubles' bit patterns: exact and
            // order-independent) and the count pick pass 2's scale
            for (int j = 0; j < d; j++) {
              const int b = iv[j];
              const unsigned long long wb = (unsigned long long)__double_as_longlong(w2);
              if (a.smem_hist) {
                atomicMax(reinterpret_cast<unsigned long long *>(s_hw) + (size_t)b * hs + j, wb);
                atomicAdd(&s_hc[b * hs + j], 1u);
              } else {
                atomicMax(reinterpret_cast<unsigned long long *>(a.hw_glob) + (size_t)j * ng + b, wb);
                atomicAdd(&a.hc_glob[j * ng + b], 1ull);
              }
            }
          } else if (RT && a.det == 2) {
            // deterministic mode, pass 2: each w2 in the fixed point of its
            // (axis, interval)'s scale 2^k (count x max < 2^62), summed with
            // 64-bit integer atomics -- exact, so the update order cannot
            // change the bits (vpb_desc flags)
            for (int j = 0; j < d; j++) {
              const int b = iv[j];
              const int kb = __ldg(a.bin_k + (size_t)j * ng + b);
              const unsigned long long q = __double2ull_rn(scalbn(w2, kb));
              if (a.smem_hist) {
                atomicAdd(reinterpret_cast<unsigned long long *>(s_hw) + (size_t)b * hs + j, q);
                atomicAdd(&s_hc[b * hs + j], 1u);
              } else {
                atomicAdd(reinterpret_cast<unsigned long long *>(a.hw_glob) + (size_t)j * ng + b, q);
                atomicAdd(&a.hc_glob[j * ng + b], 1ull);
              }
            }
          } else if (!RT || a.smem_hist) {
            // Lane-rotated dimension order: at step s lane l updates dim
            // (s + l) mod d.  Lanes of a warp usually sit in the same cube,
            // i.e. the same stratum of every axis, so with a common order
            // most CAS instructions have two lanes on one interval and
            // retry; rotated, a step's lanes are spread over d histograms.
            const int rot = lane % d;
            // flat histogram index of each axis, rotated so that slot s holds
            // axis (s + rot) mod d (XPERM: step s already holds axis s ^ xr)
            int idx[MAXD];
#pragma unroll
            for (int j = 0; j < (D > 0 ? D : d); j++) idx[j] = iv[j] * hs + (XPERM ? (j ^ xr) : j);
            if constexpr (XPERM) {
            } else if constexpr (D > 1) {
#pragma unroll
              // d >= 9: at most ~11 strata per axis at any feasible n_eval
              // (n_strat^d <= n_eval/4), so ~90+ intervals per stratum and few
              // same-slot collisions: one stage (rotation by 0/1) is enough and
              // saves 3d SELs (Roos & Arnold 10-D fill -2.3%; cfg4's d = 6 with
              // 40 intervals per stratum needs all three stages: 1 stage +10%)
              constexpr int RSTAGES = VPB_ROT_STAGES > 0 ? VPB_ROT_STAGES : (D >= 9 ? 1 : 8);
              for (int b = 1; b < D && b < (1 << RSTAGES); b <<= 1) {   // barrel rotation by rot
                const bool on = (rot & b) != 0;
                int t[D];
#pragma unroll
                for (int j = 0; j < D; j++) t[j] = on ? idx[(j + b) % D] : idx[j];
#pragma unroll
                for (int j = 0; j < D; j++) idx[j] = t[j];
              }
            } else if constexpr (D == 0) {
              int ivr[MAXD];
              for (int j = 0; j < d; j++) ivr[j] = iv[(j + rot) % d];
              for (int j = 0; j < d; j++) idx[j] = ivr[j] * hs + (j + rot) % d;
            }
            // f64: the compiler's LDS -> DADD -> ATOMS.CAST.SPIN loop.  (A
            // batched variant -- all d reads, adds and value-returning
            // ATOMS.CAS issued back to back, losers retried -- was measured
            // 17% slower on cfg2 at round start and still 8% slower after
            // the layout changes: the value-returning CAS costs more
            // shared-memory wavefronts than CAST.SPIN, and wavefronts bind.)
            if constexpr (FX) {
              fx_update<(D > 0 ? D : 1)>(idx, w2, reinterpret_cast<unsigned *>(s_hw), hs, ng,
                                         0, a);
            } else {
            // two copies of the sums: the half-warps update different copies,
            // so fewer lanes of one CAS instruction collide on an interval
            double *s_hwl = s_hw + (hcopies > 1 ? (size_t)(lane >> 4) * hs * ng : 0);
#pragma unroll
            for (int j = 0; j < (D > 0 ? D : d); j++) {
              atomicAdd(&s_hwl[idx[j]], w2);
              atomicAdd(&s_hc[idx[j]], 1u);
            }
            }
          } else {
#pragma unroll
            for (int j = 0; j < (D > 0 ? D : d); j++) {
              atomicAdd(&a.hw_glob[j * ng + iv[j]], w2);
              atomicAdd(&a.hc_glob[j * ng + iv[j]], 1ull);
            }
          }
        }
        if (__builtin_expect(sl_fast, 1)) {
          ++sl_lo;
        } else {
          unsigned long long s64 = (((unsigned long long)sl_hi << 32) | sl_lo) + 1ull;
          if (s64 == batch) { s64 = 0; base += stride_half; }
          sl_lo = (uint32_t)s64;
          sl_hi = (uint32_t)(s64 >> 32);
        }
      }
      close_segment(n);
      if constexpr (SPLIT)   // lane 0's remaining swaps (fewer runs in the tile's end)
        for (int rr = n; rr < nsteps; rr++) pair_xchg(0.0, 1.0);
    } else if constexpr (SPLIT) {
      for (int rr = 0; rr < nsteps; rr++) pair_xchg(0.0, 1.0);
    }

    // ---- warp segmented scan of the tail items (chain values flow forward)
    // element: (flag = chain restarts here, v); flag=1 also for "no tail".
    int fl = (T.key < 0) ? 1 : (t_through ? 0 : 1);
    double e1 = T.key < 0 ? 0.0 : T.v1, e2 = T.key < 0 ? 0.0 : T.v2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int pf = __shfl_up_sync(0xffffffffu, fl, o);
      const double p1 = __shfl_up_sync(0xffffffffu, e1, o);
      const double p2 = __shfl_up_sync(0xffffffffu, e2, o);
      if (lane >= o && !fl) { e1 = __dadd_rn(p1, e1); e2 = __dadd_rn(p2, e2); }
      if (lane >= o) fl |= pf;
    }
    // fl is now "rooted": the inclusive chain has a restart inside the tile
    const int pfl = __shfl_up_sync(0xffffffffu, fl, 1);
    const double pe1 = __shfl_up_sync(0xffffffffu, e1, 1);
    const double pe2 = __shfl_up_sync(0xffffffffu, e2, 1);
    // ---- heads close chains; the one whose chain began before the tile
    // (lane 0's head, or a head after an unrooted chain) is the head carry
    bool head_carry = false;
    double h1 = H.v1, h2 = H.v2;
    if (H.key >= 0) {
      if (lane > 0) { h1 = __dadd_rn(pe1, H.v1); h2 = __dadd_rn(pe2, H.v2); }
      if (lane > 0 && pfl) {
        if (!SPLIT || crank == 0) {
          a.s1[H.key] = h1;
          a.s2[H.key] = h2;
        }
      } else {
        head_carry = true;
      }
    }
    if (SPLIT && crank != 0) head_carry = false;   // CTA 0 keeps the cube sums
    if (head_carry) {
      a.ck_head[tile] = H.key;
      a.cv_head[2 * tile] = h1;
      a.cv_head[2 * tile + 1] = h2;
    }
    const unsigned any_head = __ballot_sync(0xffffffffu, head_carry);
    if (lane == 0 && any_head == 0 && (!SPLIT || crank == 0)) a.ck_head[tile] = -1;
    // ---- the tile's last lane with runs publishes the tail carry
    const int last = (int)((T1 - T0 + rpt - 1) / rpt) - 1;
    if (lane == last && (!SPLIT || crank == 0)) {
      if (T.key >= 0) {
        a.ck_tail[tile] = T.key;
        a.cv_tail[2 * tile] = e1;
        a.cv_tail[2 * tile + 1] = e2;
        a.ct_through[tile] = fl ? 0 : 1;
      } else {
        a.ck_tail[tile] = -1;
        a.ct_through[tile] = 0;
      }
    }
    // advance this lane's RNG coordinates by one grid stride of tiles
    kk += (unsigned long long)a.dk;
    slot += (unsigned long long)a.ds;
    if (slot >= batch) { slot -= batch; kk++; }
  }

  if (a.smem_hist) {
    __syncthreads();
    const int nh = LAYOUT == LAYOUT_RECORDS ? K0 : (SPLIT ? HX : d);   // axes histogrammed here
    // SPLIT: rows [ax0, ax0 + HX) of the cluster's slice
    double *hw = a.hw_part + (SPLIT ? (size_t)cid * d * ng + (size_t)ax0 * ng
                                    : (size_t)blockIdx.x * nh * ng);
    unsigned *hc = a.hc_part + (SPLIT ? (size_t)cid * d * ng + (size_t)ax0 * ng
                                      : (size_t)blockIdx.x * nh * ng);
    // records layout: the chunks of an iteration add into the CTA's slice
    const bool acc = LAYOUT == LAYOUT_RECORDS && a.tile_lo > 0;
    for (int i = tid; i < nh * ng; i += NT) {   // back to [axis][interval]
      const int j = i / ng, b = i - j * ng;
      if constexpr (FX) {   // the raw (hi:lo) limbs and the count word (with e)
        const unsigned *t = reinterpret_cast<const unsigned *>(s_hw) + 3 * (b * hs + j);
        reinterpret_cast<unsigned long long *>(hw)[i] = ((unsigned long long)t[2] << 32) | t[1];
        hc[i] = t[0];
        continue;
      }
      double v = s_hw[b * hs + j];
      if (hcopies > 1) v = __dadd_rn(v, s_hw[(size_t)hs * ng + b * hs + j]);
      hw[i] = acc ? __dadd_rn(hw[i], v) : v;
      hc[i] = acc ? hc[i] + s_hc[b * hs + j] : s_hc[b * hs + j];
    }
  }
  if constexpr (SPLIT) cluster_sync_all();   // no CTA leaves while its partner may still write
}

}  // namespace vpb
