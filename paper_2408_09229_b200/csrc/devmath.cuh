// devmath.cuh -- bit-exact arithmetic building blocks for the VEGAS+ hot path.
//
// The translation unit is compiled with -fmad=false: every plain `a*b+c` is
// two IEEE-rounded operations, exactly like the numba/numpy reference
// ("0 FMA").  Fused multiply-adds appear only where written
// explicitly as __fma_rn and are then proven exact (Markstein division,
// integer->double reconstruction) or used in functions whose reference is a
// non-bitwise libm/SIMD transcendental (exp).
#pragma once
#include <cstdint>

namespace vpb {

// ---------------------------------------------------------------- Philox --
// Philox4x32-10 (vp/rng.py:24-60).  Counter = (block lo, block hi, stream lo,
// stream hi), key = (seed lo, seed hi); returns the two 64-bit output words
// (c0<<32|c1, c2<<32|c3).  The ten round keys are hoisted into registers by
// the caller (they depend on the seed only -> uniform across the grid).
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
  PhiloxKeys() = default;
  __host__ __device__ explicit PhiloxKeys(uint64_t seed) {
    uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; r++) {
      k0[r] = a; k1[r] = b;
      a += 0x9E3779B9u; b += 0xBB67AE85u;
    }
  }
};

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       const PhiloxKeys &K, uint64_t &w0, uint64_t &w1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t p0 = (uint64_t)c0 * 0xD2511F53u;   // IMAD.WIDE.U32
    const uint64_t p1 = (uint64_t)c2 * 0xCD9E8D57u;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k0[r];   // LOP3
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  w0 = ((uint64_t)c0 << 32) | c1;
  w1 = ((uint64_t)c2 << 32) | c3;
}

// ------------------------------------------------ uniforms and division --
// u = (w >> 11) * 2^-53 exactly (vp/rng.py:68), in two FP64 ops instead of a
// quarter-rate I2F.F64.U64: the low 52 bits become the mantissa of a number
// in [1,2), and bit 52 adds 0.5.  Exhaustively argued in
// tools/proofs/markstein_div.c (checked against (double)m * 2^-53).
__device__ __forceinline__ double unit_from_word(uint64_t w) {
  const uint64_t m = w >> 11;
  const double t = __longlong_as_double((long long)(0x3FF0000000000000ull | (m & 0xFFFFFFFFFFFFFull)));
  // bit 52 of m (= bit 63 of w) adds 0.5: build 0.5 / 0.0 from the high word only
  const double half = __hiloint2double((int)(w >> 63) * 0x3FE00000, 0);
  return __fma_rn(__dadd_rn(t, -1.0), 0.5, half);   // both steps exact
}

// RN(a / b) for b = n_strat (integer) and a = a Philox uniform or an integer
// digit: q0 = RN(a*r), e = a - b*q0 (exact by FMA), q = RN(q0 + e*r) with
// r = RN(1/b).  Markstein's correction; checked bitwise against IEEE
// division for every n_strat <= 4100 (tools/proofs/markstein_div.c).
__device__ __forceinline__ double div_exact(double a, double b, double r) {
  const double q0 = __dmul_rn(a, r);
  const double e = __fma_rn(-q0, b, a);
  return __fma_rn(e, r, q0);
}

// ------------------------------------------------ one axis of one sample --
// vp/kernels.py:67-87 for dimension j of one run:
//   u = (w>>11)*2^-53, y = RN(RN(digit/N) + RN(u/N)), y >= 1 -> nextafter(1,0),
//   t = RN(y*ng), iv = min(trunc t, ng-1), frac = RN(t - iv),
//   x = RN(lo + RN(frac*dx)), jac factor RN(ng*dx).
// Operation economy (bitwise identical results):
//  * u/N without materialising u: up = 1 + (bits 11..62 of w)*2^-52 in [1,2)
//    is pure bit assembly, a = up - (1 - bit63) = 2u exactly (Sterbenz), and
//    RN(u/N) = RN(a/(2N)) by the Markstein sequence with (2N, RN(1/N)/2) --
//    the N case scaled by a power of two (tools/proofs/markstein_div.c);
//  * the y clamp on the bit pattern (y >= 0: y >= 1 iff hi word >= 0x3FF00000);
//  * trunc(t) by the 2^52 shifter in round-toward-zero, iv clamped in the
//    integer domain and converted back exactly with the same shifter.
// dq = RN(digit/N); nsf2 = 2N; rns2 = RN(1/N)/2; edge(iv, lo, dx) returns
// E[j][iv] and RN(E[j][iv+1] - E[j][iv]) of the axis.
// VPB_A_I2F: 2u as the integer w >> 11 converted exactly (I2F.F64.U64), the
// Markstein constants scaled by 2^52 / 2^-52 (sample_consts) -- the same
// quotient bits, three integer instructions fewer per axis than the bit
// assembly below.
#ifndef VPB_A_I2F
#define VPB_A_I2F 1   // measured: cfg2 fill -2.8%, cfg4b -2.6%
#endif
// VPB_YCLAMP_DMNMX: the y >= 1 clamp as fmin against 0x1.fffffffffffffp-1
// (y >= 0, never NaN: the same bits) instead of three integer instructions
// on the high/low words -- measured no better: sm_100a has no FP64 min
// instruction, fmin is DSETP.MIN + two selects.
#ifndef VPB_YCLAMP_DMNMX
#define VPB_YCLAMP_DMNMX 0
#endif
// (2N, RN(1/N)/2) for sample_axis's u/N = 2u/(2N), in the scaling its 2u uses
__host__ __device__ inline void sample_consts(double nsf, double rns, double &nsf2,
                                              double &rns2) {
  nsf2 = VPB_A_I2F ? nsf * 0x1p53 : 2.0 * nsf;
  rns2 = VPB_A_I2F ? rns * 0x1p-53 : 0.5 * rns;
}
// first: the run's first axis (a constant after unrolling) -- jac = its
// factor instead of RN(1 * factor), the same bits
template <class EdgeFn>
__device__ __forceinline__ double sample_axis(uint64_t w, double dq, double nsf2, double rns2,
                                              double ngf, int ng, EdgeFn edge, double &jac,
                                              int &iv, bool first = false) {
#if VPB_A_I2F
  const double a = __ull2double_rn(w >> 11);   // 2u * 2^52, exact (< 2^53)
#else
  uint32_t whi, wlo;   // split opaquely: keeps the bit-63 test a 32-bit compare
  asm("mov.b64 {%0, %1}, %2;" : "=r"(wlo), "=r"(whi) : "l"(w));
  const double up = __hiloint2double((int)(((whi >> 11) & 0xFFFFFu) | 0x3FF00000u),
                                     (int)__funnelshift_r(wlo, whi, 11));
  const double cm = __hiloint2double((~(int)whi >> 31) & 0x3FF00000, 0);   // 1 - bit63
  const double a = __dadd_rn(up, -cm);                                      // 2u, exact
#endif
  const double q0 = __dmul_rn(a, rns2);                                     // Markstein
  const double v = __fma_rn(__fma_rn(-q0, nsf2, a), rns2, q0);             // RN(u/N)
  const double ys = __dadd_rn(dq, v);
#if VPB_YCLAMP_DMNMX
  const double t = __dmul_rn(fmin(ys, 0x1.fffffffffffffp-1), ngf);
#else
  int yhi = __double2hiint(ys), ylo = __double2loint(ys);
  ylo = (yhi >= 0x3FF00000) ? -1 : ylo;                                     // y >= 1 ->
  yhi = min(yhi, 0x3FEFFFFF);                                               // 0x3FEFFFFFFFFFFFFF
  const double t = __dmul_rn(__hiloint2double(yhi, ylo), ngf);
#endif
  const double sh = __dadd_rz(t, 4503599627370496.0);   // 2^52 + trunc(t)
  const int ivj = min(__double2loint(sh), ng - 1);
  // 2^52 + iv has the shifter's high word (0x43300000): reuse that register
  const double fiv = __dadd_rn(__hiloint2double(__double2hiint(sh), ivj), -4503599627370496.0);
  const double frac = __dadd_rn(t, -fiv);
  double elo, dx;
  edge(ivj, elo, dx);
  jac = first ? __dmul_rn(ngf, dx) : __dmul_rn(jac, __dmul_rn(ngf, dx));
  iv = ivj;
  return __dadd_rn(elo, __dmul_rn(frac, dx));
}

// edge accessors: a row of VegasMap.edges, or a (E[i], RN(E[i+1]-E[i])) pair
// table precomputed once per fill (one 16-byte shared load per axis)
struct EdgeRow {
  const double *e;
  __device__ __forceinline__ void operator()(int i, double &lo, double &dx) const {
    lo = e[i];
    dx = __dadd_rn(e[i + 1], -lo);
  }
};
template <int RS>   // pair table laid out [interval][axis], RS axes per row
struct EdgePairsT {
  const double2 *p;   // points at the axis column
  __device__ __forceinline__ void operator()(int i, double &lo, double &dx) const {
    const double2 v = p[i * RS];
    lo = v.x;
    dx = v.y;
  }
};
struct EdgePairs {
  const double2 *p;
  __device__ __forceinline__ void operator()(int i, double &lo, double &dx) const {
    const double2 v = p[i];
    lo = v.x;
    dx = v.y;
  }
};

// ------------------------------------------------------------------ exp --
// exp(x) with < 1 ulp error on the normal range, no table, branch-free:
// k = rint(x/ln2) via the 1.5*2^52 shifter, two-step Cody-Waite reduction,
// a degree-11 near-minimax polynomial on |r| <= ln2/2 (Chebyshev fit, error
// 3.2e-18; max 0.96 ulp over 2e7 samples against expl -- the degree-13
// Taylor form it replaced measured 0.88 ulp and cost two more DFMAs),
// scaling by 2^k split in two factors so underflow/overflow saturate (to 0 /
// inf).  NaN propagates (the non-finite detection of vp/executor.py:120-126
// relies on it).  The reference evaluates numpy's SIMD exp / libm exp, which
// are not correctly rounded either: integrand values agree to a few ulp.
// Coefficients live in constant memory so the DFMAs take c[][] operands
// instead of materialising 64-bit immediates with UMOV pairs.
static __constant__ double kExp[17] = {
    6755399441055744.0,          // 0: 1.5 * 2^52 shifter
    1.4426950408889634074,       // 1: 1/ln2
    -6.93147180369123816490e-01, // 2: -ln2 hi (trailing zeros)
    -1.90821492927058770002e-10, // 3: -ln2 lo
    // 4..15: c11 .. c0
    2.5110037605963777e-08,
    2.763263963904103e-07,
    2.755724091857897e-06,
    2.4801485482328494e-05,
    0.00019841269890047113,
    0.0013888888952314775,
    0.008333333333319601,
    0.0416666666664881,
    0.1666666666666668,
    0.5000000000000019,
    1.0,
    1.0,
    1400.0};                    // 16: clamp
__device__ __forceinline__ double fast_exp_core(double x) {
  double kd = __fma_rn(x, kExp[1], kExp[0]);
  const int k = __double2loint(kd);
  kd = __dadd_rn(kd, -kExp[0]);
  double r = __fma_rn(kd, kExp[2], x);
  r = __fma_rn(kd, kExp[3], r);
  double p = kExp[4];
#pragma unroll
  for (int i = 5; i <= 15; i++) p = __fma_rn(p, r, kExp[i]);
  const int k1 = k >> 1, k2 = k - k1;
  const double s1 = __longlong_as_double((long long)(k1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(k2 + 1023) << 52);
  return __dmul_rn(__dmul_rn(p, s1), s2);
}

// General exp: NaN-propagating clamps (non-finite integrand detection).
__device__ __forceinline__ double fast_exp(double x) {
  x = (x < -kExp[16]) ? -kExp[16] : x;
  x = (x > kExp[16]) ? kExp[16] : x;
  return fast_exp_core(x);
}

// Table form (VPB_EXP_TAB, Tang's method): exp(x) = 2^m * 2^(j/32) * exp(r),
// n = 32m + j = RN(32 x / ln2), |r| <= ln2/64, so exp(r) needs a degree-6
// Taylor polynomial (truncation 3.5e-18 relative) instead of degree 11: 13
// FP64 instructions instead of 18, plus one L1-resident gather of
// RN(2^(j/32)) (256 bytes, read-only path).  Error ~1.5 ulp, like the core
// form's.  Measured slower (cfg2 fill 3.002 vs 2.942 ms, cfg5 +1%: the
// gather's latency and registers cost more than the five DFMAs), so off.
#ifndef VPB_EXP_TAB
#define VPB_EXP_TAB 0
#endif
static __device__ const double kExp2Tab[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237,
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,
    1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332,
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,
    1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072,
    1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002};
static __constant__ double kExpT[10] = {
    6755399441055744.0,        // 0: 1.5 * 2^52 shifter
    46.16624130844683,         // 1: 32/ln2
    -0x1.62e42fefa0000p-6,     // 2: -ln2/32 hi (36 bits: kd * hi exact for |kd| < 2^17)
    -5.145609244655338e-14,    // 3: -ln2/32 lo
    // 4..9: 1/6! .. 1/1!, then 1 (p = fma(p, r, 1))
    0.001388888888888889, 0.008333333333333333, 0.041666666666666664,
    0.16666666666666666, 0.5, 1.0};
__device__ __forceinline__ double fast_exp_tab(double x) {   // x in [-1400, 1400]
  double kd = __fma_rn(x, kExpT[1], kExpT[0]);
  const int n = __double2loint(kd);
  const double t = __ldg(kExp2Tab + (n & 31));   // issued early, used last
  kd = __dadd_rn(kd, -kExpT[0]);
  double r = __fma_rn(kd, kExpT[2], x);
  r = __fma_rn(kd, kExpT[3], r);
  double p = kExpT[4];
#pragma unroll
  for (int i = 5; i <= 9; i++) p = __fma_rn(p, r, kExpT[i]);
  p = __fma_rn(p, r, 1.0);
  const int m = n >> 5;   // floor(n / 32)
  const int m1 = m >> 1, m2 = m - m1;
  const double s1 = __longlong_as_double((long long)(m1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(m2 + 1023) << 52);
  return __dmul_rn(__dmul_rn(__dmul_rn(p, t), s1), s2);
}

// exp of a finite, non-positive argument (Gaussian exponents of finite
// points): one DMNMX clamp.
__device__ __forceinline__ double fast_exp_nonpos(double x) {
#if VPB_EXP_TAB
  return fast_exp_tab(fmax(x, -kExp[16]));
#else
  return fast_exp_core(fmax(x, -kExp[16]));
#endif
}

// 32-bit unsigned division by a runtime-constant divisor D in [1, 2^31]
// for numerators n < 2^31: q = (umulhi(n, m) + n) >> l with l = ceil(log2 D),
// m = floor(2^32 (2^l - D) / D) + 1 (Granlund-Montgomery).  Used for the
// mixed-radix cube digits (vp/kernels.py:76-77); checked exhaustively in
// tests/test_capi_cpu.py::test_magic_division.
struct MagicDiv {
  uint32_t m, l, d;
  MagicDiv() = default;
  __host__ __device__ explicit MagicDiv(uint32_t D) : d(D) {
    l = 0;
    while (l < 32 && (1ull << l) < D) l++;
    m = (uint32_t)((((1ull << 32) * ((1ull << l) - D)) / D) + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};

// ----------------------------------------------- numpy pairwise summation --
// numpy float64 add.reduce of a contiguous row: used for
// the integrands' `.sum(axis=1)` over a compile-time number of terms.
template <int N>
__device__ __forceinline__ double pw_sum(const double *a) {
  if constexpr (N < 8) {
    double res = 0.0;
#pragma unroll
    for (int i = 0; i < N; i++) res = __dadd_rn(res, a[i]);
    return res;
  } else if constexpr (N <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    constexpr int full = N - (N % 8);
#pragma unroll
    for (int i = 8; i < full; i += 8)
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = full; i < N; i++) res = __dadd_rn(res, a[i]);
    return res;
  } else {
    constexpr int n2 = (N / 2) - ((N / 2) % 8);
    return __dadd_rn(pw_sum<n2>(a), pw_sum<N - n2>(a + n2));
  }
}

// numpy's pairwise sum of N terms (8 <= N <= 128) accumulated as the terms
// arrive in index order: the 8 accumulators r[k] = a[k] + a[k+8] + ... are
// complete once a[full-1] is in (full = N - N%8), then the tree combines
// them and the tail a[full..N) is added in order -- bit-identical to
// pw_sum<N>, with only 8 partial sums live instead of N terms.
template <int N>
struct PairwiseAcc {
  static_assert(N >= 8 && N <= 128, "one numpy leaf");
  static constexpr int FULL = N - (N % 8);
  double r[8];
  double res;
  // j is the term index; called from fully unrolled loops, so every branch
  // folds at compile time
  __device__ __forceinline__ void add(int j, double v) {
    if (j < 8) {
      r[j] = v;
    } else if (j < FULL) {
      r[j % 8] = __dadd_rn(r[j % 8], v);
    } else {
      res = __dadd_rn(res, v);
    }
    if (j == FULL - 1)
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  }
};

// numpy's pairwise sum of N terms accumulated in index order with few live
// partials, bit-identical to pw_sum<N> (fully unrolled callers: all branches
// fold):  N < 8 sequential from 0.0;  8 <= N < 16 the 8-leaf tree
// ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) combined pair by pair (3 partials live),
// then the tail;  16 <= N <= 128 PairwiseAcc (8 partials).
template <int N>
struct StreamSum {
  static_assert(N >= 1 && N <= 128, "one numpy leaf");
  double p0, p1, q0, res;
  PairwiseAcc<(N >= 16 ? N : 16)> big;
  __device__ __forceinline__ void add(int j, double v) {
    if constexpr (N < 8) {
      res = (j == 0) ? __dadd_rn(0.0, v) : __dadd_rn(res, v);
    } else if constexpr (N < 16) {
      if (j >= 8) { res = __dadd_rn(res, v); return; }
      switch (j & 3) {
        case 0: p0 = v; break;
        case 1: p0 = __dadd_rn(p0, v); break;
        case 2: p1 = v; break;
        default: {
          const double q = __dadd_rn(p0, __dadd_rn(p1, v));
          if (j == 3) q0 = q;
          else res = __dadd_rn(q0, q);
        }
      }
    } else {
      big.add(j, v);
    }
  }
  __device__ __forceinline__ double result() const {
    if constexpr (N >= 16) return big.res;
    else return res;
  }
};

// Runtime-length version (recursion unrolled with an explicit stack).
__device__ __forceinline__ double pw_leaf(const double *a, long long n) {
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = a[j];
  long long i;
  for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ inline double pw_sum_rt(const double *a, long long n) {
  // iterative post-order traversal of numpy's split tree
  struct Frame { long long off, n; int state; double left; };
  Frame st[48];
  int sp = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame &f = st[sp];
    if (f.n <= 128) { ret = pw_leaf(a + f.off, f.n); sp--; continue; }
    long long n2 = f.n / 2; n2 -= n2 % 8;
    if (f.state == 0) { f.state = 1; st[sp + 1] = {f.off, n2, 0, 0.0}; sp++; continue; }
    if (f.state == 1) { f.left = ret; f.state = 2; st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.0}; sp++; continue; }
    ret = __dadd_rn(f.left, ret);
    sp--;
  }
  return ret;
}

}  // namespace vpb
