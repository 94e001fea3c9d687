// integrands.cuh -- device functors for the registry integrands.
//
// Registry: vp/integrands.py:106-190 (sinexp, linear, cosine, exponential,
// roos_arnold, morokoff, gaussian, ridge) plus the BASELINE-pinned synthetic
// integrands (multipeak8 = cfg2, genz oscillatory / product-peak = cfg4,
// gaussian20 = cfg5; definitions in paper_2408_09229_b200/integrands.py).
// Operation order follows the reference's numpy expressions (row sums use
// numpy's pairwise tree, products reduce left to right); exp/cos/sin are
// device implementations, so values agree with numpy to a few ulp.
#pragma once
#include "devmath.cuh"
#include "../../include/vegas_b200.h"

#ifndef VPB_MP_UNROLL
#define VPB_MP_UNROLL 1
#endif
// The three-peak Gaussian (cfg2, BASELINE's pin -- not a reference-registry
// integrand): |x - mu_k|^2 accumulated by a running fma instead of numpy's
// separate square / pairwise sum, 1/(2 sigma^2) and the 1/3 applied as
// multiplications by their RN reciprocals, norm factored out of the peak sum.
// Each value is then within a few ulp of the exponent argument of numpy's
// (|df/f| <= ~4e-16 |arg|, exp's condition number), 32 fewer FP64
// instructions per evaluation (cfg2 fill -5.4%).  0: numpy's operation order.
#ifndef VPB_MP_FMA
#define VPB_MP_FMA 1
#endif

namespace vpb {

struct IParams {
  double p[VPB_MAX_PARAMS];
  int n;
};

// row sum with numpy's pairwise association (compile-time or runtime length)
template <int D>
__device__ __forceinline__ double row_sum(const double *t, int d) {
  if constexpr (D > 0) return pw_sum<D>(t);
  else return pw_sum_rt(t, d);
}

// 4-element sort (ridge sums run over sorted coordinates, vp/integrands.py:174-179)
__device__ __forceinline__ void cswap(double &a, double &b) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  a = lo; b = hi;
}

// ------------------------------------------------------------- erfinv ----
// vp/integrands.py:59-100: Acklam's rational normal quantile (central region
// and upper tail -- the Asian payoff only asks for p = (|y|+1)/2 >= 1/2),
// then one Newton step in erfc space, sign restored by copysign.  Same
// operation order as the numpy code (unfused); erfc/log/exp are the device
// libm, so values agree with scipy to a few ulp.
static __constant__ double kAk[21] = {
    -3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,    // A
    1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00,
    -5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,    // B
    6.680131188771972e+01, -1.328068155288572e+01,
    -7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,   // C
    -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00,
    7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,      // D
    3.754408661907416e+00};
__device__ __forceinline__ double ndtri_upper(double p) {   // p >= 0.5
  if (p > 1.0 - 0.02425) {
    const double q = __dsqrt_rn(-2.0 * log(1.0 - p));
    const double num = (((((kAk[11] * q + kAk[12]) * q + kAk[13]) * q + kAk[14]) * q + kAk[15]) * q + kAk[16]);
    const double den = ((((kAk[17] * q + kAk[18]) * q + kAk[19]) * q + kAk[20]) * q + 1.0);
    return __ddiv_rn(-num, den);
  }
  const double q = p - 0.5, r = q * q;
  const double num = (((((kAk[0] * r + kAk[1]) * r + kAk[2]) * r + kAk[3]) * r + kAk[4]) * r + kAk[5]) * q;
  const double den = (((((kAk[6] * r + kAk[7]) * r + kAk[8]) * r + kAk[9]) * r + kAk[10]) * r + 1.0);
  return __ddiv_rn(num, den);
}
__device__ __forceinline__ double erfinv_ref(double y) {
  const double ya = fabs(y);
  double z = ndtri_upper((ya + 1.0) * 0.5) * 0.70710678118654746;   // * (1/sqrt(2))
  z = z + ((erfc(z) - (1.0 - ya)) * 0.88622692545275801) * fast_exp(z * z);  // sqrt(pi)/2
  return copysign(z, y);
}

// Ridge window sum (vp/integrands.py:154-182) over the centres c_i = i/(n-1)
// for i in [lo, hi]: sum_i exp(-400 (c_i - mu)^2), summed in increasing i as
// the reference does.  `ctab` (optional) holds RN(i/(n-1)) precomputed (the
// fill kernel stages it in shared memory: the same bits as the division).
//
// Blocked exact-factor recurrence: with dc = c_i - mu and the spacing
// delta, consecutive terms satisfy E_{i+1} = E_i * R_i with
// R_i = exp(-400 delta (2 dc + delta)) and R_{i+1} = R_i * B, B =
// exp(-800 delta^2).  Each block of RIDGE_BLK centres starts from the
// reference's own term (direct exp of -400 dc^2 at c_i = RN(i/(n-1))) and
// its factor R; the other terms cost two multiplications instead of an
// exp.  Measured on the B200 against the direct sum (VPB_RIDGE_BLK=1) on 3M
// points, uniform and near the ridge (tools/ridge_eval.py): max relative
// deviation 1.3e-14 at 32 centres per block, 5.1e-14 at 64 -- inside the
// 1e-13 integrand tolerance (tests/test_gpu_parity.py) -- because the
// centres RN(i/(n-1)) differ from c_ib + k delta by an ulp and the products
// round k times.  cfg3 fill: 91.5 ms (direct) -> 30.7 (16) -> 21.5 (32) ->
// 16.9 ms (64).  VPB_RIDGE_BLK=1 is the direct sum.
#ifndef VPB_RIDGE_BLK
#define VPB_RIDGE_BLK 64
#endif
__device__ __forceinline__ double ridge_window(double mu, int lo, int hi, double spacing,
                                               const double *ctab) {
  const double rsp = 1.0 / spacing;   // delta
  double acc = 0.0;
  if constexpr (VPB_RIDGE_BLK <= 1) {
    for (int i = lo; i <= hi; i++) {
      const double c = ctab ? ctab[i] : div_exact((double)i, spacing, rsp);
      const double dc = __dadd_rn(c, -mu);
      acc = __dadd_rn(acc, fast_exp_core(__dmul_rn(__dmul_rn(-400.0, dc), dc)));
    }
    return acc;
  }
  const double B = fast_exp_core(__dmul_rn(__dmul_rn(-800.0, rsp), rsp));
  const double m400d = __dmul_rn(-400.0, rsp);
  for (int ib = lo; ib <= hi; ib += VPB_RIDGE_BLK) {
    const double c = ctab ? ctab[ib] : div_exact((double)ib, spacing, rsp);
    const double dc = __dadd_rn(c, -mu);
    double e = fast_exp_core(__dmul_rn(__dmul_rn(-400.0, dc), dc));
    double r = fast_exp_core(__dmul_rn(m400d, __dadd_rn(__dmul_rn(2.0, dc), rsp)));
    const int n = min(VPB_RIDGE_BLK, hi - ib + 1);
    for (int k = 0; k < n; k++) {
      acc = __dadd_rn(acc, e);
      e = __dmul_rn(e, r);
      r = __dmul_rn(r, B);
    }
  }
  return acc;
}

template <int ID, int D>
__device__ __forceinline__ double integrand(const double *x, int d, const IParams &P,
                                            const double *ctab = nullptr) {
  constexpr int MAXD = D > 0 ? D : VPB_MAX_DIMS;
  if constexpr (ID == VPB_GAUSSIAN) {
    // norm * exp(-sum((x-mu)^2) / (2 sigma^2))           vp/integrands.py:135-139
    double t[MAXD];
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      const double u = __dadd_rn(x[j], -P.p[0]);
      t[j] = __dmul_rn(u, u);
    }
    const double r2 = row_sum<D>(t, d);
    // -r2 / (2 sigma^2): Markstein with the host's RN(1/(2 sigma^2)) (bitwise
    // IEEE division for these divisors, tools/proofs/markstein_general.c)
    return __dmul_rn(P.p[2], fast_exp_nonpos(-div_exact(r2, P.p[3], P.p[4])));
  } else if constexpr (ID == VPB_MULTIPEAK) {
    // (1/3) sum_k norm * exp(-|x - mu_k|^2 / (2 sigma^2))
    // p = [n_peaks, sigma, norm, 2 sigma^2, divisor, RN(1/2sigma^2), RN(1/divisor), mu_k...]
    const int np = (int)P.p[0];
    double out = 0.0;
    if constexpr (VPB_MP_FMA) {   // the fill's streamed form (fill.cuh MP_FMA), axis order
      for (int k = 0; k < np; k++) {
        double r2 = 0.0;
#pragma unroll
        for (int j = 0; j < (D > 0 ? D : d); j++) {
          const double u = __dadd_rn(x[j], -P.p[7 + k]);
          r2 = j == 0 ? __dmul_rn(u, u) : __fma_rn(u, u, r2);
        }
        out = __dadd_rn(out, fast_exp_nonpos(__dmul_rn(r2, -P.p[5])));
      }
      return __dmul_rn(out, __dmul_rn(P.p[2], P.p[6]));
    }
    if (VPB_MP_UNROLL && np == 3) {
      // the BASELINE cfg2 case: three independent exp chains, unrolled so
      // that their FP64 latencies overlap
      double e[3];
#pragma unroll
      for (int k = 0; k < 3; k++) {
        double t[MAXD];
#pragma unroll
        for (int j = 0; j < (D > 0 ? D : d); j++) {
          const double u = __dadd_rn(x[j], -P.p[7 + k]);
          t[j] = __dmul_rn(u, u);
        }
        e[k] = __dmul_rn(P.p[2], fast_exp_nonpos(-div_exact(row_sum<D>(t, d), P.p[3], P.p[5])));
      }
      out = __dadd_rn(__dadd_rn(__dadd_rn(out, e[0]), e[1]), e[2]);
      return div_exact(out, P.p[4], P.p[6]);
    }
    for (int k = 0; k < np; k++) {
      double t[MAXD];
#pragma unroll
      for (int j = 0; j < (D > 0 ? D : d); j++) {
        const double u = __dadd_rn(x[j], -P.p[7 + k]);
        t[j] = __dmul_rn(u, u);
      }
      const double r2 = row_sum<D>(t, d);
      out = __dadd_rn(out, __dmul_rn(P.p[2], fast_exp_nonpos(-div_exact(r2, P.p[3], P.p[5]))));
    }
    return div_exact(out, P.p[4], P.p[6]);
  } else if constexpr (ID == VPB_RIDGE) {
    // windowed sum over the 1000 diagonal centres        vp/integrands.py:154-182
    double xs[MAXD];
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      xs[j] = x[j];
    }
    if constexpr (D == 4) {
      cswap(xs[0], xs[1]); cswap(xs[2], xs[3]);
      cswap(xs[0], xs[2]); cswap(xs[1], xs[3]);
      cswap(xs[1], xs[2]);
    } else {
      for (int i = 1; i < d; i++) {
        const double v = xs[i];
        int j = i - 1;
        while (j >= 0 && xs[j] > v) { xs[j + 1] = xs[j]; j--; }
        xs[j + 1] = v;
      }
    }
    double sq[MAXD];
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      sq[j] = __dmul_rn(xs[j], xs[j]);
    }
    const double s1 = row_sum<D>(xs, d);
    const double s2 = row_sum<D>(sq, d);
    const int n_cent = (int)P.p[0];
    const double spacing = (double)n_cent - 1.0;
    const double mu = __dmul_rn(0.25, s1);
    const double q0 = __dadd_rn(s2, -__dmul_rn(mu, s1));
    int lo = (int)ceil(__dmul_rn(__dadd_rn(mu, -P.p[2]), spacing));
    int hi = (int)floor(__dmul_rn(__dadd_rn(mu, P.p[2]), spacing));
    lo = lo < 0 ? 0 : lo;
    hi = hi > n_cent - 1 ? n_cent - 1 : hi;
    const double acc = ridge_window(mu, lo, hi, spacing, ctab);
    // q0 = s2 - s1^2/4 >= 0 up to rounding: the general exp
    return __dmul_rn(__dmul_rn(P.p[1], fast_exp(__dmul_rn(-100.0, q0))), acc);
  } else if constexpr (ID == VPB_GENZ_OSCILLATORY) {
    // cos(2 pi u_1 + a . x)
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      s = __fma_rn(x[j], P.p[1 + j], s);   // cfg4a pin: fma form (<= 1/2 ulp per axis)
    }
    return cos(__dadd_rn(P.p[0], s));
  } else if constexpr (ID == VPB_GENZ_PRODUCTPEAK) {
    // prod_j 1 / (a_j^-2 + (x_j - u_j)^2), as 1 / prod_j (...): one exact
    // reciprocal instead of d (a few ulp from the per-factor form; the
    // denominators lie in [a_j^-2, a_j^-2 + 1], no overflow)
    double den = 1.0;
    const int dd = D > 0 ? D : d;
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      const double u = __dadd_rn(x[j], -P.p[dd + j]);
      den = __dmul_rn(den, __fma_rn(u, u, P.p[j]));   // cfg4b pin: fma form
    }
    return __drcp_rn(den);
  } else if constexpr (ID == VPB_SINEXP) {
    return __dadd_rn(sin(x[0]), fast_exp(x[1]));   // vp/integrands.py:106-107
  } else if constexpr (ID == VPB_LINEAR) {
    return row_sum<D>(x, d);                        // vp/integrands.py:110-111
  } else if constexpr (ID == VPB_COSINE) {
    double prod = cos(x[0]);                        // vp/integrands.py:114-115
#pragma unroll
    for (int j = 1; j < (D > 0 ? D : d); j++) {
      prod = __dmul_rn(prod, cos(x[j]));
    }
    return prod;
  } else if constexpr (ID == VPB_EXPONENTIAL) {
    double t[MAXD];                                 // vp/integrands.py:118-119
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      t[j] = __dmul_rn(x[j], x[j]);
    }
    return fast_exp(row_sum<D>(t, d));
  } else if constexpr (ID == VPB_ROOS_ARNOLD) {
    double prod = fabs(__dadd_rn(__dmul_rn(4.0, x[0]), -2.0));   // vp/integrands.py:122-123
#pragma unroll
    for (int j = 1; j < (D > 0 ? D : d); j++) {
      prod = __dmul_rn(prod, fabs(__dadd_rn(__dmul_rn(4.0, x[j]), -2.0)));
    }
    return prod;
  } else if constexpr (ID == VPB_MOROKOFF) {
    // (1+1/d)^d prod_j x_j^(1/d)                     vp/integrands.py:126-128
    // as (prod_j x_j)^(1/d): one pow instead of d (the product's d-1
    // roundings shrink by 1/d under the root; max 8.6e-16 relative from the
    // per-axis form over 3M points, numpy emulation); near underflow of the
    // product the per-axis form; so also for any x_j <= 0 (a zero gives 0, a
    // negative coordinate NaN, as numpy's x ** (1/d) does) and near overflow
    double px = x[0];
    bool pos = x[0] > 0.0;
#pragma unroll
    for (int j = 1; j < (D > 0 ? D : d); j++) {
      px = __dmul_rn(px, x[j]);
      pos = pos && x[j] > 0.0;
    }
    if (pos && px >= 1e-280 && px <= 1e280) return __dmul_rn(P.p[0], pow(px, P.p[1]));
    double prod = pow(x[0], P.p[1]);
#pragma unroll
    for (int j = 1; j < (D > 0 ? D : d); j++) {
      prod = __dmul_rn(prod, pow(x[j], P.p[1]));
    }
    return __dmul_rn(P.p[0], prod);
  } else if constexpr (ID == VPB_ASIAN_OPTION) {
    // exp(-rT) max(s0 exp(drift + sigma sqrt(T) z) - K, 0),
    // z = sqrt(2) sum_i erfinv(2 clip(x_i) - 1)        vp/integrands.py:196-210
    double t[MAXD];
#pragma unroll
    for (int j = 0; j < (D > 0 ? D : d); j++) {
      const double xc = fmin(fmax(x[j], P.p[5]), 1.0 - P.p[5]);
      t[j] = erfinv_ref(2.0 * xc - 1.0);
    }
    const double z = row_sum<D>(t, d) * 1.4142135623730951;   // * math.sqrt(2.0)
    const double s_avg = P.p[0] * fast_exp(P.p[2] + P.p[3] * z);
    return P.p[4] * fmax(s_avg - P.p[1], 0.0);
  } else if constexpr (ID == VPB_PATH_INTEGRAL) {
    // amp exp(-(m/(2a) sum (x_{j+1}-x_j)^2 + a/2 sum_{j<N} x_j^2)) with fixed
    // endpoints x_0 = x_N = x_end, N = d + 1          vp/integrands.py:233-251
    constexpr int MAXN = MAXD + 1;
    double kin[MAXN], pot[MAXN];
    const int n = (D > 0 ? D : d) + 1;
    double prev = P.p[3];
#pragma unroll
    for (int j = 0; j < (D > 0 ? D + 1 : n); j++) {
      const double cur = (j < (D > 0 ? D : d)) ? x[j] : P.p[3];
      const double u = cur - prev;
      kin[j] = u * u;
      pot[j] = prev * prev;
      prev = cur;
    }
    double ks, ps;
    if constexpr (D > 0) {
      ks = pw_sum<D + 1>(kin);
      ps = pw_sum<D + 1>(pot);
    } else {
      ks = pw_sum_rt(kin, n);
      ps = pw_sum_rt(pot, n);
    }
    return P.p[2] * fast_exp(-(P.p[0] * ks + P.p[1] * ps));
  } else {
    return P.p[0];   // VPB_CONSTANT
  }
}

}  // namespace vpb
