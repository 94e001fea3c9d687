/* Accuracy of the device exp (devmath.cuh fast_exp_core: Cody-Waite
 * reduction + degree-11 near-minimax polynomial, coefficients below) against
 * long-double expl, next to the degree-13 Taylor form it replaced.  Both
 * must stay below 1 ulp.  Build: gcc -O2 -mfma exp_accuracy.c -lm;
 * argument = samples in millions (default 20). */
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static double T13[14];
static const double C11[12] = {1.0, 1.0, 0.5000000000000019, 0.1666666666666668, 0.0416666666664881, 0.008333333333319601, 0.0013888888952314775, 0.00019841269890047113, 2.4801485482328494e-05, 2.755724091857897e-06, 2.763263963904103e-07, 2.5110037605963777e-08};
static double core(double x, const double *c, int deg) {
  double kd = fma(x, 1.4426950408889634074, 6755399441055744.0);
  int64_t kb; memcpy(&kb, &kd, 8); int k = (int)(int32_t)(kb & 0xffffffff);
  kd = kd - 6755399441055744.0;
  double r = fma(kd, -6.93147180369123816490e-01, x);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = c[deg];
  for (int i = deg - 1; i >= 0; i--) p = fma(p, r, c[i]);
  int k1 = k >> 1, k2 = k - k1;
  int64_t b1 = (int64_t)(k1 + 1023) << 52, b2 = (int64_t)(k2 + 1023) << 52;
  double s1, s2; memcpy(&s1, &b1, 8); memcpy(&s2, &b2, 8);
  return (p * s1) * s2;
}
static uint64_t s = 88172645463325252ull;
static inline uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char **argv) {
  const long total = (argc > 1 ? atol(argv[1]) : 20) * 1000000L;
  double f = 1; T13[0] = 1;
  for (int i = 1; i <= 13; i++) { f *= i; T13[i] = 1.0 / f; }
  double maxa = 0, maxb = 0; long nb_a = 0, nb_b = 0, n = 0;
  for (long i = 0; i < total; i++) {
    double x = ((double)(xr() >> 11) * 0x1p-53) * 1400.0 - 700.0;
    if (i & 1) x = ((double)(xr() >> 11) * 0x1p-53) * 60.0 - 30.0;
    long double ref = expl((long double)x);
    double ra = core(x, T13, 13), rb = core(x, C11, 11);
    double ulp = nextafter((double)ref, INFINITY) - (double)ref;
    double ea = fabsl((long double)ra - ref) / ulp, eb = fabsl((long double)rb - ref) / ulp;
    if (ea > maxa) maxa = ea; if (eb > maxb) maxb = eb;
    if (ra != (double)ref) nb_a++; if (rb != (double)ref) nb_b++;
    n++;
  }
  printf("taylor13: max %.3f ulp, not-RN %.4f%%   cheb11: max %.3f ulp, not-RN %.4f%%\n", maxa, 100.0*nb_a/n, maxb, 100.0*nb_b/n);
  return (maxa < 1.0 && maxb < 1.0) ? 0 : 1;
}
