/* Random check that the 3-op Markstein division (q0 = a*y, e = fma(-q0,b,a),
 * q = fma(e,y,q0), y = RN(1/b)) equals IEEE a/b for the integrand divisors
 * used by the device functors (2 sigma^2 of the registry Gaussians, the
 * multipeak divisor 3, the ridge spacing 999) over numerators spanning
 * [2^-60, 2^60].  Build: gcc -O2 -mfma markstein_general.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 0x9E3779B97F4A7C15ull;
static inline uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char **argv) {
  const long total = argc > 1 ? atol(argv[1]) * 1000L : 200000000L;
  const double sig[] = {0.01, 0.05, 0.1};
  double bs[8]; int nb = 0;
  for (int i = 0; i < 3; i++) bs[nb++] = 2.0 * pow(sig[i], 2.0);  /* python: 2.0 * sigma ** 2 */
  bs[nb++] = 3.0; bs[nb++] = 999.0;
  long bad = 0, n = 0;
  for (int k = 0; k < nb; k++) {
    const double b = bs[k], y = 1.0 / b;
    for (long i = 0; i < total / nb; i++) {
      uint64_t bits = (xr() & 0xFFFFFFFFFFFFFull) | ((uint64_t)(1023 - 60 + (xr() % 121)) << 52);
      double a; memcpy(&a, &bits, 8);
      double q0 = a * y, e = fma(-q0, b, a), q = fma(e, y, q0);
      if (q != a / b) { if (bad < 5) printf("FAIL b=%.17g a=%.17g\n", b, a); bad++; }
      n++;
    }
  }
  printf("checked %ld quotients over %d divisors: %ld mismatches\n", n, nb, bad);
  return bad != 0;
}
