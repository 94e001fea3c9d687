/* Exhaustive-ish check that the 3-op Markstein sequence
 *     q0 = u*r; e = fma(-q0, b, u); q = fma(e, r, q0)      r = RN(1/b)
 * returns RN(u/b) for the fill kernel's operands: u = m*2^-53 (m < 2^53
 * integer, the Philox uniform of vp/rng.py:68) and b = n_strat (integer).
 * Also checks the same for u = digit (small integers) and the 2-op
 * reconstruction of u from the 53-bit word, and the fill kernel's fused form
 * (devmath.cuh sample_axis): up = 1 + (bits 11..62 of w)*2^-52 assembled from
 * bits, a = up - (1 - bit63) = 2u exactly, RN(u/b) = Markstein(a, 2b, RN(1/b)/2).
 * Build: gcc -O2 -mfma. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s = 88172645463325252ull;
static inline uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static inline double mk(uint64_t m) {  /* 2-op exact m*2^-53 */
  uint64_t lo = m & ((1ull << 52) - 1), top = m >> 52;
  double t1; uint64_t b = 0x3FF0000000000000ull | lo; memcpy(&t1, &b, 8); t1 = t1 - 1.0;
  return fma(t1, 0.5, top ? 0.5 : 0.0);
}
int main(int argc, char **argv) {
  long bad = 0, n = 0, badu = 0;
  int per = argc > 1 ? atoi(argv[1]) : 200000;
  for (int b = 1; b <= 4100; b++) {
    double bd = b, r = 1.0 / bd;
    for (int i = 0; i < per + 64; i++) {
      uint64_t m;
      if (i < 64) { /* structured: small m, m near 2^52/2^53, multiples of b */
        uint64_t c[8] = {0, 1, 2, (uint64_t)b, (uint64_t)b * 3, (1ull << 52) - 1, (1ull << 52), (1ull << 53) - 1};
        m = c[i & 7] + (uint64_t)(i >> 3) * (uint64_t)b;
        if (m >= (1ull << 53)) m = (1ull << 53) - 1 - (i >> 3);
      } else m = xr() >> 11;
      double u = (double)m * 0x1p-53;
      if (mk(m) != u) badu++;
      { /* fused form from the 64-bit word w = m << 11 | junk, bit63 = top bit of m */
        uint64_t w = (m << 11) | (xr() & 0x7FF);
        uint64_t ub = 0x3FF0000000000000ull | ((w >> 11) & ((1ull << 52) - 1));
        double up; memcpy(&up, &ub, 8);
        double a = up - ((w >> 63) ? 0.0 : 1.0);
        double r2 = r * 0.5, b2 = 2.0 * bd;
        double p0 = a * r2, pe = fma(-p0, b2, a), pq = fma(pe, r2, p0);
        if (a != 2.0 * u || pq != u / bd) { if (bad < 10) printf("FAIL fused b=%d m=%llu\n", b, (unsigned long long)m); bad++; }
      }
      double q0 = u * r, e = fma(-q0, bd, u), q = fma(e, r, q0);
      if (q != u / bd) { if (bad < 10) printf("FAIL b=%d m=%llu\n", b, (unsigned long long)m); bad++; }
      n++;
    }
    for (int dgt = 0; dgt < b && dgt < 5000; dgt++) { /* digit/b for table entries */
      double u = dgt, q0 = u * r, e = fma(-q0, bd, u), q = fma(e, r, q0);
      if (q != u / bd) { bad++; }
    }
  }
  printf("checked %ld quotients: %ld mismatches; u reconstruction mismatches %ld\n", n, bad, badu);
  return bad != 0 || badu != 0;
}
