/*
 * vegas_oracle.c -- CPU restatement of the reference VEGAS+ hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity oracle and the CPU baseline
 * ("cpu_baseline.kind": "port").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * (paper_2408_09229_b200) never links or calls it.
 *
 * Parity status: PINNED.  Every function below is checked bit-for-bit (or to
 * the stated tolerance where the reference uses numpy SIMD transcendentals)
 * against golden vectors produced by the real reference package
 * (oracle/gen_golden.py -> tests/golden/*.npz; tests/test_oracle_golden.py).
 *
 * Reference = /root/reference/pkg/src/vegasplus (abbreviated vp/).  Each
 * function cites the lines it restates.  Compiled with -ffp-contract=off so
 * no FMA is formed (the numba kernels contain none).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VO_EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------- RNG -- */
/* Philox4x32-10 keyed counter permutation: vp/rng.py:24-60. */
static inline void philox_words(uint64_t block, uint64_t stream, uint64_t seed,
                                uint64_t *w0, uint64_t *w1) {
  uint32_t c0 = (uint32_t)block, c1 = (uint32_t)(block >> 32);
  uint32_t c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  *w0 = ((uint64_t)c0 << 32) | c1;
  *w1 = ((uint64_t)c2 << 32) | c3;
}

static const double INV_2_53 = 1.0 / 9007199254740992.0;

VO_EXPORT void vo_philox(uint64_t block, uint64_t stream, uint64_t seed, uint64_t out[2]) {
  philox_words(block, stream, seed, &out[0], &out[1]);
}

/* vp/rng.py:63-68 */
VO_EXPORT double vo_uniform_at(uint64_t seed, uint64_t stream, uint64_t pos) {
  uint64_t w0, w1;
  philox_words(pos >> 1, stream, seed, &w0, &w1);
  uint64_t w = (pos & 1) ? w1 : w0;
  return (double)(w >> 11) * INV_2_53;
}

/* ------------------------------------------------------------ sampling -- */
/* vp/kernels.py:36-88 (sample_runs): per run, walk the cube cursor, key the
 * randomness to g = run_base + run (slot = g % B, k = g / B), build y from the
 * mixed-radix cube digits (dim 0 least significant), clamp y < 1, and apply
 * the piecewise-linear map with its Jacobian. */
VO_EXPORT void vo_sample_runs(uint64_t seed, int64_t batch, int64_t run_base,
                              int64_t run_start, int64_t n, const int64_t *offsets,
                              int64_t cube_start, const double *edges, int dims, int ng,
                              int64_t n_strat, double *x, double *jac, int64_t *idx,
                              int64_t *cube) {
  const double ngf = (double)ng;
  const double nsf = (double)n_strat;
  const uint64_t stride = (uint64_t)(dims + (dims & 1));
  const double one_minus = nextafter(1.0, 0.0);
  int64_t c = cube_start;
  for (int64_t i = 0; i < n; i++) {
    int64_t run = run_start + i;
    while (offsets[c + 1] <= run) c++;
    cube[i] = c;
    int64_t g = run_base + run;
    uint64_t slot = (uint64_t)(g % batch);
    uint64_t k = (uint64_t)(g / batch);
    uint64_t base = k * stride;
    int64_t rem = c;
    double jf = 1.0;
    uint64_t w0 = 0, w1 = 0;
    for (int j = 0; j < dims; j++) {
      double u;
      if ((j & 1) == 0) {
        philox_words((base + (uint64_t)j) >> 1, slot, seed, &w0, &w1);
        u = (double)(w0 >> 11) * INV_2_53;
      } else {
        u = (double)(w1 >> 11) * INV_2_53;
      }
      int64_t digit = rem % n_strat;
      rem /= n_strat;
      double y = (double)digit / nsf + u / nsf;
      if (y >= 1.0) y = one_minus;
      double t = y * ngf;
      int64_t iv = (int64_t)t;
      if (iv > ng - 1) iv = ng - 1;
      double frac = t - (double)iv;
      const double *e = edges + (size_t)j * (ng + 1);
      double lo = e[iv];
      double dx = e[iv + 1] - lo;
      x[i * dims + j] = lo + frac * dx;
      jf *= ngf * dx;
      idx[i * dims + j] = iv;
    }
    jac[i] = jf;
  }
}

/* ----------------------------------------------------------- integrands -- */
/* Registry functions vp/integrands.py:106-190 and the BASELINE-pinned
 * synthetic ones (oracle/integrands_np.py).  params layout per id is fixed by
 * oracle/__init__.py (IntegrandOracle). */
enum {
  VO_GAUSSIAN = 0,   /* p = [mu, sigma, norm, inv_two_sigma2_denominator]  */
  VO_RIDGE = 1,      /* p = [n_centres, coef, window]                       */
  VO_MULTIPEAK = 2,  /* p = [n_peaks, sigma, norm, denom, weight, mu_k...]  */
  VO_GENZ_OSC = 3,   /* p = [phase, a_0..a_{d-1}]                           */
  VO_GENZ_PP = 4,    /* p = [a^-2_0.., u_0..]                               */
  VO_SINEXP = 5,
  VO_LINEAR = 6,
  VO_COSINE = 7,
  VO_EXPONENTIAL = 8,
  VO_ROOS_ARNOLD = 9,
  VO_MOROKOFF = 10,  /* p = [(1+1/d)^d, 1/d]                                */
  VO_CONSTANT = 11,  /* p = [c]                                             */
  VO_ASIAN = 12,     /* p = [s0, strike, drift, sigma sqrt(T), exp(-rT), clamp eps] */
  VO_PATH = 13,      /* p = [m/(2a), 0.5 a, amp, x_end]                     */
};

/* vp/integrands.py:59-100: Acklam's normal quantile (central + upper tail;
 * the callers only pass p >= 0.5) refined by one Newton step in erfc space. */
static const double AK_A[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                               -2.759285104469687e+02, 1.383577518672690e+02,
                               -3.066479806614716e+01, 2.506628277459239e+00};
static const double AK_B[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                               -1.556989798598866e+02, 6.680131188771972e+01,
                               -1.328068155288572e+01};
static const double AK_C[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                               -2.400758277161838e+00, -2.549732539343734e+00,
                               4.374664141464968e+00, 2.938163982698783e+00};
static const double AK_D[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                               2.445134137142996e+00, 3.754408661907416e+00};
static double ndtri_approx(double p) {
  if (p < 0.02425) {
    double q = sqrt(-2.0 * log(p));
    return (((((AK_C[0] * q + AK_C[1]) * q + AK_C[2]) * q + AK_C[3]) * q + AK_C[4]) * q + AK_C[5]) /
           ((((AK_D[0] * q + AK_D[1]) * q + AK_D[2]) * q + AK_D[3]) * q + 1.0);
  }
  if (p > 1.0 - 0.02425) {
    double q = sqrt(-2.0 * log(1.0 - p));
    return -(((((AK_C[0] * q + AK_C[1]) * q + AK_C[2]) * q + AK_C[3]) * q + AK_C[4]) * q + AK_C[5]) /
           ((((AK_D[0] * q + AK_D[1]) * q + AK_D[2]) * q + AK_D[3]) * q + 1.0);
  }
  double q = p - 0.5, r = q * q;
  return (((((AK_A[0] * r + AK_A[1]) * r + AK_A[2]) * r + AK_A[3]) * r + AK_A[4]) * r + AK_A[5]) * q /
         (((((AK_B[0] * r + AK_B[1]) * r + AK_B[2]) * r + AK_B[3]) * r + AK_B[4]) * r + 1.0);
}
static double vo_erfinv(double y) {   /* vp/integrands.py:83-100 */
  double ya = fabs(y);
  double z = ndtri_approx((ya + 1.0) * 0.5) * (1.0 / sqrt(2.0));
  z += (erfc(z) - (1.0 - ya)) * (sqrt(M_PI) / 2.0) * exp(z * z);
  return copysign(z, y);
}

static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x > y) - (x < y);
}

double vo_pairwise_sum(const double *a, int64_t n);

/* numpy row reductions `.sum(axis=1)` run the pairwise kernel per row (the
 * 8-accumulator path for 8 <= d <= 128); products reduce sequentially. */
static double eval_one(int id, const double *p, const double *x, int d) {
  double t[66];
  switch (id) {
    case VO_GAUSSIAN: { /* vp/integrands.py:135-139 */
      for (int j = 0; j < d; j++) { double u = x[j] - p[0]; t[j] = u * u; }
      double r2 = vo_pairwise_sum(t, d);
      return p[2] * exp(-r2 / p[3]);
    }
    case VO_RIDGE: { /* vp/integrands.py:154-182: sorted-coordinate sums */
      double xs[64];
      for (int j = 0; j < d; j++) xs[j] = x[j];
      qsort(xs, (size_t)d, sizeof(double), cmp_double);
      double s1 = vo_pairwise_sum(xs, d);
      for (int j = 0; j < d; j++) t[j] = xs[j] * xs[j];
      double s2 = vo_pairwise_sum(t, d);
      int n_cent = (int)p[0];
      double spacing = n_cent - 1.0;
      double mu = 0.25 * s1;
      double q0 = s2 - mu * s1;
      int lo = (int)ceil((mu - p[2]) * spacing);
      int hi = (int)floor((mu + p[2]) * spacing);
      if (lo < 0) lo = 0;
      if (hi > n_cent - 1) hi = n_cent - 1;
      double acc = 0.0;
      for (int i = lo; i <= hi; i++) {
        double dc = i / spacing - mu;
        acc += exp(-400.0 * dc * dc);
      }
      return p[1] * exp(-100.0 * q0) * acc;
    }
    case VO_MULTIPEAK: { /* oracle/integrands_np.py multipeak8 */
      int np_ = (int)p[0];
      double out = 0.0;
      for (int k = 0; k < np_; k++) {
        for (int j = 0; j < d; j++) { double u = x[j] - p[5 + k]; t[j] = u * u; }
        double r2 = vo_pairwise_sum(t, d);
        out += p[2] * exp(-r2 / p[3]);
      }
      return out / p[4];
    }
    case VO_GENZ_OSC: { /* cos(2 pi u1 + a.x) */
      double s = 0.0;
      for (int j = 0; j < d; j++) s += x[j] * p[1 + j];
      return cos(p[0] + s);
    }
    case VO_GENZ_PP: { /* prod 1/(a^-2 + (x-u)^2) */
      double prod = 1.0;
      for (int j = 0; j < d; j++) {
        double u = x[j] - p[d + j];
        prod *= 1.0 / (p[j] + u * u);
      }
      return prod;
    }
    case VO_SINEXP: return sin(x[0]) + exp(x[1]);
    case VO_LINEAR: return vo_pairwise_sum(x, d);
    case VO_COSINE: { double s = 1.0; for (int j = 0; j < d; j++) s *= cos(x[j]); return s; }
    case VO_EXPONENTIAL: {
      for (int j = 0; j < d; j++) t[j] = x[j] * x[j];
      return exp(vo_pairwise_sum(t, d));
    }
    case VO_ROOS_ARNOLD: {
      double s = 1.0; for (int j = 0; j < d; j++) s *= fabs(4.0 * x[j] - 2.0); return s;
    }
    case VO_MOROKOFF: {
      double s = 1.0; for (int j = 0; j < d; j++) s *= pow(x[j], p[1]); return p[0] * s;
    }
    case VO_CONSTANT: return p[0];
    case VO_ASIAN: { /* vp/integrands.py:196-210 asian_option_batch */
      for (int j = 0; j < d; j++) {
        double xc = x[j] < p[5] ? p[5] : (x[j] > 1.0 - p[5] ? 1.0 - p[5] : x[j]);
        t[j] = vo_erfinv(2.0 * xc - 1.0);
      }
      double z = vo_pairwise_sum(t, d) * sqrt(2.0);
      double s_avg = p[0] * exp(p[2] + p[3] * z);
      double pay = s_avg - p[1];
      return p[4] * (pay > 0.0 ? pay : 0.0);
    }
    case VO_PATH: { /* vp/integrands.py:233-251 path_integral_batch, d = n_slices - 1 */
      double full[66], kin[65];
      full[0] = p[3];
      full[d + 1] = p[3];
      for (int j = 0; j < d; j++) full[j + 1] = x[j];
      for (int j = 0; j <= d; j++) { double u = full[j + 1] - full[j]; kin[j] = u * u; }
      for (int j = 0; j <= d; j++) t[j] = full[j] * full[j];
      double kinetic = p[0] * vo_pairwise_sum(kin, d + 1);
      double potential = p[1] * vo_pairwise_sum(t, d + 1);
      return p[2] * exp(-(kinetic + potential));
    }
  }
  return NAN;
}

VO_EXPORT void vo_eval(int id, const double *params, const double *x, int64_t n, int d,
                       double *out) {
  for (int64_t i = 0; i < n; i++) out[i] = eval_one(id, params, x + i * d, d);
}

/* ------------------------------------------------------------- fill ----- */
#define VO_CHUNK 65536 /* vp/kernels.py:22 (chunking never changes results) */

typedef struct {
  /* inputs */
  const int64_t *offsets; int64_t n_cubes;
  const double *edges; int dims; int ng; int64_t n_strat;
  uint64_t seed; int64_t batch; int64_t run_base;
  int id; const double *params;
  int64_t start, stop;
  /* private outputs */
  double *map_w; int64_t *map_counts; double *s1; double *s2; int64_t *counts;
  /* error */
  int64_t err_run; double err_value; double err_point[64];
} shard_t;

static int64_t run_to_cube(const int64_t *offsets, int64_t n_cubes, int64_t r) {
  /* vp/strat.py:140-144: searchsorted(offsets, r, 'right') - 1 */
  int64_t lo = 0, hi = n_cubes + 1;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (offsets[mid] <= r) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

/* vp/executor.py:86-130 (fill_shard) + vp/kernels.py:91-109 (accumulate) */
static void *fill_shard(void *arg) {
  shard_t *s = (shard_t *)arg;
  s->err_run = -1;
  if (s->stop <= s->start) return NULL;
  int d = s->dims;
  int64_t cap = s->stop - s->start < VO_CHUNK ? s->stop - s->start : VO_CHUNK;
  double *x = malloc(sizeof(double) * cap * d);
  double *jac = malloc(sizeof(double) * cap);
  int64_t *idx = malloc(sizeof(int64_t) * cap * d);
  int64_t *cube = malloc(sizeof(int64_t) * cap);
  double *vals = malloc(sizeof(double) * cap);
  int64_t cursor = run_to_cube(s->offsets, s->n_cubes, s->start);
  for (int64_t c0 = s->start; c0 < s->stop; c0 += VO_CHUNK) {
    int64_t n = s->stop - c0 < VO_CHUNK ? s->stop - c0 : VO_CHUNK;
    vo_sample_runs(s->seed, s->batch, s->run_base, c0, n, s->offsets, cursor, s->edges, d,
                   s->ng, s->n_strat, x, jac, idx, cube);
    cursor = cube[n - 1];
    vo_eval(s->id, s->params, x, n, d, vals);
    for (int64_t i = 0; i < n; i++) {
      if (!isfinite(vals[i])) {
        s->err_run = c0 + i;
        s->err_value = vals[i];
        for (int j = 0; j < d && j < 64; j++) s->err_point[j] = x[i * d + j];
        goto done;
      }
    }
    for (int64_t i = 0; i < n; i++) {
      double v = jac[i] * vals[i];
      double w2 = v * v;
      for (int j = 0; j < d; j++) {
        int64_t iv = idx[i * d + j];
        s->map_w[(size_t)j * s->ng + iv] += w2;
        s->map_counts[(size_t)j * s->ng + iv] += 1;
      }
      int64_t h = cube[i];
      s->s1[h] += v;
      s->s2[h] += w2;
      s->counts[h] += 1;
    }
  }
done:
  free(x); free(jac); free(idx); free(cube); free(vals);
  return NULL;
}

/* vp/executor.py:41-57 (partition_runs) */
VO_EXPORT void vo_partition_runs(int64_t total, int64_t k, int64_t *starts, int64_t *stops) {
  int64_t q = total / k, rem = total % k, start = 0;
  for (int64_t i = 0; i < k; i++) {
    int64_t size = q + (i < rem ? 1 : 0);
    starts[i] = start;
    stops[i] = start + size;
    start += size;
  }
}

static void shard_iadd(shard_t *a, const shard_t *b) {
  size_t nm = (size_t)a->dims * a->ng;
  for (size_t i = 0; i < nm; i++) { a->map_w[i] += b->map_w[i]; a->map_counts[i] += b->map_counts[i]; }
  for (int64_t h = 0; h < a->n_cubes; h++) {
    a->s1[h] += b->s1[h]; a->s2[h] += b->s2[h]; a->counts[h] += b->counts[h];
  }
}

/* vp/executor.py:133-166 (parallel_fill) with vp/executor.py:60-83 (tree_reduce).
 * Fills runs [run_lo, run_hi) of the plan (the whole plan for one process;
 * a shard of it when the caller distributes ranks).  Outputs are overwritten.
 * Returns 0, or 1 with *err_run / err_point / *err_value set to the lowest
 * failing worker's first non-finite evaluation. */
VO_EXPORT int vo_fill(const int64_t *offsets, int64_t n_cubes, const double *edges, int dims,
                      int ng, int64_t n_strat, uint64_t seed, int64_t batch, int64_t run_base,
                      int id, const double *params, int workers, int64_t run_lo, int64_t run_hi,
                      double *map_w, int64_t *map_counts, double *s1, double *s2,
                      int64_t *counts, int64_t *err_run, double *err_point, double *err_value) {
  if (workers < 1) workers = 1;
  shard_t *sh = calloc((size_t)workers, sizeof(shard_t));
  int64_t *st = malloc(sizeof(int64_t) * workers), *sp = malloc(sizeof(int64_t) * workers);
  vo_partition_runs(run_hi - run_lo, workers, st, sp);
  size_t nm = (size_t)dims * ng;
  for (int w = 0; w < workers; w++) {
    shard_t *s = &sh[w];
    s->offsets = offsets; s->n_cubes = n_cubes; s->edges = edges; s->dims = dims; s->ng = ng;
    s->n_strat = n_strat; s->seed = seed; s->batch = batch; s->run_base = run_base;
    s->id = id; s->params = params;
    s->start = run_lo + st[w]; s->stop = run_lo + sp[w];
    if (w == 0) {
      s->map_w = map_w; s->map_counts = map_counts; s->s1 = s1; s->s2 = s2; s->counts = counts;
      memset(map_w, 0, sizeof(double) * nm); memset(map_counts, 0, sizeof(int64_t) * nm);
      memset(s1, 0, sizeof(double) * n_cubes); memset(s2, 0, sizeof(double) * n_cubes);
      memset(counts, 0, sizeof(int64_t) * n_cubes);
    } else {
      s->map_w = calloc(nm, sizeof(double)); s->map_counts = calloc(nm, sizeof(int64_t));
      s->s1 = calloc((size_t)n_cubes, sizeof(double)); s->s2 = calloc((size_t)n_cubes, sizeof(double));
      s->counts = calloc((size_t)n_cubes, sizeof(int64_t));
    }
  }
  if (workers == 1) {
    fill_shard(&sh[0]);
  } else {
    pthread_t *th = malloc(sizeof(pthread_t) * workers);
    for (int w = 0; w < workers; w++) pthread_create(&th[w], NULL, fill_shard, &sh[w]);
    for (int w = 0; w < workers; w++) pthread_join(th[w], NULL);
    free(th);
  }
  int rc = 0;
  for (int w = 0; w < workers; w++) {
    if (sh[w].err_run >= 0) {
      rc = 1;
      *err_run = sh[w].err_run;
      *err_value = sh[w].err_value;
      for (int j = 0; j < dims && j < 64; j++) err_point[j] = sh[w].err_point[j];
      break;
    }
  }
  if (!rc) {
    /* tree_reduce: adjacent pairs, left to right, ceil(log2 W) levels */
    int n = workers;
    int *live = malloc(sizeof(int) * workers);
    for (int w = 0; w < workers; w++) live[w] = w;
    while (n > 1) {
      int m = 0;
      for (int i = 0; i < n; i += 2) {
        if (i + 1 < n) shard_iadd(&sh[live[i]], &sh[live[i + 1]]);
        live[m++] = live[i];
      }
      n = m;
    }
    free(live);
  }
  for (int w = 1; w < workers; w++) {
    free(sh[w].map_w); free(sh[w].map_counts); free(sh[w].s1); free(sh[w].s2); free(sh[w].counts);
  }
  free(sh); free(st); free(sp);
  return rc;
}

/* ----------------------------------------------------- numpy pairwise -- */
/* numpy's float64 add.reduce over a contiguous 1-D array (numpy 2.3,
 * loops_utils pairwise_sum).  Call sites: vp/strat.py:106,
 * 205-206; vp/maps.py:183, 220. */
VO_EXPORT double vo_pairwise_sum(const double *a, int64_t n) {
  /* (defined here; forward-declared above the integrands) */
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return vo_pairwise_sum(a, n2) + vo_pairwise_sum(a + n2, n - n2);
  }
}

/* numpy's `array ** scalar` fast paths (1 -> copy, 2 -> square, 0.5 -> sqrt),
 * else libm pow (numpy itself uses its SIMD pow: ulp-level host dependence,
 * SURVEY.md §7 hard part 1). */
static inline double np_scalar_pow(double x, double e) {
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == 0.5) return sqrt(x);
  if (e == 0.0) return 1.0;
  return pow(x, e);
}

/* --------------------------------------------------------- allocation -- */
/* vp/strat.py:88-113 (update_evals_per_cube).  dp (optional) receives
 * d_h**beta so tests can substitute a different pow. */
VO_EXPORT void vo_update_evals(const double *d_h, int64_t n, double beta, int64_t n_eval,
                               const double *dp_in, int64_t *n_h) {
  const double ne = (double)n_eval;
  if (beta == 0.0) {
    double p = 1.0 / (double)n;
    int64_t v = (int64_t)ceil(ne * p);
    if (v < 2) v = 2;
    for (int64_t i = 0; i < n; i++) n_h[i] = v;
    return;
  }
  double *dp = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; i++) dp[i] = dp_in ? dp_in[i] : np_scalar_pow(d_h[i], beta);
  double total = vo_pairwise_sum(dp, n);
  if (total > 0.0) {
    for (int64_t i = 0; i < n; i++) {
      int64_t v = (int64_t)ceil(ne * (dp[i] / total));
      n_h[i] = v < 2 ? 2 : v;
    }
  } else {
    double p = 1.0 / (double)n;
    int64_t v = (int64_t)ceil(ne * p);
    if (v < 2) v = 2;
    for (int64_t i = 0; i < n; i++) n_h[i] = v;
  }
  free(dp);
}

/* vp/strat.py:131-137 (build_run_plan): exclusive int64 prefix sum */
VO_EXPORT void vo_build_plan(const int64_t *n_h, int64_t n, int64_t *offsets) {
  offsets[0] = 0;
  for (int64_t i = 0; i < n; i++) offsets[i + 1] = offsets[i] + n_h[i];
}

/* vp/strat.py:183-208 (compute_results).  Returns -1 (and *bad = first cube
 * with the minimal count) when a cube has < 2 samples. */
VO_EXPORT int vo_compute_results(const double *s1, const double *s2, const int64_t *counts,
                                 int64_t n, double *i_it, double *var_it, double *d_h,
                                 int64_t *bad) {
  int64_t amin = 0;
  for (int64_t h = 0; h < n; h++) if (counts[h] < counts[amin]) amin = h;
  if (counts[amin] < 2) { *bad = amin; return -1; }
  double V = 1.0 / (double)n;
  double *means = malloc(sizeof(double) * n), *rv = malloc(sizeof(double) * n);
  for (int64_t h = 0; h < n; h++) {
    double c = (double)counts[h];
    double m = s1[h] / c;
    double r = s2[h] / c - m * m;
    if (!(r >= 0.0)) r = (r != r) ? r : 0.0; /* np.maximum propagates NaN */
    means[h] = m;
    rv[h] = r;
    d_h[h] = sqrt(r) * V;
  }
  *i_it = vo_pairwise_sum(means, n) / (double)n;
  for (int64_t h = 0; h < n; h++) rv[h] = rv[h] / (double)counts[h];
  *var_it = vo_pairwise_sum(rv, n) * V * V;
  free(means); free(rv);
  return 0;
}

/* ------------------------------------------------------------- refine -- */
/* vp/maps.py:160-199 (smooth_and_damp + _damp) */
VO_EXPORT void vo_smooth_and_damp(const double *w, const int64_t *counts, int dims, int ng,
                                  double alpha, double *out) {
  double *d = malloc(sizeof(double) * ng), *sm = malloc(sizeof(double) * ng);
  for (int j = 0; j < dims; j++) {
    const double *wj = w + (size_t)j * ng;
    const int64_t *cj = counts + (size_t)j * ng;
    double *oj = out + (size_t)j * ng;
    int any = 0;
    for (int i = 0; i < ng; i++) {
      d[i] = cj[i] > 0 ? wj[i] / (double)cj[i] : 0.0;
      any |= d[i] != 0.0;
      oj[i] = 0.0;
    }
    if (!any) continue;
    sm[0] = (7.0 * d[0] + d[1]) / 8.0;
    sm[ng - 1] = (d[ng - 2] + 7.0 * d[ng - 1]) / 8.0;
    for (int i = 1; i < ng - 1; i++) sm[i] = (d[i - 1] + 6.0 * d[i] + d[i + 1]) / 8.0;
    double total = vo_pairwise_sum(sm, ng);
    if (total <= 0.0) continue;
    for (int i = 0; i < ng; i++) sm[i] /= total;
    for (int i = 0; i < ng; i++) {
      double v = sm[i];
      if (fabs(v - 1.0) < 1e-15) oj[i] = 1.0;
      else if (v >= 1e-30) oj[i] = np_scalar_pow((v - 1.0) / log(v), alpha);
      else oj[i] = 0.0;
    }
  }
  free(d); free(sm);
}

/* vp/maps.py:202-234 (update_grid).  Returns j >= 0 when dimension j lost
 * strict monotonicity (the reference raises AssertionError), else -1. */
VO_EXPORT int vo_update_grid(const double *edges, const double *damped, int dims, int ng,
                             double *out) {
  double *cum = malloc(sizeof(double) * (ng + 1));
  int bad = -1;
  memcpy(out, edges, sizeof(double) * (size_t)dims * (ng + 1));
  for (int j = 0; j < dims; j++) {
    const double *w = damped + (size_t)j * ng;
    const double *e = edges + (size_t)j * (ng + 1);
    double *o = out + (size_t)j * (ng + 1);
    double total = vo_pairwise_sum(w, ng);
    if (total <= 0.0) continue;
    cum[0] = 0.0;
    for (int i = 0; i < ng; i++) cum[i + 1] = cum[i] + w[i];
    double delta = total / ng;
    int iv = 0;
    for (int i = 1; i < ng; i++) {
      double goal = (double)i * delta;
      /* searchsorted(cum[1:], goal, 'left'): first iv with cum[iv+1] >= goal;
       * goals increase, so the search resumes from the previous iv */
      while (iv < ng - 1 && cum[iv + 1] < goal) iv++;
      double frac = (goal - cum[iv]) / w[iv];
      o[i] = e[iv] + frac * (e[iv + 1] - e[iv]);
    }
    for (int i = 0; i < ng; i++)
      if (!(o[i + 1] > o[i])) { if (bad < 0) bad = j; break; }
  }
  free(cum);
  return bad;
}
