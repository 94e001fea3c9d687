/*
 * vegas_b200.h -- C ABI of the B200-native VEGAS+ iteration hot path.
 *
 * Plain C: pointers, sizes and status codes only (no torch / CUDA types in
 * the signatures; streams are passed as void*).  The library is
 * paper_2408_09229_b200/_lib/libvegas_b200.so (built for sm_100a).
 *
 * Reference = /root/reference/pkg/src/vegasplus ("vp/").  Each entry point
 * names the reference interface it replaces.  The reference's only seam on
 * this path is Python: the per-iteration body of core.integrate
 * (vp/core.py:200-219) calling strat.build_run_plan (vp/strat.py:131-137),
 * executor.parallel_fill (vp/executor.py:133-166), strat.compute_results
 * (vp/strat.py:183-208), strat.update_evals_per_cube (vp/strat.py:88-113),
 * maps.smooth_and_damp (vp/maps.py:160-199) and maps.update_grid
 * (vp/maps.py:202-234).  INTEGRATION.md shows the ctypes binding.
 *
 * Conventions
 *  - Status: every function returns VPB_OK (0) or a VPB_ERR_* code; the
 *    message is in vpb_last_error() (thread-local).
 *  - Ownership: a context owns all of its device buffers; host pointers
 *    passed in are borrowed for the duration of the call only.
 *  - Threading: one context per host thread at a time; independent contexts
 *    may run concurrently (vp/core.py integrate() is reentrant).
 *  - Layouts (all C-contiguous, host or device as named):
 *      edges      f64[dims][n_intervals+1]          (VegasMap.edges)
 *      map_w      f64[dims][n_intervals]            (MapWeights.w)
 *      map_counts i64[dims][n_intervals]            (MapWeights.counts)
 *      s1, s2     f64[n_cubes]; counts i64[n_cubes] (CubeAccumulator)
 *      n_h        i64[n_cubes]; offsets i64[n_cubes+1] (RunPlan.offsets)
 */
#ifndef VEGAS_B200_H
#define VEGAS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPB_ABI_VERSION 3

/* status codes */
#define VPB_OK 0
#define VPB_ERR_CUDA 1          /* CUDA runtime failure                         */
#define VPB_ERR_INVALID 2       /* ContractViolationError (vp/errors.py:14-15)   */
#define VPB_ERR_NONFINITE 3     /* NonFiniteIntegrandError (vp/errors.py:18-32)  */
#define VPB_ERR_ASSERT 4        /* AssertionError (vp/strat.py:196, maps.py:232) */
#define VPB_ERR_NCCL 5          /* NCCL failure                                  */
#define VPB_ERR_UNSUPPORTED 6   /* integrand / dimension not compiled in         */

/* device integrand functors (registry names of vp/integrands.py:399-410 plus
 * the BASELINE-pinned synthetic integrands).  Parameter blobs: see
 * paper_2408_09229_b200/integrands.py. */
#define VPB_GAUSSIAN 0          /* [mu, sigma, norm, 2 sigma^2, RN(1/(2 sigma^2))] */
#define VPB_RIDGE 1             /* [n_centres, coef, window]                     */
#define VPB_MULTIPEAK 2         /* [n_peaks, sigma, norm, 2s^2, divisor, RN(1/2s^2), RN(1/divisor), mu_k...] */
#define VPB_GENZ_OSCILLATORY 3  /* [2 pi u_1, a_0 .. a_{d-1}]                    */
#define VPB_GENZ_PRODUCTPEAK 4  /* [a_0^-2 .. a_{d-1}^-2, u_0 .. u_{d-1}]        */
#define VPB_SINEXP 5
#define VPB_LINEAR 6
#define VPB_COSINE 7
#define VPB_EXPONENTIAL 8
#define VPB_ROOS_ARNOLD 9
#define VPB_MOROKOFF 10         /* [(1+1/d)^d, 1/d]                              */
#define VPB_CONSTANT 11         /* [c]                                           */
#define VPB_ASIAN_OPTION 12     /* [s0, strike, drift, sigma sqrt(T), exp(-rT), clamp eps] */
#define VPB_PATH_INTEGRAL 13    /* [m/(2a), a/2, amp, x_end]  (dims = n_slices - 1) */
#define VPB_N_INTEGRANDS 14

#define VPB_MAX_PARAMS 64
#define VPB_MAX_DIMS 64

typedef struct vpb_ctx vpb_ctx;

/* One integration run's fixed geometry and knobs: the fields of
 * IntegratorConfig (vp/core.py:29-62) that reach the hot path, plus the
 * device integrand and the domain (maps.new_uniform bounds, vp/maps.py:70). */
typedef struct vpb_desc {
  int32_t dims;
  int32_t n_intervals;        /* IntegratorConfig.n_intervals              */
  int64_t n_strat;            /* StratGrid.n_strat (vp/strat.py:49-71)     */
  int64_t n_eval;             /* IntegratorConfig.n_eval                   */
  int64_t batch_size;         /* IntegratorConfig.batch_size (RNG slots)   */
  uint64_t seed;              /* IntegratorConfig.seed                     */
  double alpha;               /* IntegratorConfig.alpha                    */
  double beta;                /* IntegratorConfig.beta                     */
  int32_t integrand;          /* VPB_* id                                  */
  int32_t n_params;
  const double *params;       /* host, n_params                            */
  const double *bounds;       /* host, 2*dims: lo_0, hi_0, lo_1, hi_1, ... */
  int32_t device;             /* CUDA ordinal; -1 = current device         */
  int32_t max_it;             /* capacity of the per-iteration history     */
  void *stream;               /* cudaStream_t to run on; NULL = own stream */
  int32_t flags;              /* VPB_FLAG_*                                */
} vpb_desc;

/* Deterministic mode: bitwise-repeatable map weights (the reference's
 * repeat criterion, tests/test_acceptance.py:153-190).  The fill runs twice
 * per iteration with the generic kernel: pass 1's f64 interval sums pick a
 * per-interval scale 2^k, pass 2 sums round(w2 2^k) with 64-bit integer
 * atomics -- exact, so neither the update order nor the sharding changes a
 * bit (the int64 sums are all-reduced exactly).  About 2-3x the fill time. */
#define VPB_FLAG_DETERMINISTIC 1

/* ---- library ------------------------------------------------------------ */
int vpb_abi_version(void);
const char *vpb_last_error(void);
/* 1 if the integrand id is compiled for this dimension with the fast
 * (compile-time dims) fill kernel, 0 if it runs the generic kernel. */
int vpb_is_specialised(int32_t integrand, int32_t dims);
/* Number of CUDA devices visible to this process (CUDA_VISIBLE_DEVICES
 * applies); 0 and VPB_OK when there is none.  The host maps LOCAL_RANK onto
 * an ordinal with it (LOCAL_RANK mod count). */
int vpb_device_count(int32_t *n);

/* ---- context: the state of one integrate() call (vp/core.py:168-238) ------ */
int vpb_create(const vpb_desc *desc, vpb_ctx **out);
int vpb_destroy(vpb_ctx *ctx);

/* Multi-GPU: ranks shard each iteration's run range with the reference's
 * partition rule (vp/executor.py:41-57) and merge accumulators with one NCCL
 * all-reduce (replaces tree_reduce, vp/executor.py:60-83).  Rank 0 creates
 * the id; the host broadcasts it (128 bytes). */
int vpb_nccl_unique_id(char id_out[128]);
int vpb_attach_nccl(vpb_ctx *ctx, const char id[128], int32_t world, int32_t rank);
/* Shard without NCCL (the host merges accumulators itself). */
int vpb_set_shard(vpb_ctx *ctx, int32_t world, int32_t rank);
/* Multi-rank without NCCL: the per-iteration exchange (the same three
 * reductions the NCCL path makes: map_w|s1|s2 f64 SUM, map_counts i64 SUM,
 * the 3-word control word i64 MAX -- failure flags and the first failing
 * run, so every rank raises the same error) goes through a host all-reduce
 * callback, e.g. torch.distributed over gloo.  Iterations then synchronise
 * at the exchange and are not graph-captured.  fn returns 0 on success. */
#define VPB_DT_F64 0
#define VPB_DT_I64 1
#define VPB_OP_SUM 0
#define VPB_OP_MAX 1
typedef int (*vpb_allreduce_fn)(void *user, void *buf, int64_t count, int32_t dtype, int32_t op);
int vpb_attach_exchange(vpb_ctx *ctx, int32_t world, int32_t rank, vpb_allreduce_fn fn,
                        void *user);

/* init phase (vp/core.py:188-196): uniform map (maps.new_uniform), uniform
 * allocation (strat.initial_grid), run_base = 0, history cleared. */
int vpb_reset(vpb_ctx *ctx);

/* Run n_it full iterations asynchronously on the context's stream:
 * plan -> fill -> [all-reduce] -> results -> allocation -> refine
 * (vp/core.py:200-219).  No host synchronisation. */
int vpb_iterate(vpb_ctx *ctx, int32_t n_it);

/* Synchronise and read the history: per-iteration estimate, variance and
 * evaluation count (plan.total).  Returns VPB_ERR_NONFINITE / VPB_ERR_ASSERT
 * if an iteration failed (history stops before it). */
int vpb_history(vpb_ctx *ctx, int32_t cap, double *estimates, double *variances,
                int64_t *evals, int32_t *n_out);
/* Details of a VPB_ERR_NONFINITE: run index within its iteration's plan,
 * the domain point (dims doubles) and the value (NonFiniteIntegrandError). */
int vpb_error_info(vpb_ctx *ctx, int64_t *run_index, double *point, double *value);
/* Device time per phase (ms, summed over iterations since reset):
 * map (allocation + plan), fill (incl. all-reduce), update (results+refine). */
int vpb_phase_times(vpb_ctx *ctx, double *map_ms, double *fill_ms, double *update_ms);
/* Device time (ms) of the last fill kernel and the number of fill launches. */
int vpb_last_fill_ms(vpb_ctx *ctx, double *ms);
int vpb_sync(vpb_ctx *ctx);
/* Device time summed over iterations [first, first+count) of this reset:
 * whole iterations and the fused fill kernel alone (CUDA events on the
 * context's stream). */
int vpb_timing(vpb_ctx *ctx, int32_t first, int32_t count, double *iter_ms,
               double *fill_kernel_ms);
/* The context's fill layout: 0 edge rows + shared histograms, 1 pair table +
 * shared histograms, 2 records (chunked fill + hist_records groups), 3
 * generic runtime-dims kernel; record chunks per iteration (0 if none); and
 * the number of this library's kernel launches per iteration. */
int vpb_fill_layout(vpb_ctx *ctx, int32_t *layout, int32_t *n_chunks,
                    int32_t *launches_per_iteration);
/* Fixed-point interval histograms (FX mode; no reference counterpart -- an
 * implementation choice behind vp/kernels.py:100-105's MapWeights sums):
 * out = [enabled for this context, iterations filled in fixed point,
 * iterations whose fixed-point sums failed the precision / wrap-around proof
 * and were refilled in f64, values summed in f64 because they exceeded the
 * fixed-point range].  Synchronises the context's stream. */
int vpb_fx_stats(vpb_ctx *ctx, int64_t out[4]);
/* Measured FP64 pipe throughput (DFMA chains on every SM; one FMA = 1 op):
 * the roofline denominator for the FP64-issue-bound fill. */
int vpb_fp64_peak(int32_t device, double *ops_per_s);

/* State access (host buffers; synchronous). */
int vpb_set_edges(vpb_ctx *ctx, const double *edges);
int vpb_get_edges(vpb_ctx *ctx, double *edges);
int vpb_set_allocation(vpb_ctx *ctx, const int64_t *n_h);
int vpb_get_plan(vpb_ctx *ctx, int64_t *n_h, int64_t *offsets);
int vpb_get_spread(vpb_ctx *ctx, double *d_h);
int vpb_get_fill(vpb_ctx *ctx, double *map_w, int64_t *map_counts, double *s1, double *s2,
                 int64_t *counts);
int vpb_get_run_base(vpb_ctx *ctx, int64_t *run_base);
int vpb_set_run_base(vpb_ctx *ctx, int64_t run_base);

/* One iteration end to end through host buffers (the e2e measurement path):
 * H2D of the map, the iteration on device, D2H of estimate/variance/evals
 * and the refined map. */
int vpb_iteration_host(vpb_ctx *ctx, const double *edges_in, double *edges_out,
                       double *estimate, double *variance, int64_t *evals);

/* Fill only (executor.parallel_fill, vp/executor.py:133-166) for the current
 * plan at the given run_base; accumulators stay on device (vpb_get_fill). */
int vpb_fill(vpb_ctx *ctx, int64_t run_base);

/* ---- stateless parity entry points (host buffers, current device) --------- */
/* rng._philox_words (vp/rng.py:38-60): out[2i], out[2i+1] = w0, w1 */
int vpb_philox_host(const uint64_t *block, const uint64_t *stream, const uint64_t *seed,
                    int64_t n, uint64_t *out);
/* rng.uniform_at (vp/rng.py:63-68) */
int vpb_uniform_at_host(const uint64_t *seed, const uint64_t *stream, const uint64_t *pos,
                        int64_t n, double *out);
/* kernels.sample_runs (vp/kernels.py:36-88) for runs [run_start, run_start+n) */
int vpb_sample_runs_host(uint64_t seed, int64_t batch, int64_t run_base, int64_t run_start,
                         int64_t n, const int64_t *offsets, int64_t n_cubes, const double *edges,
                         int32_t dims, int32_t ng, int64_t n_strat, double *x, double *jac,
                         int64_t *idx, int64_t *cube);
/* IntegrandSpec.evaluate_batch on device functors */
int vpb_eval_host(int32_t integrand, const double *params, int32_t n_params, const double *x,
                  int64_t n, int32_t dims, double *out);
/* executor.parallel_fill over runs [run_lo, run_hi) of the plan */
int vpb_fill_host(const int64_t *offsets, int64_t n_cubes, const double *edges, int32_t dims,
                  int32_t ng, int64_t n_strat, uint64_t seed, int64_t batch, int64_t run_base,
                  int32_t integrand, const double *params, int32_t n_params, int64_t run_lo,
                  int64_t run_hi, double *map_w, int64_t *map_counts, double *s1, double *s2,
                  int64_t *counts, int64_t *err_run, double *err_point, double *err_value);
/* numpy float64 add.reduce (pairwise) */
int vpb_pairwise_sum_host(const double *a, int64_t n, double *out);
/* the allocation's d_h**beta on the device, as the fill's update computes it:
 * numpy's scalar-exponent fast paths (beta 0, 1/2, 1, 2) bit-exact, else
 * CUDA pow (<= 2 ulp; numpy's pow is host-dependent) */
int vpb_pow_host(const double *x, int64_t n, double y, double *out);
/* strat.update_evals_per_cube (vp/strat.py:88-113) */
int vpb_update_evals_host(const double *d_h, int64_t n, double beta, int64_t n_eval,
                          int64_t *n_h);
/* strat.build_run_plan (vp/strat.py:131-137) */
int vpb_build_plan_host(const int64_t *n_h, int64_t n, int64_t *offsets);
/* strat.compute_results (vp/strat.py:183-208); VPB_ERR_ASSERT if a count < 2 */
int vpb_compute_results_host(const double *s1, const double *s2, const int64_t *counts,
                             int64_t n, double *estimate, double *variance, double *d_h);
/* maps.smooth_and_damp (vp/maps.py:160-199) */
int vpb_smooth_and_damp_host(const double *map_w, const int64_t *map_counts, int32_t dims,
                             int32_t ng, double alpha, double *out);
/* maps.update_grid (vp/maps.py:202-234); VPB_ERR_ASSERT on lost monotonicity */
int vpb_update_grid_host(const double *edges, const double *damped, int32_t dims, int32_t ng,
                         double *out);

#ifdef __cplusplus
}
#endif
#endif /* VEGAS_B200_H */
