"""Host-side mirrors of the reference's hot-path functions, run on the GPU.

Each function has the reference's name, argument meaning and error behaviour
and calls the C ABI (include/vegas_b200.h); none has a CPU code path.

    uniform_at, philox_words      vp/rng.py:38-68
    sample_runs                   vp/kernels.py:36-88
    parallel_fill                 vp/executor.py:133-166
    update_evals_per_cube         vp/strat.py:88-113
    build_run_plan                vp/strat.py:131-137
    compute_results               vp/strat.py:183-208
    smooth_and_damp               vp/maps.py:160-199
    update_grid                   vp/maps.py:202-234
    pairwise_sum                  numpy float64 add.reduce
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .errors import ContractViolationError, NonFiniteIntegrandError
from .integrands import resolve


def philox_words(block, stream, seed):
    """Vectorised Philox4x32-10: returns (w0, w1) uint64 arrays."""
    b, s, k = np.broadcast_arrays(N.u64(block), N.u64(stream), N.u64(seed))
    b, s, k = N.u64(b).ravel(), N.u64(s).ravel(), N.u64(k).ravel()
    out = np.empty(2 * b.size, dtype=np.uint64)
    N.check(N.load().vpb_philox_host(N.ptr(b), N.ptr(s), N.ptr(k), b.size, N.ptr(out)))
    return out[0::2], out[1::2]


def uniform_at(seed, stream_id, position):
    """u in [0, 1) at (seed, stream, position); arrays broadcast."""
    k, s, p = np.broadcast_arrays(N.u64(seed), N.u64(stream_id), N.u64(position))
    shape = k.shape
    k, s, p = N.u64(k).ravel(), N.u64(s).ravel(), N.u64(p).ravel()
    out = np.empty(k.size)
    N.check(N.load().vpb_uniform_at_host(N.ptr(k), N.ptr(s), N.ptr(p), k.size, N.ptr(out)))
    return out.reshape(shape) if shape else float(out[0])


def sample_runs(seed, batch_size, run_base, run_start, n, offsets, edges, n_strat):
    """Points, Jacobians, interval and cube indices of runs [run_start, run_start+n)."""
    offsets = N.i64(offsets)
    edges = N.f64(edges)
    dims, ng1 = edges.shape
    x = np.empty((n, dims))
    jac = np.empty(n)
    idx = np.empty((n, dims), dtype=np.int64)
    cube = np.empty(n, dtype=np.int64)
    if n:
        N.check(N.load().vpb_sample_runs_host(
            int(seed), int(batch_size), int(run_base), int(run_start), int(n), N.ptr(offsets),
            offsets.size - 1, N.ptr(edges), dims, ng1 - 1, int(n_strat), N.ptr(x), N.ptr(jac),
            N.ptr(idx), N.ptr(cube)))
    return x, jac, idx, cube


def parallel_fill(offsets, edges, n_strat, seed, batch_size, f, run_base=0, run_lo=0,
                  run_hi=None):
    """Fused fill of runs [run_lo, run_hi) -> (map_w, map_counts, s1, s2, counts)."""
    dev = resolve(f)
    offsets = N.i64(offsets)
    edges = N.f64(edges)
    dims, ng1 = edges.shape
    ng = ng1 - 1
    n_cubes = offsets.size - 1
    if run_hi is None:
        run_hi = int(offsets[-1])
    p = dev.params(dims)
    mw = np.empty((dims, ng))
    mc = np.empty((dims, ng), dtype=np.int64)
    s1 = np.empty(n_cubes)
    s2 = np.empty(n_cubes)
    cnt = np.empty(n_cubes, dtype=np.int64)
    er = ctypes.c_int64(-1)
    ev = ctypes.c_double()
    ep = np.zeros(dims)
    rc = N.load().vpb_fill_host(N.ptr(offsets), n_cubes, N.ptr(edges), dims, ng, int(n_strat),
                                int(seed), int(batch_size), int(run_base), dev.device_id,
                                N.ptr(p), p.size, int(run_lo), int(run_hi), N.ptr(mw), N.ptr(mc),
                                N.ptr(s1), N.ptr(s2), N.ptr(cnt), ctypes.byref(er), N.ptr(ep),
                                ctypes.byref(ev))
    if rc == N.VPB_ERR_NONFINITE:
        raise NonFiniteIntegrandError(ep.copy(), ev.value, er.value)
    N.check(rc, "parallel_fill")
    return mw, mc, s1, s2, cnt


def pairwise_sum(a) -> float:
    a = N.f64(a).ravel()
    out = ctypes.c_double()
    N.check(N.load().vpb_pairwise_sum_host(N.ptr(a), a.size, ctypes.byref(out)))
    return out.value


def power(x, y: float) -> np.ndarray:
    """x ** y as the allocation kernel computes it (numpy's scalar-power
    fast paths for y in {0, 0.5, 1, 2}, else device pow)."""
    x = N.f64(x).ravel()
    out = np.empty_like(x)
    N.check(N.load().vpb_pow_host(N.ptr(x), x.size, float(y), N.ptr(out)))
    return out


def update_evals_per_cube(d_h, beta: float, n_eval: int) -> np.ndarray:
    d_h = N.f64(d_h).ravel()
    out = np.empty(d_h.size, dtype=np.int64)
    N.check(N.load().vpb_update_evals_host(N.ptr(d_h), d_h.size, float(beta), int(n_eval),
                                           N.ptr(out)), "update_evals_per_cube")
    return out


def build_run_plan(n_h) -> np.ndarray:
    n_h = N.i64(n_h).ravel()
    off = np.empty(n_h.size + 1, dtype=np.int64)
    N.check(N.load().vpb_build_plan_host(N.ptr(n_h), n_h.size, N.ptr(off)), "build_run_plan")
    return off


def compute_results(s1, s2, counts):
    """-> (I_it, var_it, d_h); AssertionError if a cube has < 2 samples."""
    s1, s2, counts = N.f64(s1), N.f64(s2), N.i64(counts)
    n = s1.size
    d_h = np.empty(n)
    i_it, v_it = ctypes.c_double(), ctypes.c_double()
    N.check(N.load().vpb_compute_results_host(N.ptr(s1), N.ptr(s2), N.ptr(counts), n,
                                              ctypes.byref(i_it), ctypes.byref(v_it),
                                              N.ptr(d_h)), "compute_results")
    return i_it.value, v_it.value, d_h


def smooth_and_damp(map_w, map_counts, alpha: float) -> np.ndarray:
    if alpha < 0:
        raise ContractViolationError(f"alpha must be >= 0, got {alpha}")
    w, c = N.f64(map_w), N.i64(map_counts)
    out = np.empty_like(w)
    N.check(N.load().vpb_smooth_and_damp_host(N.ptr(w), N.ptr(c), w.shape[0], w.shape[1],
                                              float(alpha), N.ptr(out)), "smooth_and_damp")
    return out


def update_grid(edges, damped) -> np.ndarray:
    e, dm = N.f64(edges), N.f64(damped)
    if dm.shape != (e.shape[0], e.shape[1] - 1):
        raise ContractViolationError(
            f"damped weights shape {dm.shape} != {(e.shape[0], e.shape[1] - 1)}")
    out = np.empty_like(e)
    N.check(N.load().vpb_update_grid_host(N.ptr(e), N.ptr(dm), e.shape[0], e.shape[1] - 1,
                                          N.ptr(out)), "update_grid")
    return out
