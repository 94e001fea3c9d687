"""CPU oracle for the VEGAS+ hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product
(paper_2408_09229_b200) never imports it; the product fails loudly when its
CUDA library is missing instead of falling back here.

Contents
--------
* vegas_oracle.c  -- C restatement of the reference hot path (Philox,
  sample_runs, accumulate, parallel fill + tree reduce, numpy pairwise sum,
  allocation, run plan, compute_results, smooth_and_damp, update_grid,
  integrands).  Each C function cites the reference lines it restates.
* this module     -- ctypes bindings, the integrand parameter blobs (computed
  with the same Python expressions as vp/integrands.py), and
  :func:`integrate`, a restatement of vp/core.py:168-238 on top of the C code.
* integrands_np   -- numpy definitions of the BASELINE-pinned integrands.
* gen_golden.py   -- dumps golden vectors from the real reference (dev only).

Parity status: PINNED against tests/golden (see tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

from . import integrands_np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libvegas_oracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc -O3 -ffp-contract=off -pthread)."""
    src = os.path.join(HERE, "vegas_oracle.c")
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        c = ctypes
        L.vo_philox.argtypes = [c.c_uint64, c.c_uint64, c.c_uint64, _u64p]
        L.vo_uniform_at.argtypes = [c.c_uint64, c.c_uint64, c.c_uint64]
        L.vo_uniform_at.restype = c.c_double
        L.vo_sample_runs.argtypes = [c.c_uint64, c.c_int64, c.c_int64, c.c_int64, c.c_int64,
                                     _i64p, c.c_int64, _f64p, c.c_int, c.c_int, c.c_int64,
                                     _f64p, _f64p, _i64p, _i64p]
        L.vo_eval.argtypes = [c.c_int, _f64p, _f64p, c.c_int64, c.c_int, _f64p]
        L.vo_fill.argtypes = [_i64p, c.c_int64, _f64p, c.c_int, c.c_int, c.c_int64, c.c_uint64,
                              c.c_int64, c.c_int64, c.c_int, _f64p, c.c_int, c.c_int64,
                              c.c_int64, _f64p, _i64p, _f64p, _f64p, _i64p,
                              c.POINTER(c.c_int64), _f64p, c.POINTER(c.c_double)]
        L.vo_fill.restype = c.c_int
        L.vo_partition_runs.argtypes = [c.c_int64, c.c_int64, _i64p, _i64p]
        L.vo_pairwise_sum.argtypes = [_f64p, c.c_int64]
        L.vo_pairwise_sum.restype = c.c_double
        L.vo_update_evals.argtypes = [_f64p, c.c_int64, c.c_double, c.c_int64, c.c_void_p, _i64p]
        L.vo_build_plan.argtypes = [_i64p, c.c_int64, _i64p]
        L.vo_compute_results.argtypes = [_f64p, _f64p, _i64p, c.c_int64, c.POINTER(c.c_double),
                                         c.POINTER(c.c_double), _f64p, c.POINTER(c.c_int64)]
        L.vo_compute_results.restype = c.c_int
        L.vo_smooth_and_damp.argtypes = [_f64p, _i64p, c.c_int, c.c_int, c.c_double, _f64p]
        L.vo_update_grid.argtypes = [_f64p, _f64p, c.c_int, c.c_int, _f64p]
        L.vo_update_grid.restype = c.c_int
        _LIB = L
    return _LIB


# ---------------------------------------------------------------- RNG -----

def philox_words(block: int, stream: int, seed: int):
    out = np.zeros(2, dtype=np.uint64)
    lib().vo_philox(block, stream, seed, out)
    return int(out[0]), int(out[1])


def uniform_at(seed: int, stream: int, pos: int) -> float:
    return lib().vo_uniform_at(seed, stream, pos)


def sample_runs(seed, batch, run_base, run_start, n, offsets, cube_start, edges, n_strat):
    edges = np.ascontiguousarray(edges, dtype=np.float64)
    dims, ng1 = edges.shape
    x = np.empty((n, dims))
    jac = np.empty(n)
    idx = np.empty((n, dims), dtype=np.int64)
    cube = np.empty(n, dtype=np.int64)
    lib().vo_sample_runs(seed, batch, run_base, run_start, n,
                         np.ascontiguousarray(offsets, dtype=np.int64), cube_start, edges,
                         dims, ng1 - 1, n_strat, x, jac, idx, cube)
    return x, jac, idx, cube


# --------------------------------------------------------- integrands -----

ORACLE_IDS = {"gaussian": 0, "ridge": 1, "multipeak8": 2, "genz_oscillatory6": 3,
              "genz_productpeak6": 4, "sinexp": 5, "linear": 6, "cosine": 7,
              "exponential": 8, "roos_arnold": 9, "morokoff": 10, "constant": 11,
              "gaussian20": 0, "asian_option": 12, "path_integral": 13}

_DIMS = {"gaussian": 4, "ridge": 4, "multipeak8": 8, "genz_oscillatory6": 6,
         "genz_productpeak6": 6, "sinexp": 2, "linear": 10, "cosine": 10,
         "exponential": 10, "roos_arnold": 10, "morokoff": 8, "gaussian20": 20,
         "asian_option": 16, "path_integral": 7}

# vp/integrands.py:190, 226-227 (ASIAN_DEFAULTS, PATH_DEFAULTS, CLAMP_EPS)
ASIAN_DEFAULTS = dict(s0=100.0, strike=100.0, rate=0.05, sigma=0.2, maturity=1.0)
PATH_DEFAULTS = dict(mass=1.0, total_time=4.0, x_end=0.0)


def integrand_params(name: str, dims: int | None = None, value: float = 1.0,
                     **kw) -> np.ndarray:
    """Parameter blob for the C evaluator, built with the reference's own
    Python expressions (vp/integrands.py:131-251, oracle/integrands_np.py)."""
    d = dims or _DIMS.get(name, 1)
    if name == "asian_option":   # vp/integrands.py:196-210
        q = dict(ASIAN_DEFAULTS, **kw)
        drift = (q["rate"] - 0.5 * q["sigma"] * q["sigma"]) * q["maturity"]
        return np.array([q["s0"], q["strike"], drift, q["sigma"] * math.sqrt(q["maturity"]),
                         math.exp(-q["rate"] * q["maturity"]), 1e-12])
    if name == "path_integral":   # vp/integrands.py:233-251, n_slices = d + 1
        q = dict(PATH_DEFAULTS, **kw)
        n_slices = d + 1
        a = q["total_time"] / n_slices
        amp = (q["mass"] / (2.0 * math.pi * a)) ** (n_slices / 2.0)
        return np.array([q["mass"] / (2.0 * a), 0.5 * a, amp, q["x_end"]])
    if name in ("gaussian", "gaussian20"):
        mu, sigma = (0.5, 0.01) if name == "gaussian" else (0.5, 0.1)
        norm = (2.0 * math.pi * sigma ** 2) ** (-d / 2.0)
        return np.array([mu, sigma, norm, 2.0 * sigma ** 2])
    if name == "ridge":
        n = 1000
        return np.array([float(n), 10000.0 / (math.pi ** 2 * n), math.sqrt(46.0 / 400.0)])
    if name == "multipeak8":
        s = integrands_np.MP_SIGMA
        norm = (2.0 * math.pi * s ** 2) ** (-d / 2.0)
        return np.array([3.0, s, norm, 2.0 * s ** 2, 3.0] + list(integrands_np.MP_MUS))
    if name == "genz_oscillatory6":
        return np.concatenate(([2.0 * math.pi * integrands_np.GENZ_OSC_U[0]],
                               integrands_np.GENZ_OSC_A))
    if name == "genz_productpeak6":
        return np.concatenate((integrands_np.GENZ_PP_A ** -2.0, integrands_np.GENZ_PP_U))
    if name == "morokoff":
        return np.array([(1.0 + 1.0 / d) ** d, 1.0 / d])
    if name == "constant":
        return np.array([float(value)])
    return np.zeros(1)


def evaluate(name: str, x: np.ndarray, params: np.ndarray | None = None) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    p = integrand_params(name, d) if params is None else np.ascontiguousarray(params)
    out = np.empty(n)
    lib().vo_eval(ORACLE_IDS[name], p, x, n, d, out)
    return out


# --------------------------------------------------------------- strat ----

def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().vo_pairwise_sum(a, a.shape[0])


def update_evals_per_cube(d_h, beta: float, n_eval: int, dp=None) -> np.ndarray:
    d_h = np.ascontiguousarray(d_h, dtype=np.float64)
    out = np.empty(d_h.shape[0], dtype=np.int64)
    dpp = None
    if dp is not None:
        dp = np.ascontiguousarray(dp, dtype=np.float64)
        dpp = dp.ctypes.data
    lib().vo_update_evals(d_h, d_h.shape[0], float(beta), int(n_eval), dpp, out)
    return out


def build_run_plan(n_h) -> np.ndarray:
    n_h = np.ascontiguousarray(n_h, dtype=np.int64)
    off = np.empty(n_h.shape[0] + 1, dtype=np.int64)
    lib().vo_build_plan(n_h, n_h.shape[0], off)
    return off


def _iroot(x: int, d: int) -> int:
    # vp/strat.py:25-35
    if x < 1:
        return 1
    n = max(1, int(x ** (1.0 / d)))
    while n > 1 and n ** d > x:
        n -= 1
    while (n + 1) ** d <= x:
        n += 1
    return n


def compute_n_strat(n_eval: int, dims: int, cube_cap: int = 1 << 20) -> int:
    # vp/strat.py:37-46
    return min(_iroot(n_eval // 2, dims), _iroot(cube_cap, dims))


def compute_results(s1, s2, counts):
    s1 = np.ascontiguousarray(s1, dtype=np.float64)
    s2 = np.ascontiguousarray(s2, dtype=np.float64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    n = s1.shape[0]
    d_h = np.empty(n)
    i_it, var_it, bad = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    rc = lib().vo_compute_results(s1, s2, counts, n, ctypes.byref(i_it), ctypes.byref(var_it),
                                  d_h, ctypes.byref(bad))
    if rc:
        raise AssertionError(f"cube {bad.value} has {counts[bad.value]} samples; "
                             f"every cube needs >= 2")
    return i_it.value, var_it.value, d_h


def smooth_and_damp(map_w, map_counts, alpha: float) -> np.ndarray:
    w = np.ascontiguousarray(map_w, dtype=np.float64)
    c = np.ascontiguousarray(map_counts, dtype=np.int64)
    out = np.empty_like(w)
    lib().vo_smooth_and_damp(w, c, w.shape[0], w.shape[1], float(alpha), out)
    return out


def update_grid(edges, damped) -> np.ndarray:
    e = np.ascontiguousarray(edges, dtype=np.float64)
    dm = np.ascontiguousarray(damped, dtype=np.float64)
    out = np.empty_like(e)
    bad = lib().vo_update_grid(e, dm, e.shape[0], e.shape[1] - 1, out)
    if bad >= 0:
        raise AssertionError(f"grid update lost strict monotonicity in dimension {bad}")
    return out


def new_uniform_edges(dims: int, ng: int, bounds) -> np.ndarray:
    # vp/maps.py:70-88
    edges = np.empty((dims, ng + 1))
    for j, (lo, hi) in enumerate(bounds):
        edges[j] = np.linspace(float(lo), float(hi), ng + 1)
        edges[j, 0], edges[j, -1] = float(lo), float(hi)
    return edges


# ---------------------------------------------------------------- fill ----

class NonFinite(Exception):
    def __init__(self, point, value, run_index):
        super().__init__(f"non-finite {value} at {list(point)} (run {run_index})")
        self.point, self.value, self.run_index = point, value, run_index


def fill(offsets, edges, n_strat, seed, batch, run_base, name, params=None, workers=1,
         run_lo=0, run_hi=None):
    """parallel_fill (vp/executor.py:133-166) over runs [run_lo, run_hi)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    edges = np.ascontiguousarray(edges, dtype=np.float64)
    dims, ng1 = edges.shape
    ng = ng1 - 1
    n_cubes = offsets.shape[0] - 1
    if run_hi is None:
        run_hi = int(offsets[-1])
    p = integrand_params(name, dims) if params is None else np.ascontiguousarray(params)
    mw = np.empty((dims, ng))
    mc = np.empty((dims, ng), dtype=np.int64)
    s1 = np.empty(n_cubes)
    s2 = np.empty(n_cubes)
    cnt = np.empty(n_cubes, dtype=np.int64)
    er = ctypes.c_int64(-1)
    ev = ctypes.c_double()
    ep = np.zeros(64)
    rc = lib().vo_fill(offsets, n_cubes, edges, dims, ng, int(n_strat), int(seed), int(batch),
                       int(run_base), ORACLE_IDS[name], p, int(workers), int(run_lo),
                       int(run_hi), mw, mc, s1, s2, cnt, ctypes.byref(er), ep, ctypes.byref(ev))
    if rc:
        raise NonFinite(ep[:dims].copy(), ev.value, er.value)
    return mw, mc, s1, s2, cnt


# ----------------------------------------------------------- integrate ----

@dataclass
class OracleOutcome:
    estimates: list
    variances: list
    evals: list
    edges: np.ndarray
    n_h: np.ndarray
    fill_seconds: list
    n_strat: int


def integrate(name, bounds, n_eval, max_it=20, n_intervals=1024, alpha=0.5, beta=0.75,
              seed=0, batch_size=1 << 20, workers=1, params=None, cube_cap=1 << 20,
              n_strat=None) -> OracleOutcome:
    """Restatement of vp/core.py:168-219 on the C oracle (no combine step)."""
    dims = len(bounds)
    edges = new_uniform_edges(dims, n_intervals, bounds)
    ns = int(n_strat) if n_strat is not None else compute_n_strat(n_eval, dims, cube_cap)
    n_cubes = ns ** dims
    n_h = update_evals_per_cube(np.zeros(n_cubes), 0.0, n_eval)
    run_base = 0
    out = OracleOutcome([], [], [], edges, n_h, [], ns)
    for _ in range(max_it):
        offsets = build_run_plan(n_h)
        t = time.perf_counter()
        mw, mc, s1, s2, cnt = fill(offsets, edges, ns, seed, batch_size, run_base, name,
                                   params, workers)
        out.fill_seconds.append(time.perf_counter() - t)
        total = int(offsets[-1])
        run_base += total
        i_it, var_it, d_h = compute_results(s1, s2, cnt)
        n_h = update_evals_per_cube(d_h, beta, n_eval)
        damped = smooth_and_damp(mw, mc, alpha)
        edges = update_grid(edges, damped)
        out.estimates.append(i_it)
        out.variances.append(var_it)
        out.evals.append(total)
    out.edges = edges
    out.n_h = n_h
    return out
