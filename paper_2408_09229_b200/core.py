"""The iteration loop and public result types (drop-in for vp/core.py).

``integrate`` keeps the reference signature (vp/core.py:168-169) and result
types (vp/core.py:29-148).  The per-iteration body (vp/core.py:200-219) runs
entirely on the GPU through one C-ABI context: the host enqueues all
``max_it`` iterations without synchronising and reads the history once.

Extra keyword-only arguments (not in the reference; defaults keep the
reference behaviour):
  device       CUDA ordinal (default: LOCAL_RANK or the current device)
  distributed  True/False/None: shard runs over torch.distributed ranks and
               merge with NCCL (None = when a process group with >1 rank is
               initialised)
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import (ContractViolationError, IntegrationError, InvalidDomainError,
                     NonFiniteIntegrandError)
from .integrands import DeviceIntegrand, resolve

DEFAULT_MAX_IT = 20
DEFAULT_BATCH_SIZE = 1_048_576
DEFAULT_N_INTERVALS = 1024
DEFAULT_ALPHA = 0.5
DEFAULT_BETA = 0.75
DEFAULT_CUBE_CAP = 1 << 20     # vp/strat.py:19
MIN_EVALS_PER_CUBE = 2


@dataclass(frozen=True)
class IntegratorConfig:
    """Knobs of one integration run (fields, defaults, validation as
    vp/core.py:29-62).  ``workers`` is validated and kept for API
    compatibility; on the GPU the evaluation budget is spread over all SMs
    (and over ranks when distributed) regardless of it."""

    n_eval: int
    max_it: int = DEFAULT_MAX_IT
    skip: int = 0
    batch_size: int = DEFAULT_BATCH_SIZE
    n_intervals: int = DEFAULT_N_INTERVALS
    alpha: float = DEFAULT_ALPHA
    beta: float = DEFAULT_BETA
    seed: int = 0
    workers: int = 1
    cube_cap: int = DEFAULT_CUBE_CAP
    n_strat: int | None = None

    def __post_init__(self):
        if self.n_eval < 4:
            raise ContractViolationError(f"n_eval must be >= 4, got {self.n_eval}")
        if not self.max_it > self.skip >= 0:
            raise ContractViolationError(
                f"need max_it > skip >= 0, got max_it={self.max_it} skip={self.skip}")
        if self.batch_size < 1:
            raise ContractViolationError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.n_intervals < 2:
            raise ContractViolationError(f"n_intervals must be >= 2, got {self.n_intervals}")
        if self.alpha < 0 or self.beta < 0:
            raise ContractViolationError("alpha and beta must be >= 0")
        if self.workers < 1:
            raise ContractViolationError(f"workers must be >= 1, got {self.workers}")
        if self.cube_cap < 1:
            raise ContractViolationError(f"cube_cap must be >= 1, got {self.cube_cap}")


@dataclass(frozen=True)
class IterationResult:
    index: int          # 1-based
    estimate: float
    variance: float
    included: bool      # index > skip

    @property
    def sigma(self) -> float:
        return float(np.sqrt(self.variance))


@dataclass
class PhaseTimes:
    """Seconds per algorithm phase (map/fill/update: CUDA-event device time;
    init/clear: host wall time)."""

    init: float = 0.0
    map: float = 0.0
    fill: float = 0.0
    update: float = 0.0
    clear: float = 0.0

    def total(self) -> float:
        return self.init + self.map + self.fill + self.update + self.clear

    def percentages(self) -> dict[str, float]:
        tot = self.total()
        if tot <= 0.0:
            return {k: 0.0 for k in ("init", "map", "fill", "update", "clear")}
        return {
            "init": 100.0 * self.init / tot,
            "map": 100.0 * self.map / tot,
            "fill": 100.0 * self.fill / tot,
            "update": 100.0 * self.update / tot,
            "clear": 100.0 * self.clear / tot,
        }


@dataclass(frozen=True)
class IntegralOutcome:
    mean: float
    sigma: float
    chi2_dof: float
    iterations: tuple
    timing: PhaseTimes
    n_strat: int
    n_cubes: int
    evals_per_iteration: tuple

    def included(self) -> list:
        return [r for r in self.iterations if r.included]


def combine_iterations(results):
    """Inverse-variance weighted combination (vp/core.py:118-148, unchanged:
    exact math.fsum sums, zero-variance short-circuit)."""
    results = list(results)
    if not results:
        raise IntegrationError("no iteration results to combine")
    est = [float(r.estimate) for r in results]
    var = [float(r.variance) for r in results]
    if any(v < 0 for v in var):
        raise ContractViolationError("iteration variance must be >= 0")
    if 0.0 in var:
        vals = {e for e, v in zip(est, var) if v == 0.0}
        if len(vals) > 1:
            raise IntegrationError(f"conflicting exact estimates (sigma = 0): {sorted(vals)}")
        return vals.pop(), 0.0, 0.0
    if len(results) == 1:
        return est[0], var[0], 0.0
    w = [1.0 / v for v in var]
    wsum = math.fsum(w)
    mean = math.fsum(e * wi for e, wi in zip(est, w)) / wsum
    variance = 1.0 / wsum
    chi2_dof = math.fsum((e - mean) ** 2 * wi for e, wi in zip(est, w)) / (len(results) - 1)
    return mean, variance, chi2_dof


# ---------------------------------------------------------- stratification --

def _iroot(x: int, d: int) -> int:
    """Largest n >= 1 with n**d <= x (vp/strat.py:25-35)."""
    if x < 1:
        return 1
    n = max(1, int(x ** (1.0 / d)))
    while n > 1 and n ** d > x:
        n -= 1
    while (n + 1) ** d <= x:
        n += 1
    return n


def compute_n_strat(n_eval: int, dims: int, cube_cap: int = DEFAULT_CUBE_CAP) -> int:
    """Strata per axis (vp/strat.py:37-46)."""
    if dims < 1:
        raise ContractViolationError(f"dims must be >= 1, got {dims}")
    return min(_iroot(n_eval // 2, dims), _iroot(cube_cap, dims))


def _grid_strata(config: IntegratorConfig, dims: int) -> int:
    # vp/strat.py:74-85 (initial_grid validation)
    ns = int(config.n_strat) if config.n_strat is not None else \
        compute_n_strat(config.n_eval, dims, config.cube_cap)
    if ns < 1:
        raise ContractViolationError(f"n_strat must be >= 1, got {ns}")
    if ns ** dims > config.cube_cap:
        raise ContractViolationError(
            f"n_strat={ns} gives {ns ** dims} cubes, above the cap {config.cube_cap}")
    return ns


def _check_bounds(dims, n_intervals, bounds):
    # vp/maps.py:72-84
    if dims < 1:
        raise InvalidDomainError(f"dims must be >= 1, got {dims}")
    if n_intervals < 2:
        raise InvalidDomainError(f"n_intervals must be >= 2, got {n_intervals}")
    for j, (lo, hi) in enumerate(bounds):
        if not (np.isfinite(lo) and np.isfinite(hi)) or not lo < hi:
            raise InvalidDomainError(f"bad bounds for dimension {j}: ({lo}, {hi})")


def _default_device() -> int:
    """LOCAL_RANK's GPU, modulo the visible devices: launchers that set
    CUDA_VISIBLE_DEVICES per rank leave every rank one device (ordinal 0)."""
    if "LOCAL_RANK" in os.environ:
        n = ctypes.c_int32(0)
        N.check(N.load().vpb_device_count(ctypes.byref(n)), "vpb_device_count")
        return int(os.environ["LOCAL_RANK"]) % max(1, n.value)
    return -1


# ------------------------------------------------------------- integrator --

class Integrator:
    """One C-ABI context: the device-resident state of an integration
    (map edges, allocation, accumulators, history).  ``integrate`` drives one;
    bench.py and the tests drive it directly to time single iterations."""

    def __init__(self, f, bounds, config: IntegratorConfig, *, device: int | None = None,
                 distributed: bool | None = None, stream: int | None = None,
                 exchange: str | None = None, deterministic: bool | None = None):
        self.config = config
        self.bounds = [(float(lo), float(hi)) for lo, hi in bounds]
        self.dims = len(self.bounds)
        _check_bounds(self.dims, config.n_intervals, self.bounds)
        if self.dims > N.MAX_DIMS:
            raise ContractViolationError(f"at most {N.MAX_DIMS} dimensions are supported")
        self.integrand: DeviceIntegrand = resolve(f)
        self.n_strat = _grid_strata(config, self.dims)
        self.n_cubes = self.n_strat ** self.dims
        self.params = self.integrand.params(self.dims)
        self._bounds_flat = N.f64(np.array(self.bounds).ravel())
        lib = N.load()
        desc = N.VpbDesc()
        desc.dims = self.dims
        desc.n_intervals = config.n_intervals
        desc.n_strat = self.n_strat
        desc.n_eval = config.n_eval
        desc.batch_size = config.batch_size
        desc.seed = int(config.seed) & 0xFFFFFFFFFFFFFFFF
        desc.alpha = float(config.alpha)
        desc.beta = float(config.beta)
        desc.integrand = self.integrand.device_id
        desc.n_params = self.params.size
        desc.params = self.params.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        desc.bounds = self._bounds_flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        desc.device = _default_device() if device is None else int(device)
        desc.max_it = int(config.max_it)
        desc.stream = stream
        if deterministic is None:
            deterministic = os.environ.get("VPB_DETERMINISTIC", "0") == "1"
        desc.flags = N.VPB_FLAG_DETERMINISTIC if deterministic else 0
        self.deterministic = bool(deterministic)
        self._lib = lib
        ctx = ctypes.c_void_p()
        N.check(lib.vpb_create(ctypes.byref(desc), ctypes.byref(ctx)), "vpb_create")
        self._ctx = ctx
        self.world, self.rank = 1, 0
        self._exchange_cb = None
        self._maybe_distribute(distributed, exchange or os.environ.get("VPB_EXCHANGE", "nccl"))

    # -- multi-GPU ------------------------------------------------------------
    def _maybe_distribute(self, distributed, exchange="nccl"):
        if distributed is False:
            return
        try:
            import torch.distributed as dist
        except Exception:  # pragma: no cover
            if distributed:
                raise
            return
        if not (dist.is_available() and dist.is_initialized()):
            if distributed:
                raise ContractViolationError("distributed=True needs an initialised process group")
            return
        world, rank = dist.get_world_size(), dist.get_rank()
        if world == 1 and not distributed:
            return
        if exchange == "host":
            # the exchange through torch.distributed on host buffers (any
            # backend, e.g. gloo; ranks may share a GPU) instead of NCCL
            from .distributed import host_allreduce_callback
            self._exchange_cb = host_allreduce_callback()
            N.check(self._lib.vpb_attach_exchange(self._ctx, world, rank, self._exchange_cb,
                                                  None), "vpb_attach_exchange")
        elif exchange == "nccl":
            from .distributed import nccl_unique_id_broadcast
            uid = nccl_unique_id_broadcast(self._lib)
            N.check(self._lib.vpb_attach_nccl(self._ctx, uid, world, rank), "vpb_attach_nccl")
        else:
            raise ContractViolationError(f"exchange must be 'nccl' or 'host', got {exchange!r}")
        self.world, self.rank = world, rank

    # -- iteration control --------------------------------------------------------
    def reset(self):
        N.check(self._lib.vpb_reset(self._ctx), "vpb_reset")

    def iterate(self, n: int = 1):
        """Enqueue n iterations (asynchronous)."""
        N.check(self._lib.vpb_iterate(self._ctx, int(n)), "vpb_iterate")

    def sync(self):
        N.check(self._lib.vpb_sync(self._ctx))

    def history(self):
        cap = self.config.max_it
        est = np.zeros(cap)
        var = np.zeros(cap)
        ev = np.zeros(cap, dtype=np.int64)
        n = ctypes.c_int32()
        rc = self._lib.vpb_history(self._ctx, cap, N.ptr(est), N.ptr(var), N.ptr(ev),
                                   ctypes.byref(n))
        if rc == N.VPB_ERR_NONFINITE:
            self._raise_nonfinite()
        N.check(rc, "integrate")
        k = n.value
        return est[:k], var[:k], ev[:k]

    def _raise_nonfinite(self):
        run = ctypes.c_int64()
        val = ctypes.c_double()
        pt = np.zeros(self.dims)
        N.check(self._lib.vpb_error_info(self._ctx, ctypes.byref(run), N.ptr(pt),
                                         ctypes.byref(val)))
        raise NonFiniteIntegrandError(pt, val.value, run.value)

    def phase_times_ms(self):
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        N.check(self._lib.vpb_phase_times(self._ctx, ctypes.byref(a), ctypes.byref(b),
                                          ctypes.byref(c)))
        return a.value, b.value, c.value

    def timing_ms(self, first: int, count: int):
        """(iteration ms, fill-kernel ms) summed over iterations [first, first+count)."""
        a, k = ctypes.c_double(), ctypes.c_double()
        N.check(self._lib.vpb_timing(self._ctx, int(first), int(count), ctypes.byref(a),
                                     ctypes.byref(k)))
        return a.value, k.value

    _LAYOUTS = {0: "edge rows + shared histograms", 1: "pair table + shared histograms",
                2: "records + per-group shared histograms", 3: "generic runtime-dims kernel",
                4: "split: 2-CTA clusters, half the axes' map rows and histograms per SM"}

    def fill_layout(self) -> dict:
        """The fill's shared-memory layout, record chunks per iteration and
        this library's kernel launches per iteration (vpb_fill_layout)."""
        lay, ch, ln = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        N.check(self._lib.vpb_fill_layout(self._ctx, ctypes.byref(lay), ctypes.byref(ch),
                                          ctypes.byref(ln)))
        return {"layout": self._LAYOUTS.get(lay.value, str(lay.value)), "chunks": ch.value,
                "launches_per_iteration": ln.value}

    def fx_stats(self) -> dict:
        """Fixed-point interval histograms (vpb_fx_stats): whether the mode is
        on for this context, iterations filled in fixed point, iterations
        refilled in f64 after a failed proof, values summed in f64 instead."""
        out = np.zeros(4, dtype=np.int64)
        N.check(self._lib.vpb_fx_stats(self._ctx, N.ptr(out)))
        return {"enabled": bool(out[0]), "fixed_iterations": int(out[1]),
                "refilled": int(out[2]), "spilled_values": int(out[3])}

    def last_fill_ms(self) -> float:
        t = ctypes.c_double()
        N.check(self._lib.vpb_last_fill_ms(self._ctx, ctypes.byref(t)))
        return t.value

    def iteration_host(self, edges_in: np.ndarray | None, edges_out: np.ndarray | None):
        """One iteration through host buffers (e2e path)."""
        est, var, ev = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        rc = self._lib.vpb_iteration_host(
            self._ctx, None if edges_in is None else N.ptr(edges_in),
            None if edges_out is None else N.ptr(edges_out), ctypes.byref(est),
            ctypes.byref(var), ctypes.byref(ev))
        if rc == N.VPB_ERR_NONFINITE:
            self._raise_nonfinite()
        N.check(rc, "iteration")
        return est.value, var.value, ev.value

    # -- state access --------------------------------------------------------------
    def edges(self) -> np.ndarray:
        e = np.empty((self.dims, self.config.n_intervals + 1))
        N.check(self._lib.vpb_get_edges(self._ctx, N.ptr(e)))
        return e

    def set_edges(self, edges):
        e = N.f64(edges)
        if e.shape != (self.dims, self.config.n_intervals + 1):
            raise ContractViolationError("edges shape mismatch")
        N.check(self._lib.vpb_set_edges(self._ctx, N.ptr(e)))

    def plan(self):
        n_h = np.empty(self.n_cubes, dtype=np.int64)
        off = np.empty(self.n_cubes + 1, dtype=np.int64)
        N.check(self._lib.vpb_get_plan(self._ctx, N.ptr(n_h), N.ptr(off)))
        return n_h, off

    def set_allocation(self, n_h):
        n_h = N.i64(n_h)
        if n_h.shape != (self.n_cubes,):
            raise ContractViolationError("n_h shape mismatch")
        N.check(self._lib.vpb_set_allocation(self._ctx, N.ptr(n_h)))

    def spread(self) -> np.ndarray:
        d = np.empty(self.n_cubes)
        N.check(self._lib.vpb_get_spread(self._ctx, N.ptr(d)))
        return d

    def accumulators(self):
        ng = self.config.n_intervals
        mw = np.empty((self.dims, ng))
        mc = np.empty((self.dims, ng), dtype=np.int64)
        s1 = np.empty(self.n_cubes)
        s2 = np.empty(self.n_cubes)
        cnt = np.empty(self.n_cubes, dtype=np.int64)
        N.check(self._lib.vpb_get_fill(self._ctx, N.ptr(mw), N.ptr(mc), N.ptr(s1), N.ptr(s2),
                                       N.ptr(cnt)))
        return mw, mc, s1, s2, cnt

    def set_shard(self, world: int, rank: int):
        """Fill only rank's share of each plan (vp/executor.py:41-57 rule)
        without a communicator: the caller merges the accumulators (what the
        NCCL all-reduce does in a distributed run)."""
        N.check(self._lib.vpb_set_shard(self._ctx, int(world), int(rank)), "vpb_set_shard")
        self.world, self.rank = int(world), int(rank)

    def fill(self, run_base: int):
        rc = self._lib.vpb_fill(self._ctx, int(run_base))
        if rc == N.VPB_ERR_NONFINITE:
            self._raise_nonfinite()
        N.check(rc, "fill")

    def run_base(self) -> int:
        v = ctypes.c_int64()
        N.check(self._lib.vpb_get_run_base(self._ctx, ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.vpb_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def integrate(f, bounds, config: IntegratorConfig | None = None, *,
              batched: bool = False, device: int | None = None,
              distributed: bool | None = None, exchange: str | None = None,
              deterministic: bool | None = None, **overrides) -> IntegralOutcome:
    """Integrate a registered device integrand over the box given by bounds.

    Same contract as vp/core.py:168-238.  ``f`` is a registered integrand
    (``lookup(name)``, its ``.evaluate_batch``, or its name); ``batched`` is
    accepted for compatibility (device functors are always batched).
    """
    if config is None:
        config = IntegratorConfig(**overrides)
    elif overrides:
        raise TypeError("pass either a config object or keyword overrides, not both")
    bounds = [(float(lo), float(hi)) for lo, hi in bounds]
    timing = PhaseTimes()
    t0 = time.perf_counter()
    integ = Integrator(f, bounds, config, device=device, distributed=distributed,
                       exchange=exchange, deterministic=deterministic)
    timing.init = time.perf_counter() - t0
    try:
        integ.iterate(config.max_it)
        est, var, evals = integ.history()
        map_ms, fill_ms, upd_ms = integ.phase_times_ms()
        timing.map = map_ms * 1e-3
        timing.fill = fill_ms * 1e-3
        timing.update = upd_ms * 1e-3
        n_strat, n_cubes = integ.n_strat, integ.n_cubes
    finally:
        t = time.perf_counter()
        integ.close()
        timing.clear = time.perf_counter() - t
    results = [IterationResult(i + 1, float(est[i]), float(var[i]), (i + 1) > config.skip)
               for i in range(len(est))]
    included = [r for r in results if r.included]
    mean, variance, chi2_dof = combine_iterations(included)
    return IntegralOutcome(
        mean=mean,
        sigma=float(np.sqrt(variance)),
        chi2_dof=chi2_dof,
        iterations=tuple(results),
        timing=timing,
        n_strat=n_strat,
        n_cubes=n_cubes,
        evals_per_iteration=tuple(int(e) for e in evals),
    )
