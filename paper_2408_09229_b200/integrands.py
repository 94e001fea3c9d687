"""Integrand registry backed by CUDA device functors.

Same surface as vp/integrands.py:25-43, 399-436: ``IntegrandSpec``,
``lookup(name, dim=None, **params)``, ``available()`` and
``UnknownIntegrandError``.  ``spec.evaluate_batch`` is a
:class:`DeviceIntegrand`: calling it on an (n, d) array evaluates the device
functor on the GPU (csrc/integrands.cuh); passing it (or the spec, or the
name) to :func:`paper_2408_09229_b200.integrate` selects the functor that the
fused fill kernel evaluates in-register.

Registry entries
  reference registry (vp/integrands.py:299-358):
    sinexp, linear, cosine, exponential, roos_arnold, morokoff, gaussian, ridge
  BASELINE-pinned synthetic integrands:
    multipeak8        cfg2: 3 normalised Gaussians at mu_k = k/4, sigma 0.05, d=8
    genz_oscillatory6 cfg4a: cos(2 pi u_1 + a.x), default_rng(2024), sum a = 9
    genz_productpeak6 cfg4b: prod 1/(a^-2 + (x-u)^2), default_rng(2025), sum a = 7.25
    gaussian20        cfg5: d=20, mu=0.5, sigma=0.1
  plus ``constant`` (value param) for exactness tests.
  reference application integrands (vp/integrands.py:186-251, 368-396):
    asian_option      discounted Asian call payoff on erfinv-transformed uniforms
                      (dim = number of averaging dates, default 16)
    path_integral     harmonic-oscillator lattice path-integral weight
                      (dim = interior points = n_slices - 1, default 7)
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native as N
from .errors import ContractViolationError, VegasError

VPB_GAUSSIAN = 0
VPB_RIDGE = 1
VPB_MULTIPEAK = 2
VPB_GENZ_OSCILLATORY = 3
VPB_GENZ_PRODUCTPEAK = 4
VPB_SINEXP = 5
VPB_LINEAR = 6
VPB_COSINE = 7
VPB_EXPONENTIAL = 8
VPB_ROOS_ARNOLD = 9
VPB_MOROKOFF = 10
VPB_CONSTANT = 11
VPB_ASIAN_OPTION = 12
VPB_PATH_INTEGRAL = 13

# vp/integrands.py:21, 190-191, 226-227
CLAMP_EPS = 1e-12
ASIAN_DEFAULTS = dict(s0=100.0, strike=100.0, rate=0.05, sigma=0.2, maturity=1.0,
                      n_averages=16)
PATH_DEFAULTS = dict(mass=1.0, total_time=4.0, n_slices=8, x_end=0.0)
PATH_BOX_HALF_WIDTH = 5.0


class UnknownIntegrandError(VegasError, LookupError):
    def __init__(self, name):
        super().__init__(
            f"unknown integrand {name!r}; available: {', '.join(available_all())}")


class DeviceIntegrand:
    """A device functor id plus a parameter builder ``params(d)``.

    Callable like the reference's ``evaluate_batch``: (n, d) -> (n,), run on
    the GPU.  Parameters that depend on the dimension (the Gaussian
    normalisation) are rebuilt for the dimension actually integrated.
    """

    def __init__(self, name: str, device_id: int, param_fn: Callable[[int], list]):
        self.name = name
        self.device_id = device_id
        self._param_fn = param_fn

    def params(self, dims: int) -> np.ndarray:
        p = np.asarray(self._param_fn(dims), dtype=np.float64).reshape(-1)
        if p.size == 0:
            p = np.zeros(1)
        if p.size > N.MAX_PARAMS:
            raise ContractViolationError(f"{self.name}: too many parameters")
        return p

    def __call__(self, x) -> np.ndarray:
        x = N.f64(x)
        if x.ndim != 2:
            raise ContractViolationError("evaluate_batch expects an (n, d) array")
        n, d = x.shape
        p = self.params(d)
        out = np.empty(n)
        if n:
            N.check(N.load().vpb_eval_host(self.device_id, N.ptr(p), p.size, N.ptr(x), n, d,
                                           N.ptr(out)), self.name)
        return out

    def __repr__(self):
        return f"DeviceIntegrand({self.name!r})"


@dataclass(frozen=True)
class IntegrandSpec:
    name: str
    dims: int
    bounds: tuple
    evaluate_batch: DeviceIntegrand
    reference_value: float | None
    reference_method: str            # "closed form" or "oracle"
    note: str = ""

    def evaluate(self, point) -> float:
        p = np.asarray(point, dtype=np.float64)
        return float(self.evaluate_batch(p[None, :])[0])


def _unit_box(d):
    return tuple((0.0, 1.0) for _ in range(d))


# ---------------------------------------------------------------- params ----
# Built with the same Python expressions as the reference so the device sees
# bit-identical constants (vp/integrands.py:131-190).

GAUSSIAN_MU = 0.5
GAUSSIAN_SIGMA = 0.01


def _gauss_params(mu, sigma):
    def fn(d):
        norm = (2.0 * math.pi * sigma ** 2) ** (-d / 2.0)
        denom = 2.0 * sigma ** 2
        return [mu, sigma, norm, denom, 1.0 / denom]
    return fn


RIDGE_N = 1000
_RIDGE_COEF = 10000.0 / (math.pi ** 2 * RIDGE_N)
_RIDGE_WINDOW = math.sqrt(46.0 / 400.0)
_SQRT_PI_OVER_2 = math.sqrt(math.pi) / 2.0


def _ridge_reference(dims: int) -> float:
    from scipy.special import erf
    c = np.arange(RIDGE_N) / (RIDGE_N - 1.0)
    axis = _SQRT_PI_OVER_2 / 10.0 * (erf(10.0 * (1.0 - c)) + erf(10.0 * c))
    return float(_RIDGE_COEF * np.sum(axis ** dims))


MP_SIGMA = 0.05
MP_MUS = (0.25, 0.5, 0.75)


def _mp_params(d):
    norm = (2.0 * math.pi * MP_SIGMA ** 2) ** (-d / 2.0)
    denom, div = 2.0 * MP_SIGMA ** 2, float(len(MP_MUS))
    return [float(len(MP_MUS)), MP_SIGMA, norm, denom, div, 1.0 / denom, 1.0 / div] + \
        list(MP_MUS)


def _erf_axis(mu, sigma):
    s = sigma * math.sqrt(2.0)
    return 0.5 * (math.erf((1.0 - mu) / s) + math.erf(mu / s))


def _genz(seed, total, d=6):
    g = np.random.default_rng(seed)
    a = g.random(d)
    u = g.random(d)
    return a * total / a.sum(), u


GENZ_OSC_A, GENZ_OSC_U = _genz(2024, 9.0)
GENZ_PP_A, GENZ_PP_U = _genz(2025, 7.25)


def _genz_osc_reference():
    z = cmath.exp(1j * 2.0 * math.pi * GENZ_OSC_U[0])
    for aj in GENZ_OSC_A:
        z *= (cmath.exp(1j * aj) - 1.0) / (1j * aj)
    return z.real


def _genz_pp_reference():
    return float(np.prod([a * (math.atan(a * (1.0 - u)) + math.atan(a * u))
                          for a, u in zip(GENZ_PP_A, GENZ_PP_U)]))


def _fixed(params):
    return lambda d: params


def _exp_axis_quad():
    from scipy.integrate import quad
    axis, _ = quad(lambda t: math.exp(t * t), 0.0, 1.0, epsabs=1e-12, epsrel=1e-12)
    return axis


# ------------------------------------------------- application integrands --

def asian_option_reference(s0, strike, rate, sigma, maturity, n_averages):
    """Closed-form value (vp/integrands.py:213-228): the exponent is normal
    with effective volatility sigma sqrt(n T), a Black-Scholes expectation."""
    m = (rate - 0.5 * sigma * sigma) * maturity
    s = sigma * math.sqrt(maturity * n_averages)
    if strike <= 0.0:
        return math.exp(-rate * maturity) * (s0 * math.exp(m + 0.5 * s * s) - strike)
    d2 = (m + math.log(s0 / strike)) / s
    d1 = d2 + s
    phi = lambda t: 0.5 * (1.0 + math.erf(t / math.sqrt(2.0)))
    return math.exp(-rate * maturity) * (
        s0 * math.exp(m + 0.5 * s * s) * phi(d1) - strike * phi(d2))


def _asian_params(s0, strike, rate, sigma, maturity):
    # device blob of vp/integrands.py:196-210's constants, same expressions
    drift = (rate - 0.5 * sigma * sigma) * maturity
    return [s0, strike, drift, sigma * math.sqrt(maturity), math.exp(-rate * maturity),
            CLAMP_EPS]


def path_integral_lattice_exact(mass, total_time, n_slices, x_end):
    """Exact lattice integral (vp/integrands.py:254-282): the action is
    quadratic in the interior points, so it is a Gaussian determinant."""
    n_int = n_slices - 1
    a = total_time / n_slices
    amp = (mass / (2.0 * math.pi * a)) ** (n_slices / 2.0)
    const = mass / a * x_end ** 2 + 0.5 * a * x_end ** 2
    if n_int == 0:
        return amp * math.exp(-const)
    h = np.zeros((n_int, n_int))
    np.fill_diagonal(h, 2.0 * mass / a + a)
    ii = np.arange(n_int - 1)
    h[ii, ii + 1] = -mass / a
    h[ii + 1, ii] = -mass / a
    b = np.zeros(n_int)
    b[0] -= mass / a * x_end
    b[-1] -= mass / a * x_end
    sol = np.linalg.solve(h, b)
    s_min = const - 0.5 * float(b @ sol)
    sign, logdet = np.linalg.slogdet(h)
    assert sign > 0
    return float(amp * math.exp(-s_min) * (2.0 * math.pi) ** (n_int / 2.0)
                 * math.exp(-0.5 * logdet))


def oscillator_propagator(omega, total_time, x_end, mass=1.0):
    """Continuum Euclidean propagator <x|e^{-HT}|x> (vp/integrands.py:285-290)."""
    wt = omega * total_time
    return math.sqrt(mass * omega / (2.0 * math.pi * math.sinh(wt))) * math.exp(
        -mass * omega * x_end ** 2 * math.tanh(wt / 2.0))


def _path_params(mass, total_time, n_slices, x_end):
    # vp/integrands.py:233-251: A exp(-(m/(2a) sum dx^2 + a/2 sum x^2))
    a = total_time / n_slices
    amp = (mass / (2.0 * math.pi * a)) ** (n_slices / 2.0)
    return [mass / (2.0 * a), 0.5 * a, amp, x_end]


def _spec_asian_option(dim=None, **params):
    """vp/integrands.py:361-377 (same parameter handling)."""
    p = dict(ASIAN_DEFAULTS)
    if dim is not None:
        p["n_averages"] = int(dim)
    p.update(params)
    n = int(p.pop("n_averages"))
    ref = asian_option_reference(n_averages=n, **p)
    blob = _asian_params(**p)
    return _spec("asian_option", n, VPB_ASIAN_OPTION, _fixed(blob), ref, "closed form",
                 f"params {dict(p, n_averages=n)}")


def _spec_path_integral(dim=None, **params):
    """vp/integrands.py:380-396 (same parameter handling)."""
    p = dict(PATH_DEFAULTS)
    if dim is not None:
        p["n_slices"] = int(dim) + 1
    p.update(params)
    n_slices = int(p["n_slices"])
    dims = n_slices - 1
    half = float(p.pop("box_half_width", PATH_BOX_HALF_WIDTH))
    if dims < 1:
        raise ContractViolationError("path_integral needs at least one interior point")
    ref = path_integral_lattice_exact(p["mass"], p["total_time"], n_slices, p["x_end"])
    blob = _path_params(p["mass"], p["total_time"], n_slices, p["x_end"])

    def params_for(d, _blob=blob, _dims=dims):
        if d != _dims:
            raise ContractViolationError(
                f"path_integral: expected {_dims} interior points, got {d}")
        return _blob

    return _spec("path_integral", dims, VPB_PATH_INTEGRAL, params_for, ref, "oracle",
                 f"lattice Gaussian determinant; params {p}",
                 bounds=tuple((-half, half) for _ in range(dims)))


# ----------------------------------------------------------------- builders --

def _spec(name, dims, dev_id, param_fn, ref, method, note="", bounds=None):
    return IntegrandSpec(name, dims, bounds or _unit_box(dims),
                         DeviceIntegrand(name, dev_id, param_fn), ref, method, note)


_BUILDERS = {
    "sinexp": lambda: _spec("sinexp", 2, VPB_SINEXP, _fixed([0.0]),
                            math.e - math.cos(1.0), "closed form"),
    "linear": lambda: _spec("linear", 10, VPB_LINEAR, _fixed([0.0]), 5.0, "closed form", "d/2"),
    "cosine": lambda: _spec("cosine", 10, VPB_COSINE, _fixed([0.0]), math.sin(1.0) ** 10,
                            "closed form", "sin(1)^d"),
    "exponential": lambda: _spec("exponential", 10, VPB_EXPONENTIAL, _fixed([0.0]),
                                 _exp_axis_quad() ** 10, "oracle",
                                 "1D quadrature, raised to d"),
    "roos_arnold": lambda: _spec("roos_arnold", 10, VPB_ROOS_ARNOLD, _fixed([0.0]), 1.0,
                                 "closed form"),
    "morokoff": lambda: _spec("morokoff", 8, VPB_MOROKOFF,
                              lambda d: [(1.0 + 1.0 / d) ** d, 1.0 / d], 1.0, "closed form",
                              "(1+1/d)^d (d/(d+1))^d = 1"),
    "gaussian": lambda: _spec("gaussian", 4, VPB_GAUSSIAN,
                              _gauss_params(GAUSSIAN_MU, GAUSSIAN_SIGMA), 1.0, "closed form",
                              "erf(0.5/(sigma sqrt(2)))^d = 1 to machine precision"),
    "ridge": lambda: _spec("ridge", 4, VPB_RIDGE,
                           _fixed([float(RIDGE_N), _RIDGE_COEF, _RIDGE_WINDOW]),
                           _ridge_reference(4), "closed form", "sum of per-axis erf products"),
    "multipeak8": lambda: _spec("multipeak8", 8, VPB_MULTIPEAK, _mp_params,
                                sum(_erf_axis(m, MP_SIGMA) ** 8 for m in MP_MUS) / 3.0,
                                "closed form", "BASELINE cfg2: 3 Gaussians on the diagonal"),
    "genz_oscillatory6": lambda: _spec(
        "genz_oscillatory6", 6, VPB_GENZ_OSCILLATORY,
        _fixed([2.0 * math.pi * GENZ_OSC_U[0]] + list(GENZ_OSC_A)), _genz_osc_reference(),
        "closed form", "BASELINE cfg4a, default_rng(2024), sum a = 9"),
    "genz_productpeak6": lambda: _spec(
        "genz_productpeak6", 6, VPB_GENZ_PRODUCTPEAK,
        _fixed(list(GENZ_PP_A ** -2.0) + list(GENZ_PP_U)), _genz_pp_reference(),
        "closed form", "BASELINE cfg4b, default_rng(2025), sum a = 7.25"),
    "asian_option": _spec_asian_option,
    "path_integral": _spec_path_integral,
    "gaussian20": lambda: _spec("gaussian20", 20, VPB_GAUSSIAN, _gauss_params(0.5, 0.1),
                                _erf_axis(0.5, 0.1) ** 20, "closed form",
                                "BASELINE cfg5: d=20, sigma=0.1"),
}

#: the Table-of-eight benchmark functions, in their conventional order
BENCHMARK_NAMES = ("sinexp", "linear", "cosine", "exponential",
                   "roos_arnold", "morokoff", "gaussian", "ridge")


#: the reference's registry (vp/integrands.py:399-415); the BASELINE-pinned
#: functions and `constant` are extras, reachable by name through lookup()
REFERENCE_NAMES = ("sinexp", "linear", "cosine", "exponential", "roos_arnold", "morokoff",
                   "gaussian", "ridge", "asian_option", "path_integral")


def available() -> list[str]:
    """The registry's names, as the reference reports them (vp/integrands.py:417-418)."""
    return sorted(REFERENCE_NAMES)


def available_all() -> list[str]:
    """Every name lookup() accepts: the reference's registry plus the
    BASELINE-pinned integrands (multipeak8, genz_*6, gaussian20) and constant."""
    return sorted(set(_BUILDERS) | {"constant"})


def constant(value: float, dims: int = 1) -> IntegrandSpec:
    """f(x) = value (exactness checks: the estimate is exact, sigma 0)."""
    v = float(value)
    return _spec("constant", dims, VPB_CONSTANT, _fixed([v]), v, "closed form")


def lookup(name: str, dim: int | None = None, **params) -> IntegrandSpec:
    """Fetch a registered device integrand (vp/integrands.py:421-436)."""
    if name == "constant":
        return constant(params.get("value", 1.0), dim or 1)
    try:
        builder = _BUILDERS[name]
    except KeyError:
        raise UnknownIntegrandError(name) from None
    if name in ("asian_option", "path_integral"):
        return builder(dim=dim, **params)
    if dim is not None or params:
        raise ValueError(f"integrand {name!r} has fixed dimension and parameters")
    return builder()


def resolve(f) -> DeviceIntegrand:
    """Map what a caller passes as ``f`` to a device functor."""
    if isinstance(f, DeviceIntegrand):
        return f
    if isinstance(f, IntegrandSpec):
        return f.evaluate_batch
    if isinstance(f, str):
        return lookup(f).evaluate_batch
    dev = getattr(f, "device_integrand", None)
    if isinstance(dev, DeviceIntegrand):
        return dev
    raise ContractViolationError(
        "the B200 backend evaluates integrands as CUDA device functors: pass a registered "
        "integrand (lookup(name), its .evaluate_batch, or its name); Python callables "
        f"cannot run inside the fused fill kernel (got {f!r})")
