"""Numpy definitions of the synthetic integrands pinned by BASELINE.md.

TEST INFRASTRUCTURE (oracle): only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import this.  The product evaluates these
functions as CUDA device functors (paper_2408_09229_b200/csrc/integrands.cuh).

The registry integrands ``gaussian`` and ``ridge`` follow the reference
(vp/integrands.py:131-190).  cfg2, cfg4a/b and cfg5 are NOT in the reference
registry; BASELINE.md §2 / SURVEY.md §8(d) pin them and this file is the pin:

  multipeak8          cfg2   d=8, three normalised Gaussians at mu_k = k/4,
                             sigma=0.05, weight 1/3 each; ref 0.99999847
  genz_oscillatory6   cfg4a  cos(2 pi u_1 + a.x), a,u = default_rng(2024)
                             .random(6) twice, a scaled to sum 9.0;
                             closed form 0.12339808575738723
  genz_productpeak6   cfg4b  prod 1/(a_j^-2 + (x_j-u_j)^2), default_rng(2025),
                             a scaled to sum 7.25; closed form 0.14749932919581038
  gaussian20          cfg5   d=20, mu=0.5, sigma=0.1 (sigma=0.01 underflows
                             to 0 at d=20, SURVEY §7 hard part 7)

Operation order mirrors the reference's numpy style (e.g. vp/integrands.py:135-139)
so the CPU values are reproducible; the device functors agree to a few ulp.
"""

from __future__ import annotations

import cmath
import math

import numpy as np

MP_SIGMA = 0.05
MP_DIMS = 8
MP_MUS = (0.25, 0.5, 0.75)


def multipeak8(x):
    d = x.shape[1]
    norm = (2.0 * math.pi * MP_SIGMA ** 2) ** (-d / 2.0)
    out = np.zeros(x.shape[0])
    for mu in MP_MUS:
        r2 = ((x - mu) ** 2).sum(axis=1)
        out += norm * np.exp(-r2 / (2.0 * MP_SIGMA ** 2))
    return out / 3.0


def _erf_axis(mu, sigma):
    s = sigma * math.sqrt(2.0)
    return 0.5 * (math.erf((1.0 - mu) / s) + math.erf(mu / s))


def multipeak8_reference():
    return sum(_erf_axis(mu, MP_SIGMA) ** MP_DIMS for mu in MP_MUS) / 3.0


def _genz_params(seed, total, d=6):
    g = np.random.default_rng(seed)
    a = g.random(d)
    u = g.random(d)
    a = a * total / a.sum()
    return a, u


GENZ_OSC_A, GENZ_OSC_U = _genz_params(2024, 9.0)
GENZ_PP_A, GENZ_PP_U = _genz_params(2025, 7.25)


def genz_oscillatory6(x):
    return np.cos(2.0 * math.pi * GENZ_OSC_U[0] + x @ GENZ_OSC_A)


def genz_oscillatory6_reference():
    z = cmath.exp(1j * 2.0 * math.pi * GENZ_OSC_U[0])
    for aj in GENZ_OSC_A:
        z *= (cmath.exp(1j * aj) - 1.0) / (1j * aj)
    return z.real


def genz_productpeak6(x):
    return (1.0 / (GENZ_PP_A ** -2.0 + (x - GENZ_PP_U) ** 2)).prod(axis=1)


def genz_productpeak6_reference():
    return float(np.prod([a * (math.atan(a * (1.0 - u)) + math.atan(a * u))
                          for a, u in zip(GENZ_PP_A, GENZ_PP_U)]))


G20_SIGMA = 0.1
G20_MU = 0.5


def gaussian20(x):
    d = x.shape[1]
    norm = (2.0 * math.pi * G20_SIGMA ** 2) ** (-d / 2.0)
    r2 = ((x - G20_MU) ** 2).sum(axis=1)
    return norm * np.exp(-r2 / (2.0 * G20_SIGMA ** 2))


def gaussian20_reference(d=20):
    return _erf_axis(G20_MU, G20_SIGMA) ** d
