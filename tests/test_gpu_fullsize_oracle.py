"""BASELINE.json's configurations at FULL size against the CPU oracle.

The oracle (oracle/, the C restatement of vp/) runs the reference loop
(vp/core.py:200-219) at the same n_eval, seed and map size as the device,
so every per-iteration quantity can be compared, not just invariants:

* evaluations per iteration (plan.total): bitwise -- allocation
  (vp/strat.py:88-113) and the run plan are exact integer functions of the
  previous iteration's sigma_h;
* I_it to 1e-10 and var_it to 1e-8 relative, and |I - I_oracle| far inside
  3 sigma_combined (north_star's bar);
* the refined map: edges to 1e-12 relative (vp/maps.py:202-234).

The iteration counts take every configuration past run_base 2^32 where
north_star's sizes get there (cfg4: iteration 5, cfg5: iteration 2), so the
64-bit run indexing of the fill (Philox counter (k*stride + j) >> 1, slot =
g mod batch, vp/kernels.py:59-66) is compared against the oracle there too.
The oracle runs on all host cores; cfg5 (2 x 4e9 runs) is the long one.
"""

import os

import numpy as np
import pytest

import oracle as O
import paper_2408_09229_b200 as P

pytestmark = pytest.mark.gpu

WORKERS = max(1, os.cpu_count() or 1)

# (BASELINE config, integrand, dims, n_eval per iteration, iterations)
FULL = [
    ("cfg2", "multipeak8", 8, 10 ** 8, 10),
    ("cfg3", "ridge", 4, 10 ** 8, 2),
    ("cfg4a", "genz_oscillatory6", 6, 10 ** 9, 6),
    ("cfg4b", "genz_productpeak6", 6, 10 ** 9, 6),
    ("cfg5", "gaussian20", 20, 4 * 10 ** 9, 2),
]


@pytest.mark.parametrize("cfg,name,dims,n_eval,its", FULL, ids=[f[0] for f in FULL])
def test_full_size_trajectory_matches_oracle(cfg, name, dims, n_eval, its):
    bounds = [(0.0, 1.0)] * dims
    conf = P.IntegratorConfig(n_eval=n_eval, max_it=its, n_intervals=1024)
    with P.Integrator(name, bounds, conf, device=0) as it:
        it.iterate(its)
        est, var, evals = it.history()
        edges = it.edges()
    ref = O.integrate(name, bounds, n_eval, max_it=its, n_intervals=1024, workers=WORKERS)
    np.testing.assert_array_equal(evals, ref.evals)
    if cfg in ("cfg4a", "cfg4b", "cfg5"):
        assert int(np.sum(evals)) > 2 ** 32   # the last iteration's runs g = run_base + r
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-10)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-8)
    sig = np.sqrt(np.asarray(var) + np.asarray(ref.variances))
    assert np.all(np.abs(np.asarray(est) - np.asarray(ref.estimates)) < 3.0 * sig)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-12, atol=0.0)


# run_base past 2^32: the fill kernel's 32-bit tile-relative bookkeeping and
# its per-grid-stride advance of (k, slot) (fill.cuh) over plans of ~4M runs,
# i.e. several grid strides of warp tiles, against the oracle's direct g = run_base + r
@pytest.mark.parametrize("rb", [2 ** 33 + 17, 2 ** 40 + 3])
@pytest.mark.parametrize("batch", [1 << 20, 1000003])
@pytest.mark.parametrize("name,dims,ng,ns,nh", [
    ("multipeak8", 8, 256, 3, (300, 900)),         # pair table, XPERM
    ("genz_productpeak6", 6, 100, 4, (500, 1500)),  # table mode
    ("gaussian", 4, 1000, 26, (2, 20)),             # cfg1 geometry, 456,976 cubes
])
def test_fill_matches_oracle_past_2_32(rb, batch, name, dims, ng, ns, nh):
    from paper_2408_09229_b200 import ops
    g = np.random.default_rng(dims * 7 + ng)
    off = O.build_run_plan(g.integers(nh[0], nh[1], ns ** dims))
    edges = np.sort(g.random((dims, ng + 1)), axis=1)
    edges[:, 0], edges[:, -1] = 0.0, 1.0
    seed = 2024
    got = ops.parallel_fill(off, edges, ns, seed, batch, name, run_base=rb)
    ref = O.fill(off, edges, ns, seed, batch, rb, name, workers=WORKERS)
    np.testing.assert_array_equal(got[1], ref[1])   # map counts
    np.testing.assert_array_equal(got[4], ref[4])   # cube counts
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-12, atol=1e-290)
    np.testing.assert_allclose(got[3], ref[3], rtol=1e-12, atol=1e-290)
