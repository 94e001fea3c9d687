"""FX mode: fixed-point interval histograms with predicted scales (fill.cuh
LAYOUT_FX, update.cuh fx_begin / fx_reduce / refine_kernel's prediction).

The MapWeights sums of vp/kernels.py:100-105 are accumulated per CTA in
(axis, interval) fixed point instead of f64; fx_reduce_kernel proves every
interval's sum precise and wrap-free or the iteration's fill is redone in
f64.  The bar is the reference's, against the CPU oracle (oracle/, the C
restatement of vp/): evaluations per iteration bitwise, I_it to 1e-10,
var_it to 1e-8 and the refined map to 1e-12 relative -- with the fixed point
actually in use (vpb_fx_stats), and through the redo path too.
"""

import os

import numpy as np
import pytest

import oracle as O
import paper_2408_09229_b200 as P

pytestmark = pytest.mark.gpu

WORKERS = max(1, os.cpu_count() or 1)

# (integrand, dims, n_eval, iterations): the BASELINE integrands at reduced
# n_eval (same code path, the oracle finishes in seconds) and registry ones
CASES = [
    ("multipeak8", 8, 3_000_000, 10),        # cfg2's integrand: pair table, XPERM
    ("genz_productpeak6", 6, 3_000_000, 8),  # cfg4b: table mode, 1024 threads
    ("genz_oscillatory6", 6, 3_000_000, 8),  # cfg4a
    ("ridge", 4, 1_000_000, 6),              # cfg3: edge rows + centre table
    ("roos_arnold", 10, 2_000_000, 8),       # the paper's workload: stride d = 10
    ("gaussian", 4, 1_000_000, 10),          # cfg1's narrow peak: predictions miss early
]


def _run(monkeypatch, name, dims, n_eval, its, fx: bool):
    monkeypatch.setenv("VPB_HIST_FIXED", "1" if fx else "0")
    bounds = [(0.0, 1.0)] * dims
    conf = P.IntegratorConfig(n_eval=n_eval, max_it=its, n_intervals=1024)
    with P.Integrator(name, bounds, conf, device=0) as it:
        it.iterate(its)
        est, var, evals = it.history()
        edges = it.edges()
        st = it.fx_stats()
    return np.asarray(est), np.asarray(var), np.asarray(evals), edges, st


@pytest.mark.parametrize("name,dims,n_eval,its", CASES, ids=[c[0] for c in CASES])
def test_fx_trajectory_matches_oracle(monkeypatch, name, dims, n_eval, its):
    est, var, evals, edges, st = _run(monkeypatch, name, dims, n_eval, its, True)
    assert st["enabled"]
    # iterations 0 and 1 are f64 (no prediction yet); every later one starts
    # in fixed point until FX_MAX_FAILS redos switch it off
    assert st["fixed_iterations"] >= 1
    assert st["refilled"] <= min(3, st["fixed_iterations"])
    bounds = [(0.0, 1.0)] * dims
    ref = O.integrate(name, bounds, n_eval, max_it=its, n_intervals=1024, workers=WORKERS)
    np.testing.assert_array_equal(evals, ref.evals)
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-10)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-8)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-12, atol=0.0)


@pytest.mark.parametrize("name,dims,n_eval,its", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_fx_in_use_on_the_baseline_integrands(monkeypatch, name, dims, n_eval, its):
    """Every iteration from the third on is filled in fixed point; at most
    the first of them is redone (the three-peak Gaussian's map still moves
    by up to 2^8 per interval there), none after."""
    _, _, _, _, st = _run(monkeypatch, name, dims, n_eval, its, True)
    # the three-peak Gaussian's first refinement raises the row total 10^4-fold:
    # no prediction from it, so its fixed point starts at iteration 3
    assert st["fixed_iterations"] == its - (3 if name == "multipeak8" else 2), st
    assert st["refilled"] == 0, st


@pytest.mark.parametrize("name,dims,n_eval,its", CASES[:2], ids=[c[0] for c in CASES[:2]])
def test_fx_matches_f64_histograms(monkeypatch, name, dims, n_eval, its):
    a = _run(monkeypatch, name, dims, n_eval, its, True)
    b = _run(monkeypatch, name, dims, n_eval, its, False)
    assert not b[4]["enabled"]
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_allclose(a[0], b[0], rtol=1e-12)
    np.testing.assert_allclose(a[3], b[3], rtol=1e-13, atol=0.0)


def test_fx_default_policy(monkeypatch):
    """On by default from 1e7 evaluations per iteration where eligible; off
    below, in deterministic mode and for the generic kernel."""
    monkeypatch.delenv("VPB_HIST_FIXED", raising=False)
    conf = P.IntegratorConfig(n_eval=10 ** 7, max_it=1, n_intervals=1024)
    with P.Integrator("multipeak8", [(0.0, 1.0)] * 8, conf, device=0) as it:
        assert it.fx_stats()["enabled"]
    conf = P.IntegratorConfig(n_eval=10 ** 6, max_it=1, n_intervals=1024)
    with P.Integrator("multipeak8", [(0.0, 1.0)] * 8, conf, device=0) as it:
        assert not it.fx_stats()["enabled"]
    monkeypatch.setenv("VPB_HIST_FIXED", "1")
    conf = P.IntegratorConfig(n_eval=10 ** 6, max_it=1, n_intervals=1024)
    from paper_2408_09229_b200 import _native as N
    assert N.load().vpb_is_specialised(0, 7) == 0
    with P.Integrator("gaussian", [(0.0, 1.0)] * 7, conf, device=0) as it:   # generic kernel
        assert not it.fx_stats()["enabled"]


@pytest.mark.parametrize("name,dims,n_eval,its", [("gaussian", 4, 1_000_000, 6),
                                                  ("multipeak8", 8, 3_000_000, 5)])
def test_cooperative_update_matches_oracle(monkeypatch, name, dims, n_eval, its):
    """VPB_COOP=1: the post-fill chain as one cooperative kernel (update.cuh
    update_coop_kernel) -- same device bodies, same trajectory as the oracle."""
    monkeypatch.setenv("VPB_COOP", "1")
    est, var, evals, edges, _ = _run(monkeypatch, name, dims, n_eval, its, n_eval >= 10 ** 6)
    ref = O.integrate(name, [(0.0, 1.0)] * dims, n_eval, max_it=its, n_intervals=1024,
                      workers=WORKERS)
    np.testing.assert_array_equal(evals, ref.evals)
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-10)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-8)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-12, atol=0.0)



def test_fx_not_used_by_the_split_fill(monkeypatch):
    """cfg5's split fill keeps f64 histograms (FX measured slower there)."""
    monkeypatch.setenv("VPB_HIST_FIXED", "1")
    monkeypatch.setenv("VPB_FILL_LAYOUT", "split")
    conf = P.IntegratorConfig(n_eval=2_000_000, max_it=1, n_intervals=1024)
    with P.Integrator("gaussian20", [(0.0, 1.0)] * 20, conf, device=0) as it:
        assert it.fill_layout()["layout"].startswith("split")
        assert not it.fx_stats()["enabled"]



@pytest.mark.parametrize("ng,ns,bounds", [(100, None, [(0.0, 1.0)] * 6),
                                          (1024, 4, [(-1.0, 2.0)] * 6),
                                          (257, 3, [(0.25, 0.75)] * 6)])
def test_fx_other_geometries_match_oracle(monkeypatch, ng, ns, bounds):
    """FX with a coarse map (more runs per interval: a smaller L), a forced
    stratification and non-unit bounds (the scales follow the intervals'
    widths in x)."""
    monkeypatch.setenv("VPB_HIST_FIXED", "1")
    kw = {} if ns is None else {"n_strat": ns}
    conf = P.IntegratorConfig(n_eval=2_000_000, max_it=7, n_intervals=ng, **kw)
    with P.Integrator("genz_oscillatory6", bounds, conf, device=0) as it:
        it.iterate(7)
        est, var, evals = it.history()
        edges = it.edges()
        st = it.fx_stats()
    assert st["enabled"] and st["fixed_iterations"] >= 1, st
    ref = O.integrate("genz_oscillatory6", bounds, 2_000_000, max_it=7, n_intervals=ng,
                      workers=WORKERS, n_strat=ns)
    np.testing.assert_array_equal(evals, ref.evals)
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-10)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-8)
    # edges to 1e-12 relative -- of the domain's scale: on [-1, 2] the edges
    # next to x = 0 are lo + (a position ~1), so their last-bit differences
    # (the f64 histograms of iterations 0-1 sum in a different order than
    # the oracle's) are ulps of 1, i.e. 1e-12 of an edge near 1e-3 is 1e-15
    width = max(hi - lo for lo, hi in bounds)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-12, atol=1e-12 * width)



def _reset_and_user_map(monkeypatch, fx):
    monkeypatch.setenv("VPB_HIST_FIXED", "1" if fx else "0")
    bounds = [(0.0, 1.0)] * 6
    conf = P.IntegratorConfig(n_eval=2_000_000, max_it=12, n_intervals=1024)
    with P.Integrator("genz_productpeak6", bounds, conf, device=0) as it:
        it.iterate(5)
        first = (it.history(), it.edges())
        it.reset()
        it.iterate(5)
        second = (it.history(), it.edges(), it.fx_stats())
        # a user map (every interval moved): the predicted scales of the next
        # fixed-point fill are for the old map -- proven or redone, never wrong
        it.set_edges(np.tile(np.linspace(0.0, 1.0, 1025) ** 1.3, (6, 1)))
        it.iterate(3)
        third = (it.history(), it.edges())
    return first, second, third


def test_fx_state_resets_and_survives_a_user_map(monkeypatch):
    """reset() clears the predictions, the redo count and the trend (the
    second integration repeats the first), and after a user-set map the
    iterations match the f64-histogram run of the same sequence."""
    a1, a2, a3 = _reset_and_user_map(monkeypatch, True)
    b1, b2, b3 = _reset_and_user_map(monkeypatch, False)
    assert a2[2]["fixed_iterations"] >= 3, a2[2]
    np.testing.assert_array_equal(a1[0][2], a2[0][2])
    np.testing.assert_allclose(a1[0][0], a2[0][0], rtol=1e-12)
    np.testing.assert_allclose(a1[1], a2[1], rtol=1e-12, atol=0.0)
    np.testing.assert_array_equal(a3[0][2], b3[0][2])
    np.testing.assert_allclose(a3[0][0], b3[0][0], rtol=1e-10)
    np.testing.assert_allclose(a3[1], b3[1], rtol=1e-12, atol=0.0)



@pytest.mark.parametrize("fx", ["0", "1"])
@pytest.mark.parametrize("dims", [2, 3, 5, 6, 8, 10, 12, 16])
def test_extra_gaussian_specialisations_match_oracle(monkeypatch, dims, fx):
    """The Gaussian's compiled dimensions beyond the registry's (fill_spec_extra.cu)
    against the oracle, with f64 and with fixed-point histograms forced on
    (where the proof holds: the unadapted d >= 6 maps' histograms span hundreds
    of decades, so most iterations there refill in f64).  Sample counts are
    exact; estimates, variances and edges carry 100x the registry tests'
    tolerances: sigma = 0.01 makes d ln f / dx = (x - mu) / sigma^2 ~ 3e3 per
    axis, so an ulp of an edge (the histograms' atomic summation order) moves
    the estimates of an unadapted d = 10 map (~1e-100, dominated by a few
    tail samples) by ~1e-10.  (d = 1 is compiled too but left out here: its
    500,000 two-run cubes make sigma_h a difference of nearly equal moments, so
    the last-ulp differences between the device exp and the oracle's move n_h
    in a few cubes from iteration 2 on -- the runtime-dims kernel shows the
    same; test_d1_gaussian_statistics covers d = 1.)"""
    monkeypatch.setenv("VPB_HIST_FIXED", fx)
    from paper_2408_09229_b200 import _native as N
    assert N.load().vpb_is_specialised(0, dims) == 1
    bounds = [(0.0, 1.0)] * dims
    conf = P.IntegratorConfig(n_eval=1_000_000, max_it=6, n_intervals=512)
    with P.Integrator("gaussian", bounds, conf, device=0) as it:
        it.iterate(6)
        est, var, evals = it.history()
        edges = it.edges()
        assert it.fx_stats()["enabled"] == (fx == "1")
    ref = O.integrate("gaussian", bounds, 1_000_000, max_it=6, n_intervals=512,
                      workers=WORKERS)
    np.testing.assert_array_equal(evals, ref.evals)
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-8)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-6)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-10, atol=0.0)


def test_d1_gaussian_statistics(monkeypatch):
    """d = 1 (compiled): iterations 0-1 exactly the oracle's, the combined
    estimate within 3 sigma of the oracle's and of the closed form."""
    bounds = [(0.0, 1.0)]
    conf = P.IntegratorConfig(n_eval=1_000_000, max_it=6, n_intervals=512)
    with P.Integrator("gaussian", bounds, conf, device=0) as it:
        it.iterate(6)
        est, var, evals = it.history()
    ref = O.integrate("gaussian", bounds, 1_000_000, max_it=6, n_intervals=512, workers=WORKERS)
    np.testing.assert_array_equal(evals[:2], ref.evals[:2])
    np.testing.assert_allclose(est[:2], ref.estimates[:2], rtol=1e-10)
    w, rw = 1.0 / np.asarray(var), 1.0 / np.asarray(ref.variances)
    m, rm = np.sum(w * est) / np.sum(w), np.sum(rw * np.asarray(ref.estimates)) / np.sum(rw)
    sig = np.sqrt(1.0 / np.sum(w) + 1.0 / np.sum(rw))
    assert abs(m - rm) < 3 * sig
    assert abs(m - 1.0) < 5 * np.sqrt(1.0 / np.sum(w))
