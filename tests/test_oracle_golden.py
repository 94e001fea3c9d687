"""Pin the CPU oracle (oracle/vegas_oracle.c) to the reference's own outputs.

The golden vectors were produced by the real reference package
(oracle/gen_golden.py).  Integer/index/sampling work must match bit for bit;
quantities that pass through numpy's SIMD exp/log/pow (integrand values and
the damping step) match to the tolerances stated per test.
"""
import numpy as np
import pytest

import oracle as O


def test_philox_random123_kats(golden):
    d = golden("philox.npz")
    for (c0, c1, c2, c3, k0, k1), exp in zip(d["kat_in"], d["kat_out"]):
        w0, w1 = O.philox_words(int(c0) | int(c1) << 32, int(c2) | int(c3) << 32,
                                int(k0) | int(k1) << 32)
        assert [w0 >> 32, w0 & 0xFFFFFFFF, w1 >> 32, w1 & 0xFFFFFFFF] == list(map(int, exp))
    # published Random123 answers (independent of the reference)
    assert O.philox_words(0, 0, 0) == (0x6627e8d5e169c58d, 0xbc57ac4c9b00dbd8)


def test_uniform_at_matches_reference(golden):
    d = golden("philox.npz")
    u = np.array([O.uniform_at(int(s), int(t), int(p))
                  for s, t, p in zip(d["seeds"], d["streams"], d["pos"])])
    np.testing.assert_array_equal(u, d["u"])
    assert O.uniform_at(0, 0, 0) == 0.3990464708489645
    assert O.uniform_at(99, 3, 5) == 0.6347978471146558


@pytest.mark.parametrize("case", list("abcdef"))
def test_sample_runs_bitwise(golden, case):
    s = golden("sample.npz")
    dims, ng, ns, batch, rb = map(int, s[case + "_meta"])
    off = s[case + "_offsets"]
    x, jac, idx, cube = O.sample_runs(int(s[case + "_seed"][0]), batch, rb, 0, int(off[-1]),
                                      off, 0, s[case + "_edges"], ns)
    np.testing.assert_array_equal(x, s[case + "_x"])
    np.testing.assert_array_equal(jac, s[case + "_jac"])
    np.testing.assert_array_equal(idx, s[case + "_idx"])
    np.testing.assert_array_equal(cube, s[case + "_cube"])


@pytest.mark.parametrize("workers", [1, 3])
def test_fill_matches_reference(golden, workers):
    f = golden("fill.npz")
    dims, ng, ns, batch, rb, seed = map(int, f["meta"])
    mw, mc, s1, s2, cnt = O.fill(f["offsets"], f["edges"], ns, seed, batch, rb, "gaussian",
                                 workers=workers)
    k = f"w{workers}_"
    np.testing.assert_array_equal(mc, f[k + "map_counts"])
    np.testing.assert_array_equal(cnt, f[k + "counts"])
    # integrand exp: glibc vs numpy SIMD differ by <= 1-2 ulp per value
    np.testing.assert_allclose(mw, f[k + "map_w"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(s1, f[k + "s1"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(s2, f[k + "s2"], rtol=1e-13, atol=1e-300)


def test_pairwise_sum_matches_numpy():
    g = np.random.default_rng(0)
    for n in list(range(0, 300)) + [1000, 1024, 4097, 65536, 100003, 1 << 20]:
        a = g.random(n) * 10.0 ** g.integers(-8, 8, n)
        assert O.pairwise_sum(a) == a.sum()


def test_allocation_bitwise(golden):
    a = golden("alloc.npz")
    for i in range(int(a["n_cases"][0])):
        d_h = a[f"c{i}_d_h"]
        beta, _ = a[f"c{i}_pars"]
        n_eval = int(a[f"c{i}_n_eval"][0])
        # the reference's pow is numpy's SIMD pow: feed the same d**beta
        dp = d_h ** beta if beta != 0 else None
        n_h = O.update_evals_per_cube(d_h, beta, n_eval, dp=dp)
        np.testing.assert_array_equal(n_h, a[f"c{i}_n_h"], err_msg=f"case {i}")
        np.testing.assert_array_equal(O.build_run_plan(n_h), a[f"c{i}_offsets"])


def test_allocation_real_vectors_libm_pow(golden):
    # with the oracle's own (libm) pow, real spread vectors still match
    t = golden("traj_cfg1.npz")
    n_h = O.update_evals_per_cube(t["it2_d_h"], 0.75, 1_000_000)
    np.testing.assert_array_equal(n_h, t["it2_n_h"])


def test_initial_grids(golden):
    a = golden("alloc.npz")
    for n_eval, dims, ns, n_cubes, nh0, tot in a["initial_grids"]:
        assert O.compute_n_strat(int(n_eval), int(dims)) == ns
        n_h = O.update_evals_per_cube(np.zeros(int(n_cubes)), 0.0, int(n_eval))
        assert n_h[0] == nh0 and n_h.sum() == tot


def test_compute_results_bitwise(golden):
    r = golden("results.npz")
    for i in range(int(r["n_cases"][0])):
        I, var, d_h = O.compute_results(r[f"c{i}_s1"], r[f"c{i}_s2"], r[f"c{i}_counts"])
        assert I == r[f"c{i}_I"][0] and var == r[f"c{i}_I"][1]
        np.testing.assert_array_equal(d_h, r[f"c{i}_d_h"])


def test_compute_results_requires_two():
    with pytest.raises(AssertionError):
        O.compute_results(np.zeros(2), np.zeros(2), np.array([2, 1]))


def test_refine_matches_reference(golden):
    r = golden("refine.npz")
    for i in range(int(r["n_cases"][0])):
        alpha = float(r[f"c{i}_alpha"][0])
        damped = O.smooth_and_damp(r[f"c{i}_map_w"], r[f"c{i}_map_counts"], alpha)
        # numpy SIMD log (and pow for alpha not in {0.5,1,2}) vs libm: few ulp
        np.testing.assert_allclose(damped, r[f"c{i}_damped"], rtol=1e-14, atol=0)
        # update_grid on the reference's damped weights is bitwise
        new = O.update_grid(r[f"c{i}_edges"], r[f"c{i}_damped"])
        np.testing.assert_array_equal(new, r[f"c{i}_edges_out"])
        new2 = O.update_grid(r[f"c{i}_edges"], damped)
        np.testing.assert_allclose(new2, r[f"c{i}_edges_out"], rtol=1e-13, atol=1e-15)


def test_integrand_values(golden):
    g = golden("integrands.npz")
    for name, x in (("gaussian", "x4"), ("ridge", "x4"), ("multipeak8", "x8"),
                    ("genz_oscillatory6", "x6"), ("genz_productpeak6", "x6"),
                    ("gaussian20", "x20")):
        v = O.evaluate(name, g[x])
        # cos near its zeros: absolute error of the argument rounding dominates
        atol = 4e-15 if name == "genz_oscillatory6" else 1e-300
        np.testing.assert_allclose(v, g[name], rtol=2e-13, atol=atol, err_msg=name)


def test_table2_integrands(golden):
    # vp/integrands.py:106-128 (sinexp, linear, cosine, exponential,
    # roos_arnold, morokoff) against values from the reference itself
    g = golden("integrands.npz")
    for name in ("sinexp", "linear", "cosine", "exponential", "roos_arnold", "morokoff"):
        x = g[f"x_{name}"]
        with np.errstate(invalid="ignore"):
            v = O.evaluate(name, x)
        np.testing.assert_allclose(v, g[name], rtol=1e-13, atol=1e-300, err_msg=name)


def test_application_integrands(golden):
    # vp/integrands.py:196-251 (asian_option via erfinv, path_integral), default
    # and non-default parameters, against values from the reference itself.
    # The payoff max(S - K, 0) cancels near the strike: absolute tolerance.
    g = golden("integrands.npz")
    cases = [("asian_option", "x16", {}, "asian_option", 2e-11),
             ("asian_option", "x4a", dict(strike=90.0, sigma=0.3), "asian_option_k90_d4", 2e-11),
             ("path_integral", "x7", {}, "path_integral", 1e-300),
             ("path_integral", "x3", dict(x_end=0.5, total_time=2.0), "path_integral_d3_xend05",
              1e-300)]
    for name, xk, kw, key, atol in cases:
        x = g[xk]
        v = O.evaluate(name, x, O.integrand_params(name, x.shape[1], **kw))
        np.testing.assert_allclose(v, g[key], rtol=1e-12, atol=atol, err_msg=key)


@pytest.mark.parametrize("traj,name", [("traj_gauss4_small.npz", "gaussian"),
                                       ("traj_ridge_small.npz", "ridge"),
                                       ("traj_genzosc_small.npz", "genz_oscillatory6")])
def test_trajectory_matches_reference(golden, traj, name):
    t = golden(traj)
    n_eval, max_it, ng, seed, batch, dims, ns = map(int, t["meta"])
    alpha, beta = t["abeta"]
    out = O.integrate(name, [(0.0, 1.0)] * dims, n_eval, max_it=max_it, n_intervals=ng,
                      alpha=alpha, beta=beta, seed=seed, batch_size=batch)
    assert out.n_strat == ns
    np.testing.assert_array_equal(out.evals, t["evals"])
    np.testing.assert_allclose(out.estimates, t["I"], rtol=1e-11)
    np.testing.assert_allclose(out.variances, t["var"], rtol=1e-9)
    np.testing.assert_allclose(out.edges, t["edges_final"], rtol=1e-12, atol=1e-14)
