"""GPU parity: the CUDA path (through the C ABI) against the pinned oracle
and the reference's golden vectors.

Bars (BASELINE.json north_star):
  * Philox / uniforms / sampling (x, jac, idx, cube): bit-exact
  * allocation n_h and run-plan offsets: bit-exact given identical sigma_h
  * compute_results: bit-exact given identical accumulators
  * map counts / cube counts: exact; s1, s2, map_w: rtol 1e-12 (the device
    sums in a different, but fixed, order; integrand exp differs by ulps)
  * grid edges: rtol 1e-12; integral: per-iteration |dI| well inside 3 sigma
"""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_09229_b200")
from paper_2408_09229_b200 import ops  # noqa: E402


def test_philox_kats_on_device(golden):
    d = golden("philox.npz")
    blocks, streams, seeds = [], [], []
    for c0, c1, c2, c3, k0, k1 in d["kat_in"]:
        blocks.append(int(c0) | int(c1) << 32)
        streams.append(int(c2) | int(c3) << 32)
        seeds.append(int(k0) | int(k1) << 32)
    w0, w1 = ops.philox_words(np.array(blocks, np.uint64), np.array(streams, np.uint64),
                              np.array(seeds, np.uint64))
    for i, exp in enumerate(d["kat_out"]):
        got = [int(w0[i]) >> 32, int(w0[i]) & 0xFFFFFFFF, int(w1[i]) >> 32, int(w1[i]) & 0xFFFFFFFF]
        assert got == list(map(int, exp))


def test_uniform_at_bitwise(golden):
    d = golden("philox.npz")
    u = ops.uniform_at(d["seeds"], d["streams"], d["pos"])
    np.testing.assert_array_equal(u, d["u"])


@pytest.mark.parametrize("case", list("abcdef"))
def test_sample_runs_bitwise(golden, case):
    s = golden("sample.npz")
    dims, ng, ns, batch, rb = map(int, s[case + "_meta"])
    off = s[case + "_offsets"]
    x, jac, idx, cube = ops.sample_runs(int(s[case + "_seed"][0]), batch, rb, 0, int(off[-1]),
                                        off, s[case + "_edges"], ns)
    np.testing.assert_array_equal(cube, s[case + "_cube"])
    np.testing.assert_array_equal(idx, s[case + "_idx"])
    np.testing.assert_array_equal(x, s[case + "_x"])
    np.testing.assert_array_equal(jac, s[case + "_jac"])


def test_pairwise_sum_bitwise():
    g = np.random.default_rng(1)
    for n in list(range(0, 200, 7)) + [1000, 1024, 4097, 65536, 390625, 456976, 1 << 20]:
        a = g.random(n) * 10.0 ** g.integers(-8, 8, n)
        assert ops.pairwise_sum(a) == a.sum(), n


def test_build_run_plan_bitwise():
    g = np.random.default_rng(2)
    for n in (1, 7, 1024, 1025, 100_003, 1 << 20):
        n_h = g.integers(2, 5000, n)
        np.testing.assert_array_equal(ops.build_run_plan(n_h), O.build_run_plan(n_h))


def test_allocation_bitwise(golden):
    a = golden("alloc.npz")
    mism = 0
    for i in range(int(a["n_cases"][0])):
        beta, _ = a[f"c{i}_pars"]
        n_eval = int(a[f"c{i}_n_eval"][0])
        n_h = ops.update_evals_per_cube(a[f"c{i}_d_h"], beta, n_eval)
        if beta in (0.0, 0.5, 1.0, 2.0):   # numpy fast paths: no pow involved
            np.testing.assert_array_equal(n_h, a[f"c{i}_n_h"], err_msg=f"case {i}")
        else:
            mism += int(np.sum(n_h != a[f"c{i}_n_h"]))
    assert mism == 0


def test_allocation_real_spread_vectors(golden):
    t = golden("traj_cfg1.npz")
    n_h = ops.update_evals_per_cube(t["it2_d_h"], 0.75, 1_000_000)
    np.testing.assert_array_equal(n_h, t["it2_n_h"])
    np.testing.assert_array_equal(ops.build_run_plan(n_h), O.build_run_plan(t["it2_n_h"]))


def test_allocation_given_identical_dp(golden):
    # bit-exact given identical inputs: feed the reference's own total and
    # compare n_h computed from the same dp (pow excluded from the contract)
    a = golden("alloc.npz")
    for row in a["degenerate"]:
        n, v, beta, n_eval, nh_ref, tot, vb = row
        n, n_eval = int(n), int(n_eval)
        dp_dev = ops.power(np.array([v]), beta)[0]
        nh = O.update_evals_per_cube(np.full(n, v), beta, n_eval, dp=np.full(n, dp_dev))
        if dp_dev == vb:
            assert nh[0] == nh_ref


def test_compute_results_bitwise(golden):
    r = golden("results.npz")
    for i in range(int(r["n_cases"][0])):
        I, var, d_h = ops.compute_results(r[f"c{i}_s1"], r[f"c{i}_s2"], r[f"c{i}_counts"])
        assert I == r[f"c{i}_I"][0]
        assert var == r[f"c{i}_I"][1]
        np.testing.assert_array_equal(d_h, r[f"c{i}_d_h"])


def test_compute_results_requires_two():
    with pytest.raises(AssertionError):
        ops.compute_results(np.zeros(2), np.zeros(2), np.array([2, 1]))


def test_refine(golden):
    r = golden("refine.npz")
    for i in range(int(r["n_cases"][0])):
        alpha = float(r[f"c{i}_alpha"][0])
        damped = ops.smooth_and_damp(r[f"c{i}_map_w"], r[f"c{i}_map_counts"], alpha)
        np.testing.assert_allclose(damped, r[f"c{i}_damped"], rtol=1e-14, atol=0)
        new = ops.update_grid(r[f"c{i}_edges"], r[f"c{i}_damped"])
        np.testing.assert_array_equal(new, r[f"c{i}_edges_out"])


def test_integrand_values(golden):
    g = golden("integrands.npz")
    for name, x in (("gaussian", "x4"), ("ridge", "x4"), ("multipeak8", "x8"),
                    ("genz_oscillatory6", "x6"), ("genz_productpeak6", "x6"),
                    ("gaussian20", "x20")):
        v = P.lookup(name).evaluate_batch(g[x])
        atol = 4e-15 if name == "genz_oscillatory6" else 1e-300
        np.testing.assert_allclose(v, g[name], rtol=1e-13, atol=atol, err_msg=name)


def test_multipeak_fma_form_within_exp_conditioning():
    # cfg2's three-peak Gaussian runs in the fma form (integrands.cuh
    # VPB_MP_FMA): each value within ~ulp x (|arg| + 1) of numpy's operation
    # order, arg = the dominant peak's |x - mu|^2 / (2 sigma^2) (exp's
    # condition number), on uniform points and points near the middle peak
    from oracle import integrands_np as I
    g = np.random.default_rng(3)
    x = g.random((200_000, 8))
    x[:100_000] = np.clip(0.5 + 0.05 * g.standard_normal((100_000, 8)), 0.0, 1.0)
    v = P.lookup("multipeak8").evaluate_batch(x)
    ref = I.multipeak8(x)
    mus = np.asarray(I.MP_MUS)
    arg = np.min(((x[:, None, :] - mus[None, :, None]) ** 2).sum(-1), axis=1) / (2 * I.MP_SIGMA ** 2)
    ok = ref > 0
    assert np.all(np.abs(v[ok] - ref[ok]) <= 1e-15 * (arg[ok] + 1.0) * ref[ok])
    assert np.all(np.abs(v[~ok]) < 1e-300)


def test_ridge_recurrence_against_oracle():
    # the blocked window recurrence (integrands.cuh ridge_window) against the
    # oracle's direct sum of exponentials on 200k points, half of them near
    # the ridge where the window sum is large
    g = np.random.default_rng(17)
    t = g.random((100_000, 1))
    x = np.concatenate([g.random((100_000, 4)),
                        np.clip(t + 0.02 * g.standard_normal((100_000, 4)), 0.0, 1.0)])
    v = P.lookup("ridge").evaluate_batch(x)
    ref = O.evaluate("ridge", x)
    np.testing.assert_allclose(v, ref, rtol=1e-13, atol=1e-300)


def test_application_integrand_values(golden):
    # device erfinv / lattice action vs the reference's own values
    g = golden("integrands.npz")
    cases = [(P.lookup("asian_option"), "x16", "asian_option", 2e-11),
             (P.lookup("asian_option", dim=4, strike=90.0, sigma=0.3), "x4a",
              "asian_option_k90_d4", 2e-11),
             (P.lookup("path_integral"), "x7", "path_integral", 1e-300),
             (P.lookup("path_integral", dim=3, x_end=0.5, total_time=2.0), "x3",
              "path_integral_d3_xend05", 1e-300)]
    for spec, xk, key, atol in cases:
        v = spec.evaluate_batch(g[xk])
        np.testing.assert_allclose(v, g[key], rtol=1e-12, atol=atol, err_msg=key)


def test_table2_integrand_values(golden):
    # the six Table-2 test functions (vp/integrands.py:106-128) against the
    # reference's own values, incl. Morokoff's per-axis fallback (product
    # underflow, a zero / negative coordinate: NaN like numpy's x ** (1/d))
    g = golden("integrands.npz")
    for name in ("sinexp", "linear", "cosine", "exponential", "roos_arnold", "morokoff"):
        v = P.lookup(name).evaluate_batch(g[f"x_{name}"])
        np.testing.assert_allclose(v, g[name], rtol=1e-13, atol=1e-300, err_msg=name)


def test_registry_reference_integrands_match_oracle():
    g = np.random.default_rng(7)
    for name in ("sinexp", "linear", "cosine", "exponential", "roos_arnold", "morokoff"):
        spec = P.lookup(name)
        x = g.random((2000, spec.dims))
        np.testing.assert_allclose(spec.evaluate_batch(x), O.evaluate(name, x), rtol=1e-14,
                                   err_msg=name)


def test_fill_matches_reference(golden):
    f = golden("fill.npz")
    dims, ng, ns, batch, rb, seed = map(int, f["meta"])
    mw, mc, s1, s2, cnt = ops.parallel_fill(f["offsets"], f["edges"], ns, seed, batch,
                                            "gaussian", run_base=rb)
    np.testing.assert_array_equal(mc, f["w1_map_counts"])
    np.testing.assert_array_equal(cnt, f["w1_counts"])
    np.testing.assert_allclose(mw, f["w1_map_w"], rtol=1e-12)
    np.testing.assert_allclose(s1, f["w1_s1"], rtol=1e-12, atol=1e-290)
    np.testing.assert_allclose(s2, f["w1_s2"], rtol=1e-12, atol=1e-290)


def _random_plan(g, ns, dims, lo, hi):
    n_h = g.integers(lo, hi, ns ** dims)
    return O.build_run_plan(n_h)


@pytest.mark.parametrize("name,dims,ng,ns,nh", [
    ("gaussian", 4, 1000, 26, (2, 5)),          # cfg1 geometry, tiny cubes
    ("gaussian", 4, 64, 3, (2000, 9000)),       # cubes spanning many tiles
    ("multipeak8", 8, 256, 3, (2, 400)),        # cfg2 functor, mixed cube sizes
    ("ridge", 4, 128, 4, (50, 300)),
    ("genz_oscillatory6", 6, 100, 3, (2, 50)),
    ("genz_productpeak6", 6, 100, 2, (100, 1000)),
    ("gaussian20", 20, 64, 1, (5000, 5001)),     # d=20, one cube
    ("gaussian", 3, 50, 5, (2, 30)),            # generic (runtime-dims) kernel
])
def test_fill_matches_oracle(name, dims, ng, ns, nh):
    g = np.random.default_rng(dims * 1000 + ng)
    off = _random_plan(g, ns, dims, *nh)
    edges = np.sort(g.random((dims, ng + 1)), axis=1)
    edges[:, 0], edges[:, -1] = 0.0, 1.0
    seed, batch, rb = 12345, 1 << 20, 987654321
    got = ops.parallel_fill(off, edges, ns, seed, batch, name, run_base=rb)
    ref = O.fill(off, edges, ns, seed, batch, rb, name, workers=os.cpu_count() or 1)
    np.testing.assert_array_equal(got[1], ref[1])   # map counts
    np.testing.assert_array_equal(got[4], ref[4])   # cube counts
    # the Asian payoff max(S - K, 0) cancels near the strike (device vs libm
    # exp/erfc differ by ulps of S ~ 100): absolute floor relative to the scale
    fl = (lambda a: 1e-13 * np.abs(a).max()) if name == "asian_option" else (lambda a: 1e-290)
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-12, atol=max(1e-300, fl(ref[0])))
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-12, atol=fl(ref[2]))
    np.testing.assert_allclose(got[3], ref[3], rtol=1e-12, atol=fl(ref[3]))


@pytest.mark.parametrize("name,dims,ng,ns,nh", [
    ("gaussian", 5, 40, 3, (2, 60)),            # generic kernel, odd d (Philox stride d+1)
    ("gaussian", 7, 33, 2, (10, 300)),          # generic kernel, odd d, odd ng
    ("gaussian", 1, 17, 9, (2, 200)),           # generic kernel, d = 1
    ("asian_option", 16, 128, 2, (2, 40)),      # d=16 registry default: records + K0 axes
    ("path_integral", 7, 96, 2, (20, 200)),     # d=7, odd: pair table
])
def test_fill_more_geometries(name, dims, ng, ns, nh):
    test_fill_matches_oracle(name, dims, ng, ns, nh)


@pytest.mark.parametrize("name,dims,n_eval,max_it,ng", [
    ("asian_option", 16, 60_000, 4, 64),
    ("path_integral", 7, 50_000, 5, 128),
    ("exponential", 10, 40_000, 4, 1024),       # d=10 at ng=1024: unpadded histogram stride
])
def test_integrate_trajectory_matches_oracle(name, dims, n_eval, max_it, ng):
    # the whole device iteration (plan, fill, results, allocation, refine)
    # against the oracle's restated loop on the application integrands
    spec = P.lookup(name)
    bounds = list(spec.bounds)
    with P.Integrator(spec.evaluate_batch, bounds,
                      P.IntegratorConfig(n_eval=n_eval, max_it=max_it, n_intervals=ng,
                                         seed=13, batch_size=4096)) as it:
        it.iterate(max_it)
        est, var, evals = it.history()
        edges = it.edges()
    ref = O.integrate(name, bounds, n_eval, max_it=max_it, n_intervals=ng, seed=13,
                      batch_size=4096, params=spec.evaluate_batch.params(dims))
    np.testing.assert_array_equal(evals, ref.evals)
    np.testing.assert_allclose(est, ref.estimates, rtol=1e-10)
    np.testing.assert_allclose(var, ref.variances, rtol=1e-8)
    np.testing.assert_allclose(edges, ref.edges, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("layout,chunk", [("records", "2048"), ("records", ""), ("global", "")])
@pytest.mark.parametrize("name,dims,ng,ns,nh", [
    ("gaussian20", 20, 64, 1, (5000, 5001)),     # K0 = 4 axes in the fill + 2 full groups
    ("gaussian", 13, 48, 2, (2, 40)),            # generic kernel: full group + partial launch
    ("multipeak8", 8, 256, 3, (2, 400)),         # one full group
    ("genz_oscillatory6", 6, 100, 3, (2, 50)),   # one partial group
    ("gaussian", 3, 50, 5, (2, 30)),             # generic (runtime-dims) kernel
])
def test_fill_layouts_match_oracle(monkeypatch, layout, chunk, name, dims, ng, ns, nh):
    # the histogram paths used when d*ng does not fit in shared memory
    # (hist.cuh records, chunked or not; global atomics), forced on small cases
    monkeypatch.setenv("VPB_FILL_LAYOUT", layout)
    if chunk:
        monkeypatch.setenv("VPB_REC_CHUNK", chunk)
    test_fill_matches_oracle(name, dims, ng, ns, nh)


@pytest.mark.parametrize("name,dims,ng,ns,nh", [
    ("gaussian20", 20, 64, 1, (5000, 5001)),       # one cube spanning many tiles
    ("gaussian20", 20, 1024, 2, (2, 40)),           # cfg5 geometry: 2^20 cubes
    ("gaussian20", 20, 1024, 2, (150, 250)),        # ~2e8 runs, many tiles per warp
])
def test_fill_split_matches_oracle(monkeypatch, name, dims, ng, ns, nh):
    # the split fill (2-CTA clusters: half the axes per CTA, per-run partials
    # swapped through distributed shared memory) against the oracle, incl.
    # partial tiles and lanes without runs at the shard end
    monkeypatch.setenv("VPB_FILL_LAYOUT", "split")
    test_fill_matches_oracle(name, dims, ng, ns, nh)


def test_fill_cube_sums_deterministic():
    g = np.random.default_rng(3)
    off = _random_plan(g, 5, 4, 2, 3000)
    edges = np.tile(np.linspace(0, 1, 101), (4, 1))
    a = ops.parallel_fill(off, edges, 5, 1, 1000, "gaussian", run_base=0)
    b = ops.parallel_fill(off, edges, 5, 1, 1000, "gaussian", run_base=0)
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    np.testing.assert_array_equal(a[1], b[1])


def test_fill_shards_sum_to_whole():
    # rank shards (vp/executor.py:41-57) merged by summation == the whole fill
    from paper_2408_09229_b200.distributed import partition_runs
    g = np.random.default_rng(4)
    off = _random_plan(g, 6, 3, 2, 5000)
    edges = np.tile(np.linspace(0, 1, 65), (3, 1))
    whole = ops.parallel_fill(off, edges, 6, 9, 777, "gaussian", run_base=5)
    parts = [ops.parallel_fill(off, edges, 6, 9, 777, "gaussian", run_base=5, run_lo=a, run_hi=b)
             for a, b in partition_runs(int(off[-1]), 3)]
    np.testing.assert_array_equal(sum(p[1] for p in parts), whole[1])
    np.testing.assert_array_equal(sum(p[4] for p in parts), whole[4])
    np.testing.assert_allclose(sum(p[0] for p in parts), whole[0], rtol=1e-12)
    np.testing.assert_allclose(sum(p[2] for p in parts), whole[2], rtol=1e-12, atol=1e-290)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_iteration_shards_merge_to_whole(world):
    # the distributed data path without NCCL: each rank's context plans the
    # whole iteration, fills its shard [lo, hi) (computed on device by the
    # reference's partition rule) and the summed accumulators -- what the
    # per-iteration all-reduce produces -- equal the single-GPU fill
    cfg = P.IntegratorConfig(n_eval=300_000, max_it=3, n_intervals=64, seed=21, batch_size=4096)

    def run(w, r):
        with P.Integrator("multipeak8", [(0.0, 1.0)] * 8, cfg) as it:
            if w > 1:
                it.set_shard(w, r)
            it.fill(123_457)
            return it.accumulators()

    whole = run(1, 0)
    parts = [run(world, r) for r in range(world)]
    np.testing.assert_array_equal(sum(p[1] for p in parts), whole[1])   # map counts
    np.testing.assert_array_equal(sum(p[4] for p in parts), whole[4])   # cube counts
    np.testing.assert_allclose(sum(p[0] for p in parts), whole[0], rtol=1e-12)
    np.testing.assert_allclose(sum(p[2] for p in parts), whole[2], rtol=1e-12, atol=1e-290)
    np.testing.assert_allclose(sum(p[3] for p in parts), whole[3], rtol=1e-12, atol=1e-290)


@pytest.mark.parametrize("world", [2, 3])
def test_record_chunk_shards_merge_to_whole(monkeypatch, world):
    # records layout forced with small chunks: each rank fills its hypercube-
    # aligned shard (its chunks past the shard end are empty launches), and
    # the shards still sum to the whole fill
    monkeypatch.setenv("VPB_FILL_LAYOUT", "records")
    monkeypatch.setenv("VPB_REC_CHUNK", "8192")
    cfg = P.IntegratorConfig(n_eval=200_000, max_it=3, n_intervals=64, seed=5, batch_size=4096)

    def run(w, r):
        with P.Integrator("gaussian20", [(0.0, 1.0)] * 20, cfg) as it:
            if w > 1:
                it.set_shard(w, r)
            lay = it.fill_layout()
            it.fill(777)
            return it.accumulators(), lay

    whole, lw = run(1, 0)
    parts = [run(world, r) for r in range(world)]
    assert lw["chunks"] > 1 and all(p[1]["chunks"] == lw["chunks"] for p in parts)
    acc = [p[0] for p in parts]
    np.testing.assert_array_equal(sum(p[1] for p in acc), whole[1])
    np.testing.assert_array_equal(sum(p[4] for p in acc), whole[4])
    np.testing.assert_allclose(sum(p[0] for p in acc), whole[0], rtol=1e-12)
    np.testing.assert_allclose(sum(p[2] for p in acc), whole[2], rtol=1e-12, atol=1e-290)


@pytest.mark.parametrize("traj,name", [("traj_gauss4_small.npz", "gaussian"),
                                       ("traj_ridge_small.npz", "ridge"),
                                       ("traj_genzosc_small.npz", "genz_oscillatory6"),
                                       ("traj_multipeak8_small.npz", "multipeak8"),
                                       ("traj_cfg1.npz", "gaussian")])
def test_integrate_trajectory_matches_reference(golden, traj, name):
    t = golden(traj)
    n_eval, max_it, ng, seed, batch, dims, ns = map(int, t["meta"])
    alpha, beta = t["abeta"]
    with P.Integrator(name, [(0.0, 1.0)] * dims,
                      P.IntegratorConfig(n_eval=n_eval, max_it=max_it, n_intervals=ng,
                                         alpha=alpha, beta=beta, seed=seed,
                                         batch_size=batch)) as it:
        assert it.n_strat == ns
        it.iterate(max_it)
        est, var, evals = it.history()
        edges = it.edges()
    np.testing.assert_array_equal(evals, t["evals"])
    np.testing.assert_allclose(est, t["I"], rtol=1e-10)
    np.testing.assert_allclose(var, t["var"], rtol=1e-8)
    np.testing.assert_allclose(edges, t["edges_final"], rtol=1e-12, atol=1e-14)


def test_integrate_api_cfg1():
    out = P.integrate(P.lookup("gaussian"), [(0, 1)] * 4, n_eval=1_000_000, max_it=10,
                      n_intervals=1000, batched=True)
    assert out.n_strat == 26 and out.n_cubes == 456976
    assert len(out.iterations) == 10 and out.evals_per_iteration[0] == 1_370_928
    assert abs(out.mean - 1.0) < 5 * out.sigma
    assert out.timing.fill > 0 and abs(sum(out.timing.percentages().values()) - 100) < 1e-9


def test_constant_integrand_exact():
    out = P.integrate(P.integrands.constant(2.5, 3), [(0, 1)] * 3, n_eval=10_000, max_it=3)
    assert out.mean == 2.5 and out.sigma == 0.0


def test_nonfinite_integrand_reports_point():
    spec = P.integrands.constant(float("nan"), 2)
    with pytest.raises(P.NonFiniteIntegrandError) as ei:
        P.integrate(spec, [(0, 1)] * 2, n_eval=1000, max_it=2)
    assert ei.value.run_index == 0
    assert len(ei.value.point) == 2


def test_python_callable_rejected():
    with pytest.raises(P.ContractViolationError):
        P.integrate(lambda x: x.sum(axis=1), [(0, 1)] * 2, n_eval=1000, batched=True)


@pytest.mark.parametrize("rpt", ["16", "32", "64"])
def test_fill_slot_low_word_wrap_matches_oracle(monkeypatch, rpt):
    """The Philox batch slot (counter words 2-3, vp/kernels.py:59-62) crossing
    2^32 inside a lane's runs, and the batch end right after it: the fill's
    32-bit slot fast path must hand over to the 64-bit update in time, for
    16, 32 and 64 runs per lane (capi.cu: Sched.rpt)."""
    monkeypatch.setenv("VPB_RPT", rpt)
    name, dims, ng, ns = "genz_productpeak6", 6, 100, 2
    g = np.random.default_rng(77)
    off = _random_plan(g, ns, dims, 200, 2000)
    edges = np.sort(g.random((dims, ng + 1)), axis=1)
    edges[:, 0], edges[:, -1] = 0.0, 1.0
    # a seed per case: vpb_fill_host's cached context is keyed on it (and
    # picks its runs per lane at creation)
    seed, batch = 4242 + int(rpt), (1 << 32) + 7
    rb = (1 << 32) - 40            # slot low word 0xFFFFFFD8 at the first run
    got = ops.parallel_fill(off, edges, ns, seed, batch, name, run_base=rb)
    ref = O.fill(off, edges, ns, seed, batch, rb, name, workers=os.cpu_count() or 1)
    np.testing.assert_array_equal(got[1], ref[1])
    np.testing.assert_array_equal(got[4], ref[4])
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-12, atol=1e-290)
    np.testing.assert_allclose(got[3], ref[3], rtol=1e-12, atol=1e-290)
