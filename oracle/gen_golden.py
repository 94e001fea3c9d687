"""Generate golden vectors from the REAL reference package (test infrastructure).

Run in the dev container only (it imports the read-only reference from
/root/reference/pkg/src; that tree does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

Writes small compressed fixtures under tests/golden/.  Every fixture is the
output of the reference's own functions on seeded inputs:

    philox.npz      rng._philox_words / rng.uniform_at           vp/rng.py:38-68
    sample.npz      kernels.sample_runs (lockstep cases)         vp/kernels.py:36-88
    fill.npz        executor.fill_shard / parallel_fill          vp/executor.py:86-166
    alloc.npz       strat.update_evals_per_cube / build_run_plan vp/strat.py:88-137
    results.npz     strat.compute_results                        vp/strat.py:183-208
    refine.npz      maps.smooth_and_damp / maps.update_grid      vp/maps.py:160-234
    traj_*.npz      core.integrate trajectories (per-iteration I, var, evals,
                    d_h -> n_h pairs and edges)                   vp/core.py:168-238
    integrands.npz  integrand values (gaussian, ridge) on fixed points

The script is deterministic; re-running it reproduces the same files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))

import vegasplus as vp  # noqa: E402  (the reference)
from vegasplus import executor, kernels, maps, rng, strat  # noqa: E402
from vegasplus.integrands import lookup  # noqa: E402

from oracle import integrands_np  # noqa: E402  (pinned synthetic integrands)


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sorted(arrays))


def gen_philox():
    # Random123 known-answer vectors, Philox4x32-10
    # counter (c0,c1,c2,c3) -> block = c0 | c1<<32, stream = c2 | c3<<32
    kat_in = np.array([
        [0, 0, 0, 0, 0, 0],
        [0xFFFFFFFF] * 6,
        [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0],
    ], dtype=np.uint64)
    kat_out = []
    for c0, c1, c2, c3, k0, k1 in kat_in:
        block = np.uint64(int(c0) | (int(c1) << 32))
        stream = np.uint64(int(c2) | (int(c3) << 32))
        seed = np.uint64(int(k0) | (int(k1) << 32))
        w0, w1 = rng._philox_words(block, stream, seed)
        kat_out.append([int(w0) >> 32, int(w0) & 0xFFFFFFFF,
                        int(w1) >> 32, int(w1) & 0xFFFFFFFF])
    g = np.random.default_rng(101)
    n = 2000
    seeds = g.integers(0, 2 ** 63, size=n, dtype=np.uint64) * np.uint64(2) + \
        g.integers(0, 2, size=n, dtype=np.uint64)
    streams = g.integers(0, 2 ** 63, size=n, dtype=np.uint64)
    pos = g.integers(0, 2 ** 62, size=n, dtype=np.uint64)
    # a few structured cases
    seeds[:6] = [0, 0, 1, 12345, 99, 2 ** 64 - 1]
    streams[:6] = [0, 0, 0, 7, 3, 2 ** 40 + 3]
    pos[:6] = [0, 1, 0, 0, 5, 2 ** 50 + 1]
    u = np.array([rng.uniform_at(np.uint64(s), np.uint64(t), np.uint64(p))
                  for s, t, p in zip(seeds, streams, pos)])
    save("philox.npz", kat_in=kat_in, kat_out=np.array(kat_out, dtype=np.uint64),
         seeds=seeds, streams=streams, pos=pos, u=u)


def _sample_case(seed_rng, dims, ng, n_strat, batch, seed, run_base, nh_lo, nh_hi,
                 uniform_map=False, bounds=None):
    g = np.random.default_rng(seed_rng)
    if uniform_map:
        edges = maps.new_uniform(dims, ng, bounds or [(0.0, 1.0)] * dims).edges
    else:
        edges = np.sort(g.random((dims, ng + 1)), axis=1)
        lo = np.array([b[0] for b in (bounds or [(0.0, 1.0)] * dims)])
        hi = np.array([b[1] for b in (bounds or [(0.0, 1.0)] * dims)])
        edges = lo[:, None] + edges * (hi - lo)[:, None]
        edges[:, 0] = lo
        edges[:, -1] = hi
    n_h = g.integers(nh_lo, nh_hi, size=n_strat ** dims).astype(np.int64)
    plan = strat.build_run_plan(n_h)
    n = plan.total
    x = np.empty((n, dims))
    jac = np.empty(n)
    idx = np.empty((n, dims), dtype=np.int64)
    cube = np.empty(n, dtype=np.int64)
    kernels.sample_runs(np.uint64(seed), np.int64(batch), np.int64(run_base),
                        np.int64(0), np.int64(n), plan.offsets, np.int64(0),
                        edges, np.int64(n_strat), x, jac, idx, cube)
    return dict(edges=edges, n_h=n_h, offsets=plan.offsets, x=x, jac=jac, idx=idx,
                cube=cube, meta=np.array([dims, ng, n_strat, batch, run_base], dtype=np.int64),
                seed=np.array([seed], dtype=np.uint64))


def gen_sample():
    cases = {
        # the reference lockstep test configuration (tests/test_kernels.py:10-14)
        "a": _sample_case(3, 5, 12, 3, 37, 99, 12345, 2, 7),
        # odd dims, one stratum, big run_base crossing 2^32 slots, huge seed
        "b": _sample_case(4, 3, 1000, 1, 1 << 20, 2 ** 64 - 5, (1 << 33) + 17, 2, 3000),
        # d=1, many strata, batch_size 1 (k = g)
        "c": _sample_case(5, 1, 64, 50, 1, 7, 3, 2, 5),
        # cfg1-like geometry slice: d=4, ng=1000, n_strat=5, uniform map
        "d": _sample_case(6, 4, 1000, 5, 1 << 20, 0, 0, 2, 9, uniform_map=True),
        # non-unit bounds, non-uniform map, d=6
        "e": _sample_case(7, 6, 50, 2, 1000, 2024, 999_999_937, 2, 40,
                          bounds=[(-1.0, 2.0), (0.0, 0.5), (3.0, 7.0), (-5.0, 5.0),
                                  (0.0, 1.0), (1e-3, 2e-3)]),
        # y >= 1 clamp: ng huge relative to strata, n_strat=1, many runs
        "f": _sample_case(8, 2, 7, 1, 3, 1, 2 ** 40, 2, 20000),
    }
    flat = {}
    for k, v in cases.items():
        for kk, vv in v.items():
            flat[f"{k}_{kk}"] = vv
    save("sample.npz", cases=np.array(sorted(cases)), **flat)


class _Cfg:
    def __init__(self, seed, batch_size, workers):
        self.seed = seed
        self.batch_size = batch_size
        self.workers = workers


def gen_fill():
    # fill_shard on the gaussian (d=4) with a non-uniform map and random plan.
    out = {}
    g = np.random.default_rng(11)
    dims, ng, ns = 4, 40, 3
    spec = lookup("gaussian")
    edges = np.sort(g.random((dims, ng + 1)), axis=1)
    edges[:, 0], edges[:, -1] = 0.0, 1.0
    vmap = maps.VegasMap(edges)
    n_h = g.integers(2, 60, size=ns ** dims).astype(np.int64)
    grid = strat.StratGrid(dims=dims, n_strat=ns, n_h=n_h)
    plan = strat.build_run_plan(n_h)
    for workers in (1, 3):
        mw, acc = executor.parallel_fill(plan, vmap, grid, _Cfg(5, 1000, workers),
                                         spec.evaluate_batch, run_base=777)
        out[f"w{workers}_map_w"] = mw.w
        out[f"w{workers}_map_counts"] = mw.counts
        out[f"w{workers}_s1"] = acc.s1
        out[f"w{workers}_s2"] = acc.s2
        out[f"w{workers}_counts"] = acc.counts
    out.update(edges=edges, n_h=n_h, offsets=plan.offsets,
               meta=np.array([dims, ng, ns, 1000, 777, 5], dtype=np.int64))
    save("fill.npz", **out)


def _reference_loop(f_batch, bounds, n_eval, max_it, ng, alpha=0.5, beta=0.75,
                    seed=0, batch=1 << 20, workers=1, keep_edges=(1, 2),
                    keep_keys=None):
    """core.integrate's loop (vp/core.py:188-219) with the per-iteration
    intermediates captured."""
    dims = len(bounds)
    vmap = maps.new_uniform(dims, ng, bounds)
    grid = strat.initial_grid(n_eval, dims)
    cfg = _Cfg(seed, batch, workers)
    run_base = 0
    rec = dict(I=[], var=[], evals=[], n_h0=grid.n_h.copy())
    for it in range(1, max_it + 1):
        plan = strat.build_run_plan(grid.n_h)
        mw, acc = executor.parallel_fill(plan, vmap, grid, cfg, f_batch, run_base=run_base)
        run_base += plan.total
        i_it, var_it, d_h = strat.compute_results(acc, grid.cube_volume)
        n_h = strat.update_evals_per_cube(d_h, beta, n_eval)
        damped = maps.smooth_and_damp(mw, alpha)
        new = maps.update_grid(vmap, damped)
        if it in keep_edges:
            snap = dict(edges_in=vmap.edges, map_w=mw.w, map_counts=mw.counts,
                        s1=acc.s1, s2=acc.s2, d_h=d_h, n_h=n_h, damped=damped,
                        edges_out=new.edges)
            for k, v in snap.items():
                if keep_keys is None or k in keep_keys:
                    rec[f"it{it}_{k}"] = np.array(v, copy=True)
        grid.n_h = n_h
        grid.d_h = d_h
        vmap = new
        rec["I"].append(i_it)
        rec["var"].append(var_it)
        rec["evals"].append(plan.total)
    rec["edges_final"] = vmap.edges.copy()
    rec["I"] = np.array(rec["I"])
    rec["var"] = np.array(rec["var"])
    rec["evals"] = np.array(rec["evals"], dtype=np.int64)
    rec["meta"] = np.array([n_eval, max_it, ng, seed, batch, dims, grid.n_strat],
                           dtype=np.int64)
    rec["abeta"] = np.array([alpha, beta])
    return rec


def gen_trajectories():
    # (1) small gaussian-4D trajectory: full intermediates at it 1, 2, 5
    rec = _reference_loop(lookup("gaussian").evaluate_batch, [(0.0, 1.0)] * 4,
                          n_eval=100_000, max_it=5, ng=100, keep_edges=(1, 2, 5))
    save("traj_gauss4_small.npz", **rec)
    # (2) cfg1 as specified (gaussian-4D, n_eval=1e6, 10 its, ng=1000):
    # per-iteration I/var/evals + edges; cube arrays only for it 2 (compressed)
    rec = _reference_loop(lookup("gaussian").evaluate_batch, [(0.0, 1.0)] * 4,
                          n_eval=1_000_000, max_it=10, ng=1000, keep_edges=(2,),
                          keep_keys=("edges_in", "map_w", "map_counts", "d_h", "n_h",
                                     "damped", "edges_out"))
    save("traj_cfg1.npz", **rec)
    # (3) pinned multipeak-8D at a reduced budget (cfg2 integrand), 3 its
    rec = _reference_loop(integrands_np.multipeak8, [(0.0, 1.0)] * 8,
                          n_eval=200_000, max_it=3, ng=256, keep_edges=(1,))
    save("traj_multipeak8_small.npz", **rec)
    # (4) ridge-4D at a small budget, 2 its
    rec = _reference_loop(lookup("ridge").evaluate_batch, [(0.0, 1.0)] * 4,
                          n_eval=20_000, max_it=2, ng=64, keep_edges=(1,))
    save("traj_ridge_small.npz", **rec)
    # (5) non-unit bounds, beta=0.25, alpha=1.0, batch 1000, seed 3
    rec = _reference_loop(integrands_np.genz_oscillatory6, [(0.0, 1.0)] * 6,
                          n_eval=50_000, max_it=3, ng=50, alpha=1.0, beta=0.25,
                          seed=3, batch=1000, keep_edges=(1,))
    save("traj_genzosc_small.npz", **rec)


def gen_alloc():
    g = np.random.default_rng(41)
    out = {}
    cases = []
    # real spread vectors captured from the cfg1-like trajectory
    traj = np.load(os.path.join(OUT, "traj_gauss4_small.npz"))
    for it in (1, 2, 5):
        cases.append((traj[f"it{it}_d_h"], 0.75, 100_000))
    cfg1 = np.load(os.path.join(OUT, "traj_cfg1.npz"))
    # (the cfg1 it-2 vector lives in traj_cfg1.npz; tests read it from there)
    # random
    for _ in range(12):
        n = int(g.integers(1, 5000))
        d_h = g.random(n) * g.integers(0, 2, n) * 10.0 ** g.integers(-30, 10)
        cases.append((d_h, float(g.choice([0.0, 0.25, 0.5, 0.75, 1.0, 1.7])),
                      int(g.integers(4, 10 ** 9))))
    # degenerate equal-spread vectors (pow accuracy stress): stored as specs
    degen = []
    for n, n_eval in ((7, 1000), (1000, 10 ** 6), (10 ** 6, 10 ** 9), (390625, 10 ** 8),
                      (1 << 20, 4 * 10 ** 9), (456976, 10 ** 6)):
        for v in (3.3, 1e-7, 0.123456789, 2.0 ** -20):
            for beta in (0.75, 0.25):
                n_h = strat.update_evals_per_cube(np.full(n, v), beta, n_eval)
                assert np.all(n_h == n_h[0])
                tot = (np.full(n, v) ** beta).sum()
                degen.append([n, v, beta, n_eval, n_h[0], tot, v ** beta])
    out["degenerate"] = np.array(degen, dtype=np.float64)
    cases.append((np.zeros(5), 0.75, 50))
    cases.append((np.array([5.0, 1.0, 0.0, 2.0]), 0.0, 100))
    cases.append((np.array([1.0, 3.0]), 1.0, 8))
    for i, (d_h, beta, n_eval) in enumerate(cases):
        n_h = strat.update_evals_per_cube(d_h, beta, n_eval)
        plan = strat.build_run_plan(n_h)
        out[f"c{i}_d_h"] = np.asarray(d_h, dtype=np.float64)
        out[f"c{i}_n_h"] = n_h
        out[f"c{i}_offsets"] = plan.offsets
        out[f"c{i}_pars"] = np.array([beta, float(n_eval)])
        out[f"c{i}_n_eval"] = np.array([n_eval], dtype=np.int64)
        # the reference's intermediate: the pairwise total of d_h**beta
        if beta != 0.0:
            out[f"c{i}_total"] = np.array([(np.asarray(d_h, dtype=np.float64) ** beta).sum()])
    out["n_cases"] = np.array([len(cases)])
    # initial grid for the BASELINE configs
    init = []
    for n_eval, dims in ((10 ** 6, 4), (10 ** 8, 8), (10 ** 8, 4), (10 ** 9, 6), (4 * 10 ** 9, 20)):
        gr = strat.initial_grid(n_eval, dims)
        init.append([n_eval, dims, gr.n_strat, gr.n_cubes, int(gr.n_h[0]), int(gr.n_h.sum())])
    out["initial_grids"] = np.array(init, dtype=np.int64)
    save("alloc.npz", **out)


def gen_results():
    g = np.random.default_rng(43)
    out = {}
    ncase = 0
    for n_cubes in (1, 2, 27, 1000, 4097, 20_011):
        counts = g.integers(2, 50, size=n_cubes).astype(np.int64)
        vals = g.normal(1.0, 0.5, size=(n_cubes,)) * 10.0 ** g.integers(-3, 3, size=n_cubes)
        s1 = vals * counts
        s2 = vals * vals * counts * (1.0 + g.random(n_cubes))
        acc = strat.CubeAccumulator(n_cubes)
        acc.s1[:], acc.s2[:], acc.counts[:] = s1, s2, counts
        i_it, var_it, d_h = strat.compute_results(acc, 1.0 / n_cubes)
        out[f"c{ncase}_s1"], out[f"c{ncase}_s2"], out[f"c{ncase}_counts"] = s1, s2, counts
        out[f"c{ncase}_I"] = np.array([i_it, var_it])
        out[f"c{ncase}_d_h"] = d_h
        ncase += 1
    out["n_cases"] = np.array([ncase])
    save("results.npz", **out)


def gen_refine():
    g = np.random.default_rng(47)
    out = {}
    ncase = 0
    for dims, ng, alpha in ((1, 4, 1.0), (2, 16, 0.5), (4, 1000, 0.5), (8, 1024, 0.5),
                            (3, 77, 0.0), (2, 129, 1.5), (20, 1024, 0.5)):
        mw = maps.MapWeights(dims, ng)
        mw.counts[:] = g.integers(0, 40, size=(dims, ng))
        mw.w[:] = g.random((dims, ng)) * mw.counts * 10.0 ** g.integers(-40, 5, size=(dims, ng))
        if dims >= 2:
            mw.w[1] = 0.0   # an all-zero dimension is skipped
            mw.counts[1] = 0
        bounds = [(-1.0 - j, 2.0 + 0.5 * j) for j in range(dims)]
        edges = np.sort(g.random((dims, ng + 1)), axis=1)
        lo = np.array([b[0] for b in bounds])
        hi = np.array([b[1] for b in bounds])
        edges = lo[:, None] + edges * (hi - lo)[:, None]
        edges[:, 0], edges[:, -1] = lo, hi
        damped = maps.smooth_and_damp(mw, alpha)
        new = maps.update_grid(maps.VegasMap(edges), damped)
        for k, v in dict(map_w=mw.w.copy(), map_counts=mw.counts.copy(), edges=edges,
                         damped=damped, edges_out=new.edges, alpha=np.array([alpha])).items():
            out[f"c{ncase}_{k}"] = v
        ncase += 1
    out["n_cases"] = np.array([ncase])
    save("refine.npz", **out)


def gen_integrands():
    g = np.random.default_rng(53)
    out = {}
    x4 = g.random((4096, 4))
    x4[:8] = [[0.5] * 4, [0.0] * 4, [1.0] * 4, [0.49, 0.51, 0.5, 0.5],
              [0.3, 0.3, 0.3, 0.3], [0.0, 1.0, 0.0, 1.0], [0.25] * 4, [0.75] * 4]
    out["x4"] = x4
    out["gaussian"] = lookup("gaussian").evaluate_batch(x4)
    out["ridge"] = lookup("ridge").evaluate_batch(x4)
    out["ridge_reference"] = np.array([lookup("ridge").reference_value])
    x8 = g.random((4096, 8))
    out["x8"] = x8
    out["multipeak8"] = integrands_np.multipeak8(x8)
    x6 = g.random((4096, 6))
    out["x6"] = x6
    out["genz_oscillatory6"] = integrands_np.genz_oscillatory6(x6)
    out["genz_productpeak6"] = integrands_np.genz_productpeak6(x6)
    x20 = 0.5 + 0.15 * g.standard_normal((4096, 20))
    out["x20"] = x20
    out["gaussian20"] = integrands_np.gaussian20(x20)
    # reference application integrands (vp/integrands.py:196-251), default
    # and non-default parameters, straight from the reference
    x16 = g.random((4096, 16))
    x16[:4] = [[0.0] * 16, [1.0] * 16, [0.5] * 16, [1e-13] * 16]
    out["x16"] = x16
    out["asian_option"] = lookup("asian_option").evaluate_batch(x16)
    x4a = g.random((4096, 4))
    out["x4a"] = x4a
    out["asian_option_k90_d4"] = lookup("asian_option", dim=4, strike=90.0,
                                        sigma=0.3).evaluate_batch(x4a)
    x7 = -5.0 + 10.0 * g.random((4096, 7))
    x7[:1024] *= 0.2          # points near the classical path (non-negligible weights)
    out["x7"] = x7
    out["path_integral"] = lookup("path_integral").evaluate_batch(x7)
    x3 = -5.0 + 10.0 * g.random((4096, 3))
    x3 *= 0.3
    out["x3"] = x3
    out["path_integral_d3_xend05"] = lookup("path_integral", dim=3, x_end=0.5,
                                            total_time=2.0).evaluate_batch(x3)
    # the six Table-2 test functions (vp/integrands.py:106-128) at their
    # registry dimensions, straight from the reference; drawn after all the
    # arrays above so those stay unchanged
    for name in ("sinexp", "linear", "cosine", "exponential", "roos_arnold", "morokoff"):
        spec = lookup(name)
        x = g.random((4096, spec.dims))
        x[:3] = [[0.0] * spec.dims, [1.0] * spec.dims, [0.5] * spec.dims]
        if name == "morokoff":
            # product underflow (per-axis form), a zero coordinate, off the
            # unit box (a negative coordinate: NaN in the reference, twice:
            # an even count), coordinates > 1
            x[3] = 1e-40
            x[4, 2] = 0.0
            x[5, 1] = -0.25
            x[6, 1] = x[6, 4] = -0.25
            x[7] = 3.0
        out[f"x_{name}"] = x
        with np.errstate(invalid="ignore"):
            out[name] = spec.evaluate_batch(x)
    save("integrands.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["integrands"]:
        gen_integrands()
        sys.exit(0)
    gen_philox()
    gen_sample()
    gen_fill()
    gen_trajectories()
    gen_alloc()
    gen_results()
    gen_refine()
    gen_integrands()
