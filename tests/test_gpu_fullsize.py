"""BASELINE.json's full sizes, checked through size-independent properties.

The oracle cannot run 1e8-4e9 evaluations per iteration in test time, so at
the configurations `bench.py` measures the iteration is checked against what
must hold at any size (the reference's own invariants):

* allocation (vp/strat.py:88-113): every n_h >= 2, n_eval <= sum n_h <=
  n_eval + 2 n_cubes, offsets = the exclusive prefix sum (vp/strat.py:131-137);
* the map (vp/maps.py:202-234): edges strictly increasing, end points exact;
* accumulate (vp/kernels.py:91-109): every run lands exactly once in every
  axis histogram (map counts per axis = plan total) and in its cube
  (cube counts = n_h), weights finite and non-negative -- at 4e9 runs per
  iteration (cfg5) that exercises the 64-bit run indexing and the records
  path's per-chunk slices;
* sharding (vp/executor.py:41-57): two rank shards of the full-size plan sum
  to the whole fill (counts exact, weights to the cube-sum tolerance);
* the estimate agrees with the closed form within 5 sigma.
"""

import numpy as np
import pytest

import paper_2408_09229_b200 as P

pytestmark = pytest.mark.gpu

FULL = [
    ("multipeak8", 8, 10 ** 8, 3),          # cfg2 (the headline)
    ("genz_productpeak6", 6, 10 ** 9, 2),   # cfg4b
    ("gaussian20", 20, 4 * 10 ** 9, 1),     # cfg5 (records path)
]


@pytest.mark.parametrize("name,dims,n_eval,its", FULL)
def test_full_size_iteration_invariants(name, dims, n_eval, its):
    cfg = P.IntegratorConfig(n_eval=n_eval, max_it=its + 1, n_intervals=1024)
    with P.Integrator(name, [(0.0, 1.0)] * dims, cfg) as it:
        it.iterate(its)
        est, var, ev = it.history()
        assert len(ev) == its and all(int(x) >= n_eval for x in ev)
        e = it.edges()
        assert np.all(np.diff(e, axis=1) > 0)
        assert np.all(e[:, 0] == 0.0) and np.all(e[:, -1] == 1.0)
        # one more fill at the allocation the last update produced
        it.fill(it.run_base())
        n_h, off = it.plan()
        assert n_h.min() >= 2
        assert n_eval <= int(n_h.sum()) <= n_eval + 2 * it.n_cubes
        assert off[0] == 0 and np.array_equal(np.diff(off), n_h)
        total = int(off[-1])
        mw, mc, s1, s2, cnt = it.accumulators()
        assert np.all(mc.sum(axis=1) == total)
        assert np.array_equal(cnt, n_h)
        assert np.all(np.isfinite(mw)) and mw.min() >= 0.0
        assert np.all(np.isfinite(s1)) and np.all(np.isfinite(s2)) and s2.min() >= 0.0
    ref = P.lookup(name).reference_value
    assert abs(est[-1] - ref) < 5.0 * np.sqrt(var[-1]), (est[-1], ref, np.sqrt(var[-1]))


def test_full_size_shards_sum_to_whole():
    # cfg2 after two adapted iterations: the state (map + allocation) copied
    # into two rank contexts, each filling its half of the 1e8-run plan
    cfg = P.IntegratorConfig(n_eval=10 ** 8, max_it=3, n_intervals=1024, seed=3)
    bounds = [(0.0, 1.0)] * 8
    with P.Integrator("multipeak8", bounds, cfg) as it:
        it.iterate(2)
        edges, (n_h, _), rb = it.edges(), it.plan(), it.run_base()
        it.fill(rb)
        whole = it.accumulators()
    parts = []
    for r in range(2):
        with P.Integrator("multipeak8", bounds, cfg, distributed=False) as sh:
            sh.set_edges(edges)
            sh.set_allocation(n_h)
            sh.set_shard(2, r)
            sh.fill(rb)
            parts.append(sh.accumulators())
    np.testing.assert_array_equal(parts[0][1] + parts[1][1], whole[1])
    np.testing.assert_array_equal(parts[0][4] + parts[1][4], whole[4])
    np.testing.assert_allclose(parts[0][0] + parts[1][0], whole[0], rtol=1e-12)
    np.testing.assert_allclose(parts[0][2] + parts[1][2], whole[2], rtol=1e-12, atol=1e-290)
    np.testing.assert_allclose(parts[0][3] + parts[1][3], whole[3], rtol=1e-12, atol=1e-290)
